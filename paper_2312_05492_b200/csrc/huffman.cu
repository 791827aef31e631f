// Histogram, canonical Huffman codebook, single-stream MSB-first encode and
// self-synchronising parallel decode for sm_100a.
//
// Reference semantics: huffman.py:60-74 (build_histogram), :77-102
// (_code_lengths: min-heap keyed by (freq, smallest symbol)), :128-160
// (Codebook.from_lengths: canonical (length, symbol) order), :167-202 and
// _kernels.py:36-92 (one MSB-first stream over all n codes, no chunk index;
// decode of exactly n codes, TruncatedStream on exhaustion / >32-bit codes).
#include "common.cuh"

namespace cszi {
void launch_zero16(void *p, u64 bytes, cudaStream_t st);

// ---------------------------------------------------------------------------
// histogram of int32 codes (fine-grained API; the compress path bins inside
// the predictor kernel)
// ---------------------------------------------------------------------------
__global__ void k_hist_i32(const int32_t *__restrict__ codes, u64 n, int R, u64 *hist,
                           cszi_ctl *ctl) {
  extern __shared__ uint32_t hs[];
  const int nb = 2 * R;
  const bool sm = nb <= 8192;
  if (sm)
    for (int i = threadIdx.x; i < nb; i += blockDim.x) hs[i] = 0;
  __syncthreads();
  bool bad = false;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
       i += (u64)gridDim.x * blockDim.x) {
    const int64_t c = codes[i];
    if (c <= -R || c >= R) {
      bad = true;
      continue;
    }
    if (sm) atomicAdd(&hs[c + R], 1u);
    else atomicAdd(&hist[c + R], 1ull);
  }
  if (bad) atomicOr(&ctl->flags, 0x80000000u);  // OutOfRange marker
  __syncthreads();
  if (sm)
    for (int i = threadIdx.x; i < nb; i += blockDim.x)
      if (hs[i]) atomicAdd(&hist[i], (u64)hs[i]);
}

// ---------------------------------------------------------------------------
// codebook: lengths (two-queue merge == heap merge order) + canonical words
// ---------------------------------------------------------------------------
// The heap of huffman.py:77-102 pops the minimum (freq, minsym) key.  Leaves
// sorted by that key plus internal nodes in creation order form two sorted
// queues (an internal node created later never has a smaller key: equal
// frequencies imply its children had larger minimum symbols), so popping
// the smaller queue head reproduces the heap's merge sequence exactly.
constexpr int CB_NT = 1024;

DEV void bitonic_sort_u64(u64 *keys, int n_pow2) {
  for (int k = 2; k <= n_pow2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n_pow2; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const u64 a = keys[i], b = keys[ixj];
          const bool up = (i & k) == 0;
          if ((a > b) == up) {
            keys[i] = b;
            keys[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
}

// Canonical words from lengths (huffman.py:128-160).  Also emits the decode
// tables when `dec` != nullptr.
struct DecTables {
  uint32_t lut[4096];  // 12-bit prefix -> sym | len << 16 (len 0: slow path)
  u64 first_code[33];
  uint32_t first_index[33];
  uint32_t counts[33];
  uint32_t max_len;
  uint32_t pad_;
  // followed by uint16 sorted symbols [nbins]
};

DEV void canonical_block(const uint8_t *len_s, int nbins, uint32_t *words, DecTables *dec,
                         uint16_t *sorted_out, cszi_ctl *ctl) {
  __shared__ uint32_t cnt[33];
  __shared__ uint32_t fidx[33];
  __shared__ u64 fcode[33];
  __shared__ uint32_t maxlen;
  if (threadIdx.x < 33) cnt[threadIdx.x] = 0;
  if (threadIdx.x == 0) maxlen = 0;
  __syncthreads();
  bool over = false;
  for (int s = threadIdx.x; s < nbins; s += blockDim.x) {
    const uint32_t l = len_s[s];
    if (l > 32) over = true;
    else if (l) {
      atomicAdd(&cnt[l], 1u);
      atomicMax(&maxlen, l);
    }
  }
  if (over) atomicOr(&ctl->flags, (uint32_t)CSZI_F_LENGTH_OVERFLOW);
  __syncthreads();
  if (threadIdx.x == 0) {
    u64 code = 0;
    uint32_t idx = 0;
    int prev = 0;
    for (int l = 1; l <= 32; ++l) {
      fidx[l] = idx;
      if (cnt[l]) {
        code <<= (l - prev);
        fcode[l] = code;
        code += cnt[l];
        prev = l;
      } else {
        fcode[l] = 0;
      }
      idx += cnt[l];
    }
    fcode[0] = 0;
    fidx[0] = 0;
    ctl->max_len = maxlen;
  }
  __syncthreads();
  // rank of each symbol inside its length class, in symbol order: one warp
  // per length walks the symbols with ballots.
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int l = 1 + warp; l <= 32; l += blockDim.x >> 5) {
    if (!cnt[l]) continue;
    uint32_t rank = 0;
    for (int base = 0; base < nbins; base += 32) {
      const int s = base + lane;
      const bool hit = s < nbins && len_s[s] == (uint32_t)l;
      const uint32_t m = __ballot_sync(CSZI_FULL, hit);
      if (hit) {
        const uint32_t r = rank + __popc(m & ((1u << lane) - 1));
        if (words) words[s] = (uint32_t)(fcode[l] + r);
        if (sorted_out) sorted_out[fidx[l] + r] = (uint16_t)s;
      }
      rank += __popc(m);
    }
  }
  for (int s = threadIdx.x; s < nbins; s += blockDim.x)
    if (words && len_s[s] == 0) words[s] = 0;
  if (dec) {
    for (int l = threadIdx.x; l < 33; l += blockDim.x) {
      dec->first_code[l] = fcode[l];
      dec->first_index[l] = fidx[l];
      dec->counts[l] = cnt[l];
    }
    if (threadIdx.x == 0) dec->max_len = maxlen;
    __syncthreads();
    // LUT: first match by ascending length among lengths <= 12
    for (int p = threadIdx.x; p < 4096; p += blockDim.x) {
      uint32_t e = 0;
      for (int l = 1; l <= 12; ++l) {
        if (!cnt[l]) continue;
        const u64 cur = (u64)(p >> (12 - l));
        if (cur >= fcode[l] && cur - fcode[l] < cnt[l]) {
          const uint32_t sym = sorted_out[fidx[l] + (uint32_t)(cur - fcode[l])];
          e = sym | ((uint32_t)l << 16);
          break;
        }
      }
      dec->lut[p] = e;
    }
  }
}

__global__ void __launch_bounds__(CB_NT) k_codebook(const u64 *__restrict__ hist, int nbins,
                                                    uint8_t *lengths, uint32_t *words,
                                                    cszi_ctl *ctl, int set_bits) {
  // shared layout: keys[npow2] | ik[nbins] | parent[2*nbins] | dep[nbins] | len[nbins]
  extern __shared__ __align__(16) unsigned char sm_raw[];
  int npow2 = 1;
  while (npow2 < nbins) npow2 <<= 1;
  u64 *keys = reinterpret_cast<u64 *>(sm_raw);
  u64 *ik = keys + npow2;
  int32_t *parent = reinterpret_cast<int32_t *>(ik + nbins);
  int32_t *dep = parent + 2 * nbins;
  uint8_t *len_s = reinterpret_cast<uint8_t *>(dep + nbins);
  __shared__ int alive;
  __shared__ int overflow;
  if (threadIdx.x == 0) {
    alive = 0;
    overflow = 0;
  }
  __syncthreads();
  // compact the non-empty bins (any order: they are sorted next), so the
  // sort runs over the next power of two of the leaf count (31 leaves at
  // the bench's 1e-3) instead of all 2R bins
  for (int s = threadIdx.x; s < nbins; s += blockDim.x) {
    const u64 f = hist[s];
    len_s[s] = 0;
    if (f) keys[atomicAdd(&alive, 1)] = (f << 16) | (u64)s;
  }
  __syncthreads();
  const int m = alive;
  int mp2 = 1;
  while (mp2 < m) mp2 <<= 1;
  for (int s = m + threadIdx.x; s < mp2; s += blockDim.x) keys[s] = ~0ull;
  __syncthreads();
  if (m == 0) {
    if (threadIdx.x == 0) ctl->flags |= CSZI_F_EMPTY_HISTOGRAM;
    for (int s = threadIdx.x; s < nbins; s += blockDim.x) {
      lengths[s] = 0;
      words[s] = 0;
    }
    return;
  }
  bitonic_sort_u64(keys, mp2);
  // keys[0..m) = leaves sorted by (freq, symbol); leaf i is node i,
  // internal node k (creation order) is node m + k.
  if (threadIdx.x == 0) {
    if (m == 1) {
      len_s[keys[0] & 0xffff] = 1;
    } else {
      int li = 0, ii = 0, ni = 0;
      for (int step = 0; step < m - 1; ++step) {
        int pick[2];
        u64 pk[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const bool take_leaf = li < m && (ii >= ni || keys[li] < ik[ii]);
          if (take_leaf) {
            pick[r] = li;
            pk[r] = keys[li];
            li++;
          } else {
            pick[r] = m + ii;
            pk[r] = ik[ii];
            ii++;
          }
        }
        const u64 f = (pk[0] >> 16) + (pk[1] >> 16);
        const u64 ms = min(pk[0] & 0xffffull, pk[1] & 0xffffull);
        parent[pick[0]] = m + ni;
        parent[pick[1]] = m + ni;
        ik[ni] = (f << 16) | ms;
        ni++;
      }
      // depth = number of merges above a node; parents are created later
      dep[m - 2] = 0;  // root = internal node m-2
      for (int k = m - 3; k >= 0; --k) dep[k] = dep[parent[m + k] - m] + 1;
      int ovf = 0;
      for (int i = 0; i < m; ++i) {
        const int d = dep[parent[i] - m] + 1;
        if (d > 32) ovf = 1;
        len_s[keys[i] & 0xffff] = (uint8_t)min(d, 255);
      }
      overflow = ovf;
    }
  }
  __syncthreads();
  if (overflow && threadIdx.x == 0) ctl->flags |= CSZI_F_LENGTH_OVERFLOW;
  // set_bits: stream length = sum of count x length (what k_total_bits
  // computes; the encoder's scan rewrites the same value), one launch less
  // for cszi_compress (a slab encode's histogram is not this one)
  __shared__ u64 bsum[CB_NT / 32];
  u64 bits = 0;
  for (int s = threadIdx.x; s < nbins; s += blockDim.x) {
    lengths[s] = len_s[s];
    bits += hist[s] * len_s[s];
  }
  bits = warp_sum(bits);
  if ((threadIdx.x & 31) == 0) bsum[threadIdx.x >> 5] = bits;
  __syncthreads();
  if (threadIdx.x < 32) {
    bits = (threadIdx.x < (int)(blockDim.x >> 5)) ? bsum[threadIdx.x] : 0;
    bits = warp_sum(bits);
    if (threadIdx.x == 0 && set_bits) ctl->bits = bits;
  }
  canonical_block(len_s, nbins, words, nullptr, nullptr, ctl);
}

__global__ void __launch_bounds__(CB_NT) k_canonical(const uint8_t *__restrict__ lengths,
                                                     int nbins, uint32_t *words,
                                                     DecTables *dec, cszi_ctl *ctl,
                                                     u64 expect_raw_len) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  // pass-2 length check of the decompress path (was its own 1-thread launch)
  if (expect_raw_len && threadIdx.x == 0 && ctl->raw_len != expect_raw_len)
    atomicOr(&ctl->flags, (uint32_t)CSZI_F_P2_LENGTH);
  uint8_t *len_s = sm_raw;
  for (int s = threadIdx.x; s < nbins; s += blockDim.x) len_s[s] = lengths[s];
  __syncthreads();
  uint16_t *sorted = dec ? reinterpret_cast<uint16_t *>(dec + 1) : nullptr;
  canonical_block(len_s, nbins, words, dec, sorted, ctl);
}

// ---------------------------------------------------------------------------
// encode: one MSB-first stream (count -> scan -> pack), warp-granular
// ---------------------------------------------------------------------------
// The unit of work is a warp chunk of ENC_CH = 1024 symbols (32 per lane), so
// no phase needs a block barrier and the ~40 resident warps of an SM stream
// independently (a block-tile look-back encoder was latency-bound: every
// 16 KB tile waited a chain of L2 round trips for its offset):
//   k_enc_count  per chunk: code-length and outlier totals,
//   k_scan_pair  exclusive prefixes of both (decoupled look-back),
//   k_enc_pack   per chunk: a warp scan gives each lane its bit offset,
//                codes are packed MSB-first in a 64-bit register accumulator
//                and ORed as whole 32-bit words into a per-warp shared
//                buffer, funnel-shifted to the chunk's global bit offset and
//                stored coalesced; the two words a chunk shares with its
//                neighbours are merged with one 64-bit atomic (second arriver
//                writes).  The next chunk's symbols load while one is packed.
// Outliers (symbol 0 in MODE 0) are compacted in flat order on the way.
constexpr int ENC_NT = 256;
constexpr int ENC_NW = ENC_NT / 32;
constexpr int ENC_SPT = 32;
constexpr int ENC_CH = 32 * ENC_SPT;
constexpr int ENC_SW = ENC_CH + 2;  // staged words per warp (max 32 bits per symbol)

struct EncScratch {
  uint16_t *lane_pre;  // per chunk, per lane: bit offset of the lane inside the chunk
  uint32_t *ch_bits;
  uint32_t *ch_out;
  u64 *bit_off;
  u64 *out_off;
  u64 *st_bits;  // look-back status of the pair scan
  u64 *st_out;
  uint32_t *ticket;
  uint32_t *nz_lane;  // bitmap path: per super-chunk and lane, packed exclusive prefixes
};


// Symbols of one lane: MODE 0 keeps the uint16 pairs packed (16 regs),
// MODE 1 (int32 codes of the fine-grained API) holds validated indices.
// Positions past n read as the zero-length LUT entry `nbins`.
template <int MODE> struct EncSyms;
template <> struct EncSyms<0> {
  uint32_t w[ENC_SPT / 2];
  DEV uint32_t get(int j) const { return (j & 1) ? (w[j >> 1] >> 16) : (w[j >> 1] & 0xffffu); }
  DEV void load(const void *src, u64 n, int, int nbins, u64 base, bool &) {
    const uint16_t *sp = reinterpret_cast<const uint16_t *>(src) + base;
    if (base + ENC_SPT <= n && (((uintptr_t)sp) & 15) == 0) {
#pragma unroll
      for (int q = 0; q < ENC_SPT / 8; ++q) {
        const uint4 a = __ldcs(reinterpret_cast<const uint4 *>(sp) + q);
        w[4 * q] = a.x;
        w[4 * q + 1] = a.y;
        w[4 * q + 2] = a.z;
        w[4 * q + 3] = a.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < ENC_SPT; j += 2) {
        const uint32_t lo = (base + j < n) ? sp[j] : (uint32_t)nbins;
        const uint32_t hi = (base + j + 1 < n) ? sp[j + 1] : (uint32_t)nbins;
        w[j >> 1] = lo | (hi << 16);
      }
    }
  }
};
template <> struct EncSyms<1> {
  uint32_t s[ENC_SPT];
  uint32_t w[ENC_SPT / 2];  // unused (MODE 0 fast path only)
  DEV uint32_t get(int j) const { return s[j]; }
  DEV void load(const void *src, u64 n, int R, int nbins, u64 base, bool &unknown) {
    const int32_t *cp = reinterpret_cast<const int32_t *>(src) + base;
#pragma unroll
    for (int j = 0; j < ENC_SPT; ++j) {
      if (base + j < n) {
        const int64_t v = (int64_t)cp[j] + R;
        const bool ok = v >= 0 && v < nbins;
        unknown |= !ok;
        s[j] = ok ? (uint32_t)v : (uint32_t)nbins;
      } else {
        s[j] = (uint32_t)nbins;
      }
    }
  }
};

// LUT of (word, length) per symbol; MODE 0 codes the outlier sentinel 0 as
// symbol R (huffman.py:60-74 counts outliers as code 0); [nbins] = (0, 0).
template <int MODE>
DEV void enc_load_lut(uint2 *lut, const uint8_t *lengths, const uint32_t *words, int R) {
  const int nbins = 2 * R;
  for (int i = threadIdx.x; i <= nbins; i += blockDim.x) {
    const int sI = (MODE == 0 && i == 0) ? R : i;
    lut[i] = (i == nbins) ? make_uint2(0u, 0u) : make_uint2(words[sI], lengths[sI]);
  }
}

template <int MODE>
DEV uint32_t enc_bits(const EncSyms<MODE> &sy, const uint2 *lut, int nbins, bool &unknown,
                      uint32_t &outmask, uint32_t zz2) {
  uint32_t nbits = 0;
  outmask = 0;
#pragma unroll
  for (int j = 0; j < ENC_SPT; j += 2) {
    if (MODE == 0 && sy.w[j >> 1] == zz2) {  // two 1-bit "0" codewords
      nbits += 2;
      continue;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t s = sy.get(j + h);
      const uint32_t l = lut[s].y;
      unknown |= (l == 0) && (s != (uint32_t)nbins);
      nbits += l;
      if (MODE == 0) outmask |= (uint32_t)(s == 0) << (j + h);
    }
  }
  return nbits;
}

// Sparse stream (MODE 0): R owns the 1-bit "0" codeword and at most n/8
// symbols are not R (every other codeword has >= 2 bits, so bits - n bounds
// their count).  The stream is then zeroed and only the codewords holding
// 1-bits are ORed in at their offsets (k_enc_sparse); otherwise k_enc_pack
// packs every chunk.  Both kernels evaluate the same predicate on device.
DEV bool enc_sparse(const uint8_t *lengths, const uint32_t *words, int R, u64 n,
                    const cszi_ctl *ctl) {
  const u64 bits = ctl->bits;
  return lengths[R] == 1 && words[R] == 0 && bits >= n && (bits - n) <= n / 8;
}

// k_enc_count: lengths and outlier flags come from one u32 LUT entry
// (length | outlier << 16) so a lane sums both with one add per symbol.
template <int MODE>
__global__ void __launch_bounds__(ENC_NT) k_enc_count(const void *__restrict__ src, u64 n, int R,
                                                     const uint8_t *__restrict__ lengths,
                                                     EncScratch S, u64 nch, cszi_ctl *ctl,
                                                     const uint32_t *skip_words) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  // the k_enc_nz_* kernels encode the sparse case (ctl->bits known beforehand)
  if (skip_words && enc_sparse(lengths, skip_words, R, n, ctl)) return;
  uint32_t *lut = reinterpret_cast<uint32_t *>(sm_raw);
  const int nbins = 2 * R;
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i <= nbins; i += blockDim.x) {
    const int sI = (MODE == 0 && i == 0) ? R : i;
    lut[i] = (i == nbins) ? 0u : ((uint32_t)lengths[sI] | ((MODE == 0 && i == 0) ? 0x10000u : 0u));
  }
  const uint32_t zz2 = (MODE == 0 && lengths[R] == 1) ? ((uint32_t)R | ((uint32_t)R << 16))
                                                     : 0xffffffffu;
  __syncthreads();
  bool unknown = false;
  const u64 stride = (u64)gridDim.x * ENC_NW;
  u64 c = (u64)blockIdx.x * ENC_NW + (threadIdx.x >> 5);
  EncSyms<MODE> sy;
  if (c < nch) sy.load(src, n, R, nbins, c * ENC_CH + (u64)lane * ENC_SPT, unknown);
  while (c < nch) {
    const u64 cn = c + stride;
    EncSyms<MODE> nx;
    if (cn < nch) nx.load(src, n, R, nbins, cn * ENC_CH + (u64)lane * ENC_SPT, unknown);
    uint32_t acc = 0;
#pragma unroll
    for (int j = 0; j < ENC_SPT; j += 2) {
      if (MODE == 0 && sy.w[j >> 1] == zz2) {  // two 1-bit "0" codewords
        acc += 2;
        continue;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t e = lut[sy.get(j + h)];
        // MODE 1: a symbol inside the code range without a codeword; MODE 0
        // symbols come from the predictor whose histogram built the codebook
        if (MODE == 1) unknown |= (e == 0) && (sy.get(j + h) != (uint32_t)nbins);
        acc += e;
      }
    }
    // lane offsets inside the chunk (bits < 2^15 per chunk: u16) for the
    // sparse packer, chunk totals for the scan
    const uint32_t incl = warp_incl_scan(acc);
    if (MODE == 0) S.lane_pre[c * 32 + lane] = (uint16_t)((incl - acc) & 0xffffu);
    if (lane == 31) {
      S.ch_bits[c] = incl & 0xffffu;
      S.ch_out[c] = incl >> 16;
    }
    sy = nx;
    c = cn;
  }
  if (unknown) atomicOr(&ctl->flags, (uint32_t)CSZI_F_UNKNOWN_SYMBOL);
}

// exclusive prefixes of (bits, outliers) per chunk; totals -> ctl
constexpr int PS_NT = 256, PS_IPT = 8, PS_TILE = PS_NT * PS_IPT;
__global__ void __launch_bounds__(PS_NT) k_scan_pair(EncScratch S, u64 nch, int mode,
                                                    uint32_t *out, u64 cap_words, cszi_ctl *ctl,
                                                    uint32_t bit_base, const uint8_t *p_len,
                                                    const uint32_t *p_words, int R, u64 n,
                                                    int when) {
  __shared__ u64 ws[PS_NT / 32 + 1];
  __shared__ u64 s_t, s_pb, s_po;
  // when: 0 always, 1 dense streams only, 2 sparse streams only.  The two
  // conditional launches draw tickets from separate counters, so the ticket
  // is requested together with the predicate's loads (one latency, not two).
  if (threadIdx.x == 0) s_t = atomicAdd(S.ticket + (when == 2 ? 1 : 0), 1u);
  if (when && enc_sparse(p_len, p_words, R, n, ctl) != (when == 2)) return;
  __syncthreads();
  const u64 t = s_t;
  const u64 base = t * PS_TILE + (u64)threadIdx.x * PS_IPT;
  uint32_t vb[PS_IPT], vo[PS_IPT];
  u64 sb = 0, so = 0;
#pragma unroll
  for (int i = 0; i < PS_IPT; ++i) {
    vb[i] = (base + i < nch) ? S.ch_bits[base + i] : 0u;
    vo[i] = (base + i < nch) ? S.ch_out[base + i] : 0u;
    sb += vb[i];
    so += vo[i];
  }
  u64 tb, to;
  const u64 eb = block_excl_scan<PS_NT, u64>(sb, ws, tb);
  const u64 eo = block_excl_scan<PS_NT, u64>(so, ws, to);
  if (threadIdx.x < 32) {
    const u64 p = lookback_exclusive(S.st_bits, t, tb);
    if (threadIdx.x == 0) s_pb = p;
  } else if (threadIdx.x < 64) {
    const u64 p = lookback_exclusive(S.st_out, t, to);
    if (threadIdx.x == 32) s_po = p;
  }
  __syncthreads();
  u64 rb = s_pb + eb, ro = s_po + eo;
#pragma unroll
  for (int i = 0; i < PS_IPT; ++i) {
    if (base + i < nch) {
      S.bit_off[base + i] = rb;
      S.out_off[base + i] = ro;
      // a word holding an unaligned chunk boundary is ORed by both chunks
      // (the bitmap path zeroed the whole stream already)
      const u64 ab = rb + bit_base;  // bit position in the output words
      if (when != 2 && (ab & 31) && (ab >> 5) < cap_words) out[ab >> 5] = 0u;
    }
    rb += vb[i];
    ro += vo[i];
  }
  if ((t + 1) * PS_TILE >= nch && threadIdx.x == 0) {
    ctl->bits = s_pb + tb;
    if (mode == 0) ctl->n_outliers = s_po + to;
  }
}

// zero the sparse stream's words [0, bits + bit_base + 1 word), grid-strided
DEV void zero_stream(uint32_t *out, u64 cap_words, const cszi_ctl *ctl, uint32_t bit_base) {
  u64 nw = (ctl->bits + bit_base + 31) / 32 + 1;
  if (nw > cap_words) nw = cap_words;
  // words up to the first 16-byte boundary, then 16-byte stores
  const u64 lead = min((u64)(((16 - (reinterpret_cast<uintptr_t>(out) & 15)) & 15) / 4), nw);
  const u64 tid = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  const u64 nthr = (u64)gridDim.x * blockDim.x;
  if (tid < lead) out[tid] = 0u;
  uint4 *o4 = reinterpret_cast<uint4 *>(out + lead);
  const u64 nv = (nw - lead) / 4;
  for (u64 i = tid; i < nv; i += nthr) o4[i] = make_uint4(0, 0, 0, 0);
  for (u64 i = lead + nv * 4 + tid; i < nw; i += nthr) out[i] = 0u;
}

__global__ void k_enc_zero(const uint8_t *lengths, const uint32_t *words, int R, u64 n,
                           uint32_t *out, u64 cap_words, const cszi_ctl *ctl, uint32_t bit_base) {
  if (!enc_sparse(lengths, words, R, n, ctl)) return;
  zero_stream(out, cap_words, ctl, bit_base);
}

// OR one codeword (word, len) into the zeroed MSB-first stream at bit pos.
DEV void sp_put(uint32_t *out, u64 cap_words, u64 pos, uint32_t word, uint32_t len,
                bool &cap_hit) {
  const u64 w = pos >> 5;
  const uint32_t off = (uint32_t)(pos & 31);
  if (w + 1 >= cap_words) {
    cap_hit = true;
  } else if (off + len <= 32) {
    atomicOr(out + w, bswap32(word << (32 - off - len)));
  } else {
    const uint32_t sh = off + len - 32;  // bits spilling into word w + 1
    atomicOr(out + w, bswap32(word >> sh));
    atomicOr(out + w + 1, bswap32(word << (32 - sh)));
  }
}

__global__ void __launch_bounds__(ENC_NT, 3) k_enc_sparse(const uint16_t *__restrict__ src, u64 n,
                                                          int R, const uint8_t *__restrict__ lengths,
                                                          const uint32_t *__restrict__ words,
                                                          uint32_t *__restrict__ out, u64 cap_words,
                                                          const float *__restrict__ xval,
                                                          u64 *o_idx, float *o_val, u64 o_cap,
                                                          EncScratch S, u64 nch, u64 idx_offset,
                                                          cszi_ctl *ctl, uint32_t bit_base) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  if (!enc_sparse(lengths, words, R, n, ctl)) return;
  const int nbins = 2 * R;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint2 *lut = reinterpret_cast<uint2 *>(sm_raw);
  enc_load_lut<0>(lut, lengths, words, R);
  const uint32_t zz2 = (uint32_t)R | ((uint32_t)R << 16);
  __syncthreads();
  bool unknown = false, cap_hit = false;
  const u64 stride = (u64)gridDim.x * ENC_NW;
  u64 c = (u64)blockIdx.x * ENC_NW + warp;
  EncSyms<0> sy;
  if (c < nch) sy.load(src, n, R, nbins, c * ENC_CH + (u64)lane * ENC_SPT, unknown);
  while (c < nch) {
    const u64 cn = c + stride;
    EncSyms<0> nx;
    if (cn < nch) nx.load(src, n, R, nbins, cn * ENC_CH + (u64)lane * ENC_SPT, unknown);
    const u64 ob = S.out_off[c];
    u64 pos = S.bit_off[c] + bit_base + S.lane_pre[c * 32 + lane];
    uint32_t outmask = 0;
#pragma unroll
    for (int j = 0; j < ENC_SPT; j += 2) {
      if (sy.w[j >> 1] == zz2) {
        pos += 2;
        continue;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t s = sy.get(j + h);
        const uint2 e = lut[s];
        outmask |= (uint32_t)(s == 0) << (j + h);
        if (e.x) sp_put(out, cap_words, pos, e.x, e.y, cap_hit);
        pos += e.y;
      }
    }
    if (__any_sync(CSZI_FULL, outmask != 0)) {
      const uint32_t no = (uint32_t)__popc(outmask);
      u64 k = ob + (warp_incl_scan(no) - no);
      const u64 base = c * ENC_CH + (u64)lane * ENC_SPT;
      for (uint32_t mm = outmask; mm; mm &= mm - 1) {
        const u64 gi = base + (__ffs(mm) - 1);
        if (k < o_cap) {
          o_idx[k] = gi + idx_offset;
          o_val[k] = xval[gi];
        } else {
          cap_hit = true;
        }
        k++;
      }
    }
    sy = nx;
    c = cn;
  }
  if (cap_hit) atomicOr(&ctl->flags, (uint32_t)CSZI_F_CAPACITY);
}

// Bitmap-driven sparse encoder (MODE 0).  The predictor also wrote one bit
// per symbol, set when the symbol is not R (outliers included), as u32 words
// in symbol order (n % 32 == 0), and k_total_bits computed the stream length
// from the histogram, so the sparse case is known before encoding.  Then R
// is the 1-bit "0" and symbol J starts at bit J + (extra bits of the non-R
// codewords before J).  One warp per 4096-symbol super-chunk, a lane per
// 128 symbols (4 bitmap words): the lane reads only the 16-byte groups of
// symbols under set bits -- about 5% of the groups on smooth fields -- so
// runs of R cost one bitmap bit each.  k_enc_nz_count (extra bits and
// outliers per super-chunk, lane prefixes) -> k_scan_pair over the
// super-chunks -> k_enc_nz_emit.  (Tried: a single-pass decoupled look-back
// over the 32k super-chunks -- 3x slower, the per-tile work is too small to
// hide the walk; shared-memory position lists -- dense super-chunks at the
// field's edges serialise one warp for ~100 us.)
constexpr int NZ_SC = 4096;  // symbols per super-chunk (128 bitmap words)
constexpr int NZ_FW = 4;     // warps per block

__global__ void k_total_bits(const u64 *__restrict__ hist, const uint8_t *__restrict__ lengths,
                             int nbins, cszi_ctl *ctl) {
  __shared__ u64 ws[32];
  u64 v = 0;
  for (int i = threadIdx.x; i < nbins; i += blockDim.x) v += hist[i] * lengths[i];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = (threadIdx.x < (blockDim.x >> 5)) ? ws[threadIdx.x] : 0;
    v = warp_sum(v);
    if (threadIdx.x == 0) ctl->bits = v;
  }
}

// Super-chunk of the calling warp, last first: the densest super-chunks
// (the far edge planes of the field, extrapolated) then start early instead
// of forming the kernel's tail.
DEV u64 nz_tile(u64 nsc) {
  const u64 r = (u64)blockIdx.x * NZ_FW + (threadIdx.x >> 5);
  return r < nsc ? nsc - 1 - r : nsc;
}

// The lane's 4 bitmap words of super-chunk t; returns the lane's set-bit count.
DEV uint32_t nz_words(const uint32_t *__restrict__ nzmap, u64 n, u64 t, int lane,
                      uint32_t wv[4]) {
  const u64 nwords = n / 32, w0 = t * (NZ_SC / 32) + 4 * (u64)lane;
  if (w0 + 4 <= nwords) {
    const uint4 q = __ldcs(reinterpret_cast<const uint4 *>(nzmap + w0));
    wv[0] = q.x, wv[1] = q.y, wv[2] = q.z, wv[3] = q.w;
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) wv[i] = (w0 + i < nwords) ? nzmap[w0 + i] : 0u;
  }
  return __popc(wv[0]) + __popc(wv[1]) + __popc(wv[2]) + __popc(wv[3]);
}

// Calls f(j, symbol) for every set bit j (lane-local, increasing) of the
// lane's 128 symbols at sp.  Per bitmap word the 16-byte groups holding set
// bits are loaded together (one memory latency) and parked in the lane's
// 64-byte shared-memory slot; the rolled loop over set bits reads them back
// with one LDS each and keeps f to a single call site (an unrolled
// per-symbol body overflows the instruction cache).
template <class F>
DEV void nz_visit(const uint16_t *__restrict__ sp, const uint32_t wv[4], uint4 *slot, F &&f) {
  const uint16_t *s16 = reinterpret_cast<const uint16_t *>(slot);
#pragma unroll 1
  for (int i = 0; i < 4; ++i) {
    const uint32_t w = i == 0 ? wv[0] : i == 1 ? wv[1] : i == 2 ? wv[2] : wv[3];  // no local array
    if (!w) continue;
    uint4 q[4];
#pragma unroll
    for (int g = 0; g < 4; ++g)
      if ((w >> (8 * g)) & 0xffu) q[g] = __ldcs(reinterpret_cast<const uint4 *>(sp + 32 * i + 8 * g));
#pragma unroll
    for (int g = 0; g < 4; ++g)
      if ((w >> (8 * g)) & 0xffu) slot[g] = q[g];
#pragma unroll 1
    for (uint32_t m = w; m; m &= m - 1) {
      const uint32_t b = __ffs(m) - 1;
      f(32 * i + b, (uint32_t)s16[b]);
    }
  }
}

// Combining writer of one lane's codewords into the zeroed MSB-first
// stream: bits of the same 32-bit word are merged in a register.  A lane's
// range covers >= 128 bits, so only its first and last words can be shared
// (with the neighbouring lanes): those are ORed in atomically, the words in
// between are plain stores.
struct WordOr {
  uint32_t *out;
  u64 cap_words;
  u64 first;  // the lane's first word
  u64 cur = ~0ull;
  uint32_t acc = 0;
  bool cap_hit = false;
  DEV void put_word(u64 w, uint32_t v) {
    if (w != cur) {
      flush(false);
      cur = w;
    }
    acc |= v;
  }
  DEV void flush(bool last) {
    if (cur != ~0ull && acc) {
      if (cur >= cap_words) cap_hit = true;
      else if (last || cur == first) atomicOr(out + cur, bswap32(acc));
      else out[cur] = bswap32(acc);
    }
    acc = 0;
  }
  DEV void put(u64 pos, uint32_t word, uint32_t len) {
    const u64 w = pos >> 5;
    const uint32_t off = (uint32_t)(pos & 31);
    if (off + len <= 32) {
      put_word(w, word << (32 - off - len));
    } else {
      const uint32_t sh = off + len - 32;
      put_word(w, word >> sh);
      put_word(w + 1, word << (32 - sh));
    }
  }
};

// Balanced path: a super-chunk with K <= NZ_LCAP set bits (all but the few
// dense edge super-chunks) lists them as (j | symbol << 16) in symbol order
// in shared memory -- each lane loads the symbol groups under its own bits
// -- and the lanes then take contiguous rank ranges of the list, so the
// per-symbol work is spread evenly instead of following the bitmap's lanes.
constexpr int NZ_LCAP = 256;

DEV uint32_t nz_pairs(const uint16_t *__restrict__ sp_lane, const uint32_t wv[4], uint32_t pc,
                      int lane, uint4 *slot, uint32_t *lst) {
  const uint32_t incl = warp_incl_scan(pc);
  const uint32_t K = __shfl_sync(CSZI_FULL, incl, 31);
  if (K > (uint32_t)NZ_LCAP) return K;
  uint32_t k = incl - pc;
  nz_visit(sp_lane, wv, slot,
           [&](uint32_t j, uint32_t s) { lst[k++] = (uint32_t)(lane * 128) + j | (s << 16); });
  __syncwarp();
  return K;
}

// per super-chunk: stream bits (R = 1 bit) and outliers -> S.ch_bits /
// S.ch_out; dense super-chunks also the per-lane exclusive prefixes
// (extra bits | outliers << 18) for the emit's per-lane path
__global__ void __launch_bounds__(NZ_FW * 32) k_enc_nz_count(
    const uint16_t *__restrict__ src, const uint32_t *__restrict__ nzmap, u64 n, int R,
    const uint8_t *__restrict__ lengths, const uint32_t *__restrict__ words, EncScratch S,
    u64 nsc, const cszi_ctl *ctl, uint32_t *out, u64 cap_words, uint32_t bit_base) {
  __shared__ uint4 slots[NZ_FW * 32][4];
  __shared__ uint32_t lsts[NZ_FW][NZ_LCAP];
  const int lane = threadIdx.x & 31;
  if (!enc_sparse(lengths, words, R, n, ctl)) return;
  zero_stream(out, cap_words, ctl, bit_base);  // (k_enc_zero's job, one launch less)
  const u64 t = nz_tile(nsc);
  if (t >= nsc) return;
  uint32_t wv[4];
  const uint32_t pc = nz_words(nzmap, n, t, lane, wv);
  const uint16_t *sp_lane = src + t * NZ_SC + 128 * lane;
  uint32_t *lst = lsts[threadIdx.x >> 5];
  const uint32_t K = nz_pairs(sp_lane, wv, pc, lane, slots[threadIdx.x], lst);
  const uint32_t lenR1 = 1u;  // sparse streams: R is the 1-bit "0"
  uint32_t tot;
  if (K <= (uint32_t)NZ_LCAP) {
    uint32_t v = 0;
    for (uint32_t i = lane; i < K; i += 32) {
      const uint32_t s = lst[i] >> 16;
      v += ((uint32_t)__ldg(lengths + (s ? s : (uint32_t)R)) - lenR1) | ((uint32_t)(s == 0) << 18);
    }
    tot = warp_sum(v);
  } else {
    uint32_t ex = 0, o = 0;
    nz_visit(sp_lane, wv, slots[threadIdx.x], [&](uint32_t, uint32_t s) {
      ex += (uint32_t)__ldg(lengths + (s ? s : (uint32_t)R)) - lenR1;  // outlier 0 is coded as R
      o += s == 0;
    });
    // ex < 2^17 (128 symbols x 31 extra bits), o <= 128: one packed scan
    const uint32_t v = ex | (o << 18);
    const uint32_t incl = warp_incl_scan(v);
    S.nz_lane[t * 32 + lane] = incl - v;
    tot = __shfl_sync(CSZI_FULL, incl, 31);
  }
  if (lane == 0) {
    S.ch_bits[t] = (uint32_t)min((u64)NZ_SC, n - t * NZ_SC) + (tot & 0x3ffffu);
    S.ch_out[t] = tot >> 18;
  }
}

__global__ void __launch_bounds__(NZ_FW * 32, 12) k_enc_nz_emit(
    const uint16_t *__restrict__ src, const uint32_t *__restrict__ nzmap, u64 n, int R,
    const uint8_t *__restrict__ lengths, const uint32_t *__restrict__ words,
    uint32_t *__restrict__ out, u64 cap_words, const float *__restrict__ xval, u64 *o_idx,
    float *o_val, u64 o_cap, EncScratch S, u64 nsc, u64 idx_offset, cszi_ctl *ctl,
    uint32_t bit_base) {
  __shared__ uint4 slots[NZ_FW * 32][4];
  __shared__ uint32_t lsts[NZ_FW][NZ_LCAP];
  const int lane = threadIdx.x & 31;
  const u64 t = nz_tile(nsc);
  if (t >= nsc) return;
  uint32_t wv[4];
  const uint32_t pc = nz_words(nzmap, n, t, lane, wv);
  if (!enc_sparse(lengths, words, R, n, ctl)) return;
  if (!__any_sync(CSZI_FULL, pc != 0)) return;
  const u64 sc0 = t * NZ_SC;
  const uint16_t *sp_lane = src + sc0 + 128 * lane;
  uint32_t *lst = lsts[threadIdx.x >> 5];
  const uint32_t K = nz_pairs(sp_lane, wv, pc, lane, slots[threadIdx.x], lst);
  // bit_off counts whole symbols: super-chunk symbol j starts at
  // base + j + (extra bits of the codewords before it)
  const u64 base = S.bit_off[t] + bit_base;
  bool cap_hit = false;
  if (K <= (uint32_t)NZ_LCAP) {
    const uint32_t per = (K + 31) / 32;
    const uint32_t r0 = min(lane * per, K), r1 = min(r0 + per, K);
    uint32_t v = 0;
    for (uint32_t i = r0; i < r1; ++i) {
      const uint32_t s = lst[i] >> 16;
      v += ((uint32_t)__ldg(lengths + (s ? s : (uint32_t)R)) - 1u) | ((uint32_t)(s == 0) << 18);
    }
    const uint32_t pre = warp_incl_scan(v) - v;
    if (r0 < r1) {
      uint32_t extra = pre & 0x3ffffu;
      u64 ko = S.out_off[t] + (pre >> 18);
      WordOr wo{out, cap_words, (base + (lst[r0] & 0xffffu) + extra) >> 5};
      for (uint32_t i = r0; i < r1; ++i) {
        const uint32_t pr = lst[i], j = pr & 0xffffu, s = pr >> 16;
        const uint32_t sI = s ? s : (uint32_t)R;
        const uint32_t len = __ldg(lengths + sI), cw = __ldg(words + sI);
        if (cw) wo.put(base + j + extra, cw, len);
        extra += len - 1;
        if (s == 0) {  // values: gathered by k_assemble
          if (ko < o_cap) o_idx[ko] = sc0 + j + idx_offset;
          else cap_hit = true;
          ko++;
        }
      }
      wo.flush(true);
      cap_hit |= wo.cap_hit;
    }
  } else if (pc) {
    const uint32_t lp = S.nz_lane[t * 32 + lane];
    const u64 g0 = sc0 + 128 * (u64)lane;
    const u64 pos0 = base + 128 * (u64)lane + (lp & 0x3ffffu);
    u64 ko = S.out_off[t] + (lp >> 18);
    uint32_t extra = 0;
    WordOr wo{out, cap_words, pos0 >> 5};
    nz_visit(sp_lane, wv, slots[threadIdx.x], [&](uint32_t j, uint32_t s) {
      const uint32_t sI = s ? s : (uint32_t)R;
      const uint32_t len = __ldg(lengths + sI), cw = __ldg(words + sI);
      if (cw) wo.put(pos0 + j + extra, cw, len);
      extra += len - 1;
      if (s == 0) {
        if (ko < o_cap) o_idx[ko] = g0 + j + idx_offset;
        else cap_hit = true;
        ko++;
      }
    });
    wo.flush(true);
    cap_hit |= wo.cap_hit;
  }
  if (cap_hit) atomicOr(&ctl->flags, (uint32_t)CSZI_F_CAPACITY);
}

template <int MODE>
__global__ void __launch_bounds__(ENC_NT, 3) k_enc_pack(const void *__restrict__ src, u64 n, int R,
                                                       const uint8_t *__restrict__ lengths,
                                                       const uint32_t *__restrict__ words,
                                                       uint32_t *__restrict__ out, u64 cap_words,
                                                       const float *__restrict__ xval, u64 *o_idx,
                                                       float *o_val, u64 o_cap, EncScratch S,
                                                       u64 nch, u64 idx_offset, cszi_ctl *ctl, uint32_t bit_base) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  if (MODE == 0 && enc_sparse(lengths, words, R, n, ctl)) return;  // k_enc_sparse's case
  const int nbins = 2 * R;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint2 *lut = reinterpret_cast<uint2 *>(sm_raw);
  uint32_t *stage = reinterpret_cast<uint32_t *>(lut + nbins + 2) + warp * ENC_SW;
  enc_load_lut<MODE>(lut, lengths, words, R);
  for (int i = lane; i < ENC_SW; i += 32) stage[i] = 0u;
  // R coded as the 1-bit "0" (the usual case): pairs of R take the fast path
  const uint32_t zz2 = (MODE == 0 && lengths[R] == 1 && words[R] == 0)
                           ? ((uint32_t)R | ((uint32_t)R << 16))
                           : 0xffffffffu;
  __syncthreads();
  bool unknown = false;  // reported by k_enc_count
  bool cap_hit = false;
  const u64 stride = (u64)gridDim.x * ENC_NW;
  u64 c = (u64)blockIdx.x * ENC_NW + warp;
  EncSyms<MODE> sy;
  if (c < nch) sy.load(src, n, R, nbins, c * ENC_CH + (u64)lane * ENC_SPT, unknown);
  while (c < nch) {
    const u64 cn = c + stride;
    EncSyms<MODE> nx;
    if (cn < nch) nx.load(src, n, R, nbins, cn * ENC_CH + (u64)lane * ENC_SPT, unknown);
    const u64 tb = S.bit_off[c] + bit_base;
    const u64 ob = (MODE == 0) ? S.out_off[c] : 0;
    uint32_t outmask;
    const uint32_t nbits = enc_bits<MODE>(sy, lut, nbins, unknown, outmask, zz2);
    const uint32_t incl = warp_incl_scan(nbits);
    const uint32_t bexcl = incl - nbits;
    const uint32_t tot_bits = __shfl_sync(CSZI_FULL, incl, 31);
    {  // pack at chunk-relative bit offsets (staging words start zeroed, so
       // all-zero words need no store)
      uint32_t w = bexcl >> 5;
      uint32_t nb = bexcl & 31;
      u64 acc = 0;
#pragma unroll
      for (int j = 0; j < ENC_SPT; j += 2) {
        if (MODE == 0 && sy.w[j >> 1] == zz2) {
          acc <<= 2;
          nb += 2;
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint2 e = lut[sy.get(j + h)];
            acc = (acc << e.y) | (u64)e.x;
            nb += e.y;
            if (nb >= 32) {
              nb -= 32;
              const uint32_t v = (uint32_t)(acc >> nb);
              if (v) atomicOr(&stage[w], v);
              w++;
            }
          }
          continue;
        }
        if (nb >= 32) {
          nb -= 32;
          const uint32_t v = (uint32_t)(acc >> nb);
          if (v) atomicOr(&stage[w], v);
          w++;
        }
      }
      if (nb > 0) {
        const uint32_t v = (uint32_t)(acc << (32 - nb));
        if (v) atomicOr(&stage[w], v);
      }
    }
    if (MODE == 0 && __any_sync(CSZI_FULL, outmask != 0)) {
      const uint32_t no = (uint32_t)__popc(outmask);
      u64 k = ob + (warp_incl_scan(no) - no);
      const u64 base = c * ENC_CH + (u64)lane * ENC_SPT;
      for (uint32_t m = outmask; m; m &= m - 1) {
        const u64 gi = base + (__ffs(m) - 1);
        if (k < o_cap) {
          o_idx[k] = gi + idx_offset;
          o_val[k] = xval[gi];
        } else {
          cap_hit = true;
        }
        k++;
      }
    }
    __syncwarp();
    // write out: global word gw0 + i = stage bits shifted right by off0
    const uint32_t off0 = (uint32_t)(tb & 31);
    const u64 gw0 = tb >> 5;
    const u64 end_bits = tb + tot_bits;
    const uint32_t nw = tot_bits ? (uint32_t)(((end_bits - 1) >> 5) - gw0 + 1) : 0;
    const bool head_shared = off0 != 0 && c > 0;
    const bool tail_shared = (end_bits & 31) != 0 && c + 1 < nch;
    for (uint32_t i = lane; i < nw; i += 32) {
      const uint32_t cur = stage[i];
      const uint32_t prv = i ? stage[i - 1] : 0u;
      const uint32_t val = off0 ? ((cur >> off0) | (prv << (32 - off0))) : cur;
      const u64 gw = gw0 + i;
      if (gw >= cap_words) {
        cap_hit = true;
        continue;
      }
      if ((i == 0 && head_shared) || (i == nw - 1 && tail_shared))
        atomicOr(out + gw, bswap32(val));
      else
        out[gw] = bswap32(val);
    }
    __syncwarp();
    for (uint32_t i = lane; i <= nw; i += 32) stage[i] = 0u;
    __syncwarp();
    sy = nx;
    c = cn;
  }
  if (cap_hit) atomicOr(&ctl->flags, (uint32_t)CSZI_F_CAPACITY);
}

// ---------------------------------------------------------------------------
// decode: self-synchronising chunked decode of one stream
// ---------------------------------------------------------------------------
constexpr u64 DEC_C = 256;  // bits per chunk (8 words)

struct DecSmem {
  const uint32_t *lut;  // global, read through L1 (16 KB, hot)
  u64 first_code[33];
  uint32_t first_index[33];
  uint32_t counts[33];
  int zrun;       // 1: exactly one length-1 codeword; canonically it is "0"
  uint32_t zsym;  // its symbol
};

DEV void load_dec_smem(DecSmem &T, const DecTables *G, const uint16_t *sorted) {
  if (threadIdx.x == 0) T.lut = G->lut;
  for (int i = threadIdx.x; i < 33; i += blockDim.x) {
    T.first_code[i] = G->first_code[i];
    T.first_index[i] = G->first_index[i];
    T.counts[i] = G->counts[i];
  }
  if (threadIdx.x == 0) {
    // canonical order (huffman.py:128-160): the first codeword is all
    // zeros, so a single length-1 symbol owns "0" and a run of z zero bits
    // is z copies of it -- counted / emitted per run instead of per bit
    T.zrun = (G->counts[1] == 1 && G->first_code[1] == 0) ? 1 : 0;
    T.zsym = T.zrun ? sorted[G->first_index[1]] : 0u;
  }
  __syncthreads();
}

struct Stream {
  const uint32_t *w;  // aligned-down word pointer
  u64 nwords;
  u64 b0;   // bit offset of the stream start inside w
  u64 nb;   // stream length in bits
};

struct BitReader {
  u64 buf;
  u64 cw;
  DEV uint32_t word(const Stream &s, u64 i) const {
    return i < s.nwords ? bswap32(__ldg(s.w + i)) : 0u;
  }
  DEV void init() { cw = ~0ull - 1; }  // never equal to wi or wi - 1
  // next 32 bits at stream bit position pos (MSB-first)
  DEV uint32_t peek(const Stream &s, u64 pos) {
    const u64 a = pos + s.b0;
    const u64 wi = a >> 5;
    if (wi != cw) {
      if (wi == cw + 1) buf = (buf << 32) | word(s, wi + 1);
      else buf = ((u64)word(s, wi) << 32) | word(s, wi + 1);
      cw = wi;
    }
    return (uint32_t)((buf << (a & 31)) >> 32);
  }
};

// Decode the codeword starting at stream position pos.  Returns the symbol
// and sets len (0 if no codeword of length <= 32 matches; the caller also
// treats pos + len > nb as exhaustion) — _kernels.py:74-91.
DEV uint32_t decode_at(const DecSmem &T, const uint16_t *sorted, uint32_t win, uint32_t &len) {
  const uint32_t e = __ldg(T.lut + (win >> 20));
  if (e >> 16) {
    len = e >> 16;
    return e & 0xffffu;
  }
  for (uint32_t l = 13; l <= 32; ++l) {
    const uint32_t c = T.counts[l];
    if (!c) continue;
    const u64 cur = (u64)(win >> (32 - l));
    const u64 fc = T.first_code[l];
    if (cur >= fc && cur - fc < c) {
      len = l;
      return sorted[T.first_index[l] + (uint32_t)(cur - fc)];
    }
  }
  len = 0;
  return 0;
}

// Stream words of a block's chunks staged in shared memory: thread j of the
// block decodes chunk j0 + j; a chunk walk never reads more than one word
// past the block's last chunk (a codeword is at most 32 bits).
constexpr int DEC_NT = 128;
constexpr int DEC_W = (int)(DEC_C / 32);           // words per chunk
constexpr int DEC_SW = DEC_NT * DEC_W + 4;         // staged words per block

struct SmemStream {
  const uint32_t *w;  // staged words; w[0] = stream word wbase
  u64 wbase;
  u64 b0, nb;
};

DEV void stage_words(uint32_t *sw, const Stream &s, u64 j0, SmemStream &ss) {
  const u64 wbase = (j0 * DEC_C + s.b0) >> 5;
  for (int i = threadIdx.x; i < DEC_SW; i += blockDim.x) {
    const u64 wi = wbase + i;
    sw[i] = wi < s.nwords ? bswap32(__ldg(s.w + wi)) : 0u;
  }
  ss.w = sw;
  ss.wbase = wbase;
  ss.b0 = s.b0;
  ss.nb = s.nb;
}

struct SmemReader {
  u64 buf;
  int cw;
  DEV void init() { cw = -2; }
  DEV uint32_t peek(const SmemStream &s, u64 pos) {
    const u64 a = pos + s.b0;
    const int wi = (int)((a >> 5) - s.wbase);
    if (wi != cw) {
      if (wi == cw + 1) buf = (buf << 32) | s.w[wi + 1];
      else buf = ((u64)s.w[wi] << 32) | s.w[wi + 1];
      cw = wi;
    }
    return (uint32_t)((buf << (a & 31)) >> 32);
  }
};

// canonical (huffman.py:128-160): a single length-1 codeword is "0"
DEV bool zrun_tables(const DecTables *G) { return G->counts[1] == 1 && G->first_code[1] == 0; }

// Phase 1: speculative decode of chunk j from its first bit.
// (chunks jbase + blockIdx * DEC_NT + threadIdx < M: a range of the stream)
__global__ void __launch_bounds__(DEC_NT) k_dec_spec(Stream s, const DecTables *G,
                                                    const uint16_t *sorted, u64 M, u64 *spec_exit,
                                                    uint32_t *spec_cnt, uint8_t *spec_dead,
                                                    u64 jbase, u64 *fd_init) {
  __shared__ DecSmem T;
  __shared__ uint32_t sw[DEC_SW];
  // the write phase's first-dead-chunk minimum starts at ~0 (no set kernel)
  if (fd_init && blockIdx.x == 0 && threadIdx.x == 0) *fd_init = ~0ull;
  const u64 j0 = jbase + (u64)blockIdx.x * DEC_NT;
  SmemStream ss;
  stage_words(sw, s, j0, ss);
  load_dec_smem(T, G, sorted);  // ends with __syncthreads()
  const u64 j = j0 + threadIdx.x;
  if (j >= M) return;
  SmemReader br;
  br.init();
  // 32-bit chunk-relative position (a chunk ends at most 32 bits past its window)
  const u64 pos0 = j * DEC_C;
  const uint32_t pend = (uint32_t)(min((j + 1) * DEC_C, s.nb) - pos0);
  const uint32_t plim = (uint32_t)min(s.nb - pos0, (u64)0xffffffffu);
  uint32_t p = 0;
  uint32_t cnt = 0;
  uint8_t dead = 0;
  const bool zr = T.zrun != 0;
  while (p < pend) {
    const uint32_t w = br.peek(ss, pos0 + p);
    if (zr && !(w >> 31)) {  // run of the "0" codeword
      const uint32_t adv = min((uint32_t)__clz(w), pend - p);
      p += adv;
      cnt += adv;
      continue;
    }
    uint32_t len;
    decode_at(T, sorted, w, len);
    if (len == 0 || p + len > plim) {
      dead = 1;
      break;
    }
    p += len;
    cnt++;
    if (zr && len < 32) {  // the "0" codewords after it in the same window
      const uint32_t adv = min(min((uint32_t)__clz(w << len), 32u - len), pend - p);
      p += adv;
      cnt += adv;
    }
  }
  spec_exit[j] = pos0 + p;
  spec_cnt[j] = cnt;
  spec_dead[j] = dead;
}

// Phase 2 (iteration `it`): chunk j decoded from its current entry estimate,
// walked in lockstep with its speculative decode until both chains meet.
// it == 0: entry = 0 (j == 0) or spec_exit[j-1]; it > 0: entry = X_prev[j-1]
// for chunks whose entry changed in the previous iteration.
// (chunks [jbase, M): a range of the stream whose first chunk enters at
// *entry_dev -- 0 for the stream start, a neighbour's true exit, or the
// speculative exit of chunk jbase - 1)
__global__ void __launch_bounds__(256) k_dec_sync(Stream s, const DecTables *G,
                                                 const uint16_t *sorted, u64 M, int it,
                                                 const u64 *spec_exit, const uint32_t *spec_cnt,
                                                 const uint8_t *spec_dead, const u64 *X_prev,
                                                 const uint8_t *chg_prev, u64 *X, uint32_t *K,
                                                 uint8_t *D, uint8_t *chg, uint32_t *nchg,
                                                 u64 jbase, u64 *entry_dev, u64 e0) {
  __shared__ DecSmem T;
  // nothing moved in iteration 0 (the common case): every later iteration
  // is a no-op and X already holds the result (the last iteration, `iters`
  // odd, writes X as iteration 0 did)
  if (it > 0 && *(nchg - it) == 0) return;
  const u64 j = jbase + blockIdx.x * (u64)blockDim.x + threadIdx.x;
  // iterations > 0: only chunks whose predecessor moved re-walk; blocks
  // without one skip the table load (most of them once the chains meet)
  bool need = j < M;
  if (need && it > 0 && (j == jbase || !chg_prev[j - 1])) {
    X[j] = X_prev[j];
    chg[j] = 0;
    need = false;
  }
  if (!__syncthreads_or(need)) return;
  load_dec_smem(T, G, sorted);
  if (!need) return;
  // the range's entry (iteration 0 only: later ones copy chunk jbase): e0,
  // or ~0 for the speculative exit of chunk jbase - 1; recorded in *entry_dev
  u64 e;
  if (j == jbase) {
    e = (e0 != ~0ull) ? e0 : spec_exit[j - 1];
    *entry_dev = e;
  } else {
    e = (it == 0) ? spec_exit[j - 1] : X_prev[j - 1];
  }
  const u64 end = min((j + 1) * DEC_C, s.nb);
  BitReader ba, bb;
  ba.init();
  bb.init();
  u64 a = e, b = j * DEC_C;
  uint32_t ca = 0, cb = 0;
  bool b_alive = true;
  u64 xo;
  uint32_t ko;
  uint8_t dd = 0;
  for (;;) {
    if (b_alive && a == b) {  // synchronised with the speculative chain
      xo = spec_exit[j];
      ko = ca + (spec_cnt[j] - cb);
      dd = spec_dead[j];
      break;
    }
    if (a >= end) {
      xo = a;
      ko = ca;
      break;
    }
    if (!b_alive || a < b) {
      const uint32_t w = ba.peek(s, a);
      if (T.zrun && !(w >> 31)) {  // zero run: every bit is a boundary
        u64 adv = min((u64)__clz(w), end - a);
        if (b_alive && b > a) adv = min(adv, b - a);
        a += adv;
        ca += (uint32_t)adv;
        continue;
      }
      uint32_t len;
      decode_at(T, sorted, w, len);
      if (len == 0 || a + len > s.nb) {
        xo = a;
        ko = ca;
        dd = 1;
        break;
      }
      a += len;
      ca++;
    } else {
      if (b >= end) {
        b_alive = false;
        continue;
      }
      const uint32_t w = bb.peek(s, b);
      if (T.zrun && !(w >> 31)) {
        const u64 adv = min(min((u64)__clz(w), end - b), a - b > 0 ? a - b : (u64)1);
        b += adv;
        cb += (uint32_t)adv;
        continue;
      }
      uint32_t len;
      decode_at(T, sorted, w, len);
      if (len == 0 || b + len > s.nb) {
        b_alive = false;
        continue;
      }
      b += len;
      cb++;
    }
  }
  X[j] = xo;
  K[j] = ko;
  D[j] = dd;
  // the next chunk's entry estimate was spec_exit[j] (it 0) or X_prev[j]
  const u64 prev_est = (it == 0) ? spec_exit[j] : X_prev[j];
  const uint8_t c = (xo != prev_est) ? 1 : 0;
  chg[j] = c;
  if (c && j + 1 < M) atomicAdd(nchg, 1u);  // (M: the range end)
}

// Phase 3 (after the generic exclusive scan of K into off): truncation
// check.  Decodable symbols = offset + count of the first chunk whose chain
// dies (invalid code / exhausted stream), or the total when none dies.
__global__ void k_dec_first_dead(u64 M, const uint8_t *D, u64 *first_dead,
                                 const uint32_t *nchg_last, u64 *nchg_out) {
  const u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  // chains still moving after the last sync iteration -> ctl (no copy node)
  if (nchg_out && j == 0) *nchg_out = *nchg_last;
  if (j < M && D[j]) atomicMin(first_dead, j);
}
// decoded-symbol count / truncation check, run by thread 0 of block 0 of
// whichever write kernel proceeds (one launch less)
struct DecCheck {
  const u64 *first_dead;
  const u64 *total;
  cszi_ctl *ctl;
};
DEV void dec_check(const u64 *off, const uint32_t *K, u64 n, const DecCheck &C) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  const u64 fd = *C.first_dead;
  const u64 avail = (fd != ~0ull) ? off[fd] + K[fd] : *C.total;
  C.ctl->decoded_symbols = avail;
  if (avail < n) atomicOr(&C.ctl->flags, (uint32_t)CSZI_F_TRUNCATED);
}

// Fallback for streams whose chunks do not self-synchronise (e.g. codebooks
// with all lengths equal): exact per-chunk transfer tables over every entry
// offset 0 <= d < lmax, composed by the chain resolver.
__global__ void __launch_bounds__(256) k_dec_table(Stream s, const DecTables *G,
                                                  const uint16_t *sorted, u64 M, int lmax,
                                                  uint8_t *tab, uint32_t *ktab, uint8_t *dtab) {
  __shared__ DecSmem T;
  load_dec_smem(T, G, sorted);
  const u64 w = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  if (w >= M * (u64)lmax) return;
  const u64 j = w / lmax;
  const int d = (int)(w - j * lmax);
  const u64 end = min((j + 1) * DEC_C, s.nb);
  u64 pos = j * DEC_C + d;
  uint32_t cnt = 0;
  uint8_t dead = 0;
  BitReader br;
  br.init();
  while (pos < end) {
    uint32_t len;
    decode_at(T, sorted, br.peek(s, pos), len);
    if (len == 0 || pos + len > s.nb) {
      dead = 1;
      break;
    }
    pos += len;
    cnt++;
  }
  const u64 ex = (!dead && pos >= (j + 1) * DEC_C) ? pos - (j + 1) * DEC_C : 0;
  tab[w] = (uint8_t)min(ex, (u64)(lmax - 1));
  ktab[w] = cnt;
  dtab[w] = dead;
}
__global__ void k_dec_from_tab(u64 M, int lmax, const uint8_t *E, const uint32_t *ktab,
                               const uint8_t *dtab, u64 *X, uint32_t *K, uint8_t *D) {
  const u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  if (j >= M) return;
  const int e = E[j];
  K[j] = ktab[j * lmax + e];
  D[j] = dtab[j * lmax + e];
  X[j] = (j + 1 < M) ? (j + 1) * DEC_C + E[j + 1] : 0;
}

// Phase 4: final decode of each chunk from its true entry.  Symbols are
// produced in rounds of DEC_K per thread into a per-warp shared buffer and
// flushed cooperatively (lane l writes symbol l of one thread's run), so
// every store instruction of a warp covers one contiguous 64-128 B span.
constexpr int DEC_K = 32;

// Both write kernels store symbol k at out[k - w0] for k in [w0, w1) only
// (a z-slab's window of the stream; [0, n) for a whole grid); chunks
// outside the window are not decoded.
template <typename OutT>
__global__ void __launch_bounds__(DEC_NT) k_dec_write(Stream s, const DecTables *G,
                                                     const uint16_t *sorted, u64 M, const u64 *X,
                                                     const u64 *off, const uint32_t *cnts,
                                                     u64 n, int R, OutT *__restrict__ out, u64 w0,
                                                     u64 w1, DecCheck C) {
  if (zrun_tables(G)) return;  // zero-run streams: k_dec_write_zr
  dec_check(off, cnts, n, C);
  __shared__ DecSmem T;
  __shared__ uint32_t sw[DEC_SW];
  constexpr int K = (sizeof(OutT) == 2) ? DEC_K : DEC_K / 2;
  __shared__ OutT ob[DEC_NT / 32][32][K + 1];
  const u64 j0 = (u64)blockIdx.x * DEC_NT;
  SmemStream ss;
  stage_words(sw, s, j0, ss);
  load_dec_smem(T, G, sorted);
  const u64 j = j0 + threadIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  u64 k = (j < M) ? off[j] : n;
  u64 pos = (j < M) ? ((j == 0) ? 0 : X[j - 1]) : 0;
  const u64 end = (j < M) ? min((j + 1) * DEC_C, s.nb) : 0;
  bool active = j < M && k < n && k < w1 && k + cnts[j] > w0;
  SmemReader br;
  br.init();
  if (T.zrun) return;  // zero-run streams: k_dec_write_zr
  while (__any_sync(CSZI_FULL, active)) {
    int cnt = 0;
    if (active) {
      while (cnt < K && pos < end && k + cnt < n) {
        const uint32_t w = br.peek(ss, pos);
        if (T.zrun && !(w >> 31)) {  // run of the "0" codeword
          u64 adv = min((u64)__clz(w), end - pos);
          adv = min(adv, (u64)(K - cnt));
          adv = min(adv, n - k - cnt);
          const OutT zv = (sizeof(OutT) == 4) ? (OutT)((int32_t)T.zsym - R) : (OutT)T.zsym;
          for (int i = 0; i < (int)adv; ++i) ob[warp][lane][cnt + i] = zv;
          cnt += (int)adv;
          pos += adv;
          continue;
        }
        uint32_t len;
        const uint32_t sym = decode_at(T, sorted, w, len);
        if (len == 0 || pos + len > s.nb) {
          pos = end;  // dead chain: truncation is reported by dec_check
          break;
        }
        pos += len;
        ob[warp][lane][cnt++] = (sizeof(OutT) == 4) ? (OutT)((int32_t)sym - R) : (OutT)sym;
      }
    }
    __syncwarp();
    for (int i = 0; i < 32; ++i) {
      const int ci = __shfl_sync(CSZI_FULL, cnt, i);
      const u64 ki = __shfl_sync(CSZI_FULL, k, i);
      if (lane < ci && ki + lane >= w0 && ki + lane < w1) out[ki + lane - w0] = ob[warp][i][lane];
    }
    __syncwarp();
    k += cnt;
    active = active && cnt == K && pos < end && k < n && k < w1;
  }
}

// Zero-run streams: the warp fills its chunks' output range with the run
// symbol (coalesced), then each lane stores only its chunk's other symbols.
// Separate from k_dec_write so that neither the staging buffer nor the
// registers of the dense path limit its occupancy.
template <typename OutT>
__global__ void __launch_bounds__(DEC_NT) k_dec_write_zr(Stream s, const DecTables *G,
                                                        const uint16_t *sorted, u64 M,
                                                        const u64 *X, const u64 *off,
                                                        const uint32_t *cnts, u64 n, int R,
                                                        OutT *__restrict__ out, u64 w0, u64 w1, DecCheck C) {
  if (!zrun_tables(G)) return;  // k_dec_write handles other streams
  dec_check(off, cnts, n, C);
  __shared__ DecSmem T;
  __shared__ uint32_t sw[DEC_SW];
  const u64 j0 = (u64)blockIdx.x * DEC_NT;
  SmemStream ss;
  stage_words(sw, s, j0, ss);
  load_dec_smem(T, G, sorted);
  const u64 j = j0 + threadIdx.x;
  const int lane = threadIdx.x & 31;
  u64 k = (j < M) ? off[j] : n;
  u64 pos = (j < M) ? ((j == 0) ? 0 : X[j - 1]) : 0;
  const u64 end = (j < M) ? min((j + 1) * DEC_C, s.nb) : 0;
  const bool active = j < M && k < n && k < w1 && k + cnts[j] > w0;
  SmemReader br;
  br.init();
  {
    // Sparse path: the warp's 32 chunks own the contiguous output range
    // [k(lane 0), k1(lane 31)); the warp fills it with the run symbol in
    // coalesced 16-byte stores, then each lane stores only the other
    // symbols of its chunk (after __syncwarp, so they win).  Runs cost O(1).
    const u64 k1 = active ? min(min(k + cnts[j], n), w1) : k;
    const OutT zv = (sizeof(OutT) == 4) ? (OutT)((int32_t)T.zsym - R) : (OutT)T.zsym;
    constexpr int PER = 16 / sizeof(OutT);
    {
      u64 wa = active ? max(k, w0) : ~0ull, wb = active ? k1 : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        wa = min(wa, __shfl_xor_sync(CSZI_FULL, wa, o));
        wb = max(wb, __shfl_xor_sync(CSZI_FULL, wb, o));
      }
      if (wa < wb) {  // window coordinates (out is 16-byte aligned at w0 when PER | w0)
        uint4 zz;
        OutT tmp[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) tmp[i] = zv;
        memcpy(&zz, tmp, 16);
        const u64 ra = wa - w0, rb = wb - w0;
        const bool vec = (w0 % PER) == 0;
        const u64 va = vec ? (ra + PER - 1) / PER : rb, vb = vec ? rb / PER : rb;
        if (vec && va <= vb) {
          // 32-bit loop counters relative to the warp's range (< 2^32 symbols)
          const int lead = (int)(va * PER - ra), nv = (int)(vb - va), tail = (int)(rb - vb * PER);
          if (lane < lead) out[ra + lane] = zv;
          uint4 *o4 = reinterpret_cast<uint4 *>(out) + va;
          int v = lane;
#pragma unroll 1
          for (; v + 96 < nv; v += 128) {
            __stcs(o4 + v, zz);
            __stcs(o4 + v + 32, zz);
            __stcs(o4 + v + 64, zz);
            __stcs(o4 + v + 96, zz);
          }
          for (; v < nv; v += 32) __stcs(o4 + v, zz);
          if (lane < tail) out[vb * PER + lane] = zv;
        } else {
          for (u64 f = ra + lane; f < rb; f += 32) out[f] = zv;
        }
      }
    }
    __syncwarp();
    if (!active) return;
    // 32-bit counters relative to the chunk (a chunk holds at most DEC_C
    // symbols and ends at most 32 bits past its DEC_C-bit window)
    const u64 pos0 = pos, kb = k;
    const uint32_t pend = (uint32_t)(end - pos0), kend = (uint32_t)(k1 - kb);
    const uint32_t plim = (uint32_t)min(s.nb - pos0, (u64)0xffffffffu);
    uint32_t p = 0, kk = 0;
    OutT *o = out + (kb - w0);  // may point below out; only written at kb + kk >= w0
    const uint32_t kskip = kb >= w0 ? 0u : (uint32_t)(w0 - kb);
    while (p < pend && kk < kend) {
      const uint32_t w = br.peek(ss, pos0 + p);
      if (!(w >> 31)) {
        const uint32_t adv = min(min((uint32_t)__clz(w), pend - p), kend - kk);
        p += adv;
        kk += adv;
        continue;
      }
      uint32_t len;
      const uint32_t sym = decode_at(T, sorted, w, len);
      if (len == 0 || p + len > plim) break;  // dead chain: reported by dec_check
      p += len;
      if (kk >= kskip) o[kk] = (sizeof(OutT) == 4) ? (OutT)((int32_t)sym - R) : (OutT)sym;
      ++kk;
      if (len < 32) {  // the "0" codewords after it in the same window (run fill wrote them)
        const uint32_t adv =
            min(min(min((uint32_t)__clz(w << len), 32u - len), pend - p), kend - kk);
        p += adv;
        kk += adv;
      }
    }
    return;
  }
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
int launch_hist_i32(const int32_t *codes, u64 n, int R, u64 *hist, cszi_ctl *ctl,
                    cudaStream_t st) {
  cudaMemsetAsync(hist, 0, sizeof(u64) * 2 * (size_t)R, st);
  const int nb = 2 * R;
  const size_t smem = nb <= 8192 ? sizeof(uint32_t) * nb : 0;
  u64 blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  k_hist_i32<<<(unsigned)blocks, 256, smem, st>>>(codes, n, R, hist, ctl);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

int launch_codebook(const u64 *hist, int nbins, uint8_t *lengths, uint32_t *words,
                    cszi_ctl *ctl, cudaStream_t st, bool set_bits) {
  if (nbins > 16384 || nbins < 1) return CSZI_E_UNSUPPORTED;
  int npow2 = 1;
  while (npow2 < nbins) npow2 <<= 1;
  // keys[npow2] + parent[2*nbins] + len[nbins] + internal keys / depths
  const size_t smem = sizeof(u64) * (npow2 + nbins) + sizeof(int32_t) * 3 * nbins + nbins + 16;
  ensure_smem((const void *)k_codebook, smem);
  k_codebook<<<1, CB_NT, smem, st>>>(hist, nbins, lengths, words, ctl, set_bits ? 1 : 0);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

size_t dec_tables_bytes(int nbins) { return sizeof(DecTables) + sizeof(uint16_t) * nbins + 16; }

int launch_canonical(const uint8_t *lengths, int nbins, uint32_t *words, void *dec_tables,
                     cszi_ctl *ctl, cudaStream_t st,
                     u64 expect_raw_len) {
  if (nbins > 65536 || nbins < 1) return CSZI_E_UNSUPPORTED;
  const size_t smem = nbins + 16;
  ensure_smem((const void *)k_canonical, smem);
  k_canonical<<<1, CB_NT, smem, st>>>(lengths, nbins, words,
                                      reinterpret_cast<DecTables *>(dec_tables), ctl, expect_raw_len);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

// dst |= src bits placed at bit offset dst_bit (both MSB-first byte streams)
__global__ void k_concat_bits(uint8_t *dst, u64 dst_bit, const uint8_t *src, u64 nbits) {
  const u64 b0 = dst_bit >> 3;
  const int sh = (int)(dst_bit & 7);
  const u64 nbytes_out = ((dst_bit + nbits + 7) >> 3) - b0;
  const u64 nsrc = (nbits + 7) >> 3;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < nbytes_out;
       i += (u64)gridDim.x * blockDim.x) {
    uint32_t v = 0;
    if (i < nsrc) v |= (uint32_t)src[i] >> sh;
    if (sh && i >= 1 && i - 1 < nsrc) v |= ((uint32_t)src[i - 1] << (8 - sh)) & 0xffu;
    if (v) dst[b0 + i] |= (uint8_t)v;
  }
}

__global__ void k_pack_outliers(const u64 *idx, const float *val, u64 k, uint8_t *out) {
  const u64 tid = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  if (tid < 8) out[tid] = (uint8_t)(k >> (8 * tid));
  for (u64 r = tid; r < k; r += (u64)gridDim.x * blockDim.x) {
    uint8_t *q = out + 8 + 12 * r;
    const u64 ix = idx[r];
    const uint32_t vb = __float_as_uint(val[r]);
    for (int b = 0; b < 8; ++b) q[b] = (uint8_t)(ix >> (8 * b));
    for (int b = 0; b < 4; ++b) q[8 + b] = (uint8_t)(vb >> (8 * b));
  }
}

int launch_concat_bits(uint8_t *dst, u64 dst_bit, const uint8_t *src, u64 nbits,
                       cudaStream_t st) {
  if (nbits == 0) return CSZI_OK;
  const u64 nb = (nbits + 8 + 7) / 8;
  u64 blocks = (nb + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  k_concat_bits<<<(unsigned)blocks, 256, 0, st>>>(dst, dst_bit, src, nbits);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

int launch_pack_outliers(const u64 *idx, const float *val, u64 k, uint8_t *out,
                         cudaStream_t st) {
  u64 blocks = (k + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  if (blocks < 1) blocks = 1;
  k_pack_outliers<<<(unsigned)blocks, 256, 0, st>>>(idx, val, k, out);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

u64 enc_scratch_bytes(u64 n) {
  const u64 nc = (n + ENC_CH - 1) / ENC_CH + 2;
  const u64 nt = (nc + PS_TILE - 1) / PS_TILE + 2;
  const u64 nsc = n / NZ_SC + 2;
  return nc * (4 + 4 + 8 + 8 + 2 * 32) + nt * 16 + 64 + nsc * 4 * 32;
}

// mode 0: uint16 symbols with outlier sentinel; mode 1: int32 codes
int launch_encode(int mode, const void *src, u64 n, int R, const uint8_t *lengths,
                  const uint32_t *words, uint32_t *out, u64 cap_bytes, const float *xval,
                  u64 *o_idx, float *o_val, u64 o_cap, void *scratch, cszi_ctl *ctl,
                  cudaStream_t st, u64 idx_offset, uint32_t bit_base,
                  const uint32_t *nzmap, const u64 *hist, bool bits_known) {
  if (n == 0) return CSZI_OK;
  if (mode != 0 || (n & 31) || (reinterpret_cast<uintptr_t>(src) & 15)) nzmap = nullptr;
  const u64 nch = (n + ENC_CH - 1) / ENC_CH;
  const u64 nc = nch + 2;
  const u64 npt = (nch + PS_TILE - 1) / PS_TILE;
  const u64 nt = npt + 2;
  unsigned char *p = reinterpret_cast<unsigned char *>(scratch);
  EncScratch S;
  S.st_bits = reinterpret_cast<u64 *>(p);  // zeroed: st_bits, st_out, ticket
  S.st_out = S.st_bits + nt;
  S.ticket = reinterpret_cast<uint32_t *>(S.st_out + nt);
  S.bit_off = reinterpret_cast<u64 *>(S.ticket + 4);
  S.out_off = S.bit_off + nc;
  S.ch_bits = reinterpret_cast<uint32_t *>(S.out_off + nc);
  S.ch_out = S.ch_bits + nc;
  S.lane_pre = reinterpret_cast<uint16_t *>(S.ch_out + nc);
  S.nz_lane = reinterpret_cast<uint32_t *>(S.lane_pre + 32 * nc);
  launch_zero16(p, (u64)(nt * 16 + 16), st);  // (a kernel: no memset node in the graph)
  const int nbins = 2 * R;
  int sms = sm_count(), per_sm = 1;
  const size_t smem_c = sizeof(uint32_t) * (nbins + 2) + 16;
  const size_t smem_p = sizeof(uint2) * (nbins + 2) + 16 + sizeof(uint32_t) * ENC_SW * ENC_NW;
  auto kc = mode == 0 ? k_enc_count<0> : k_enc_count<1>;
  auto kp = mode == 0 ? k_enc_pack<0> : k_enc_pack<1>;
  ensure_smem((const void *)kc, smem_c);
  ensure_smem((const void *)kp, smem_p);
  const u64 wblocks = (nch + ENC_NW - 1) / ENC_NW;
  per_sm = occupancy((const void *)kc, ENC_NT, smem_c);
  u64 blocks = (u64)sms * (per_sm < 1 ? 1 : per_sm);
  if (blocks > wblocks) blocks = wblocks;
  // bitmap path: needs the bitmap and the histogram (stream length known
  // up front); count / scan / pack over 1024-symbol chunks then run only
  // for a dense stream, the k_enc_nz_* kernels only for a sparse one
  const bool nzp = nzmap && (hist || bits_known);
  if (nzp && !bits_known) {
    k_total_bits<<<1, 1024, 0, st>>>(hist, lengths, nbins, ctl);
    note_launch();
  }
  kc<<<(unsigned)blocks, ENC_NT, smem_c, st>>>(src, n, R, lengths, S, nch, ctl,
                                               nzp ? words : nullptr);
  k_scan_pair<<<(unsigned)npt, PS_NT, 0, st>>>(S, nch, mode, out, cap_bytes / 4, ctl, bit_base,
                                                lengths, words, R, n, nzp ? 1 : 0);
  per_sm = occupancy((const void *)kp, ENC_NT, smem_p);
  blocks = (u64)sms * (per_sm < 1 ? 1 : per_sm);
  if (blocks > wblocks) blocks = wblocks;
  kp<<<(unsigned)blocks, ENC_NT, smem_p, st>>>(src, n, R, lengths, words, out, cap_bytes / 4,
                                               xval, o_idx, o_val, o_cap, S, nch, idx_offset,
                                               ctl, bit_base);
  note_launch(3);
  if (mode == 0) {
    // sparse alternative (each kernel checks the same device-side predicate)
    if (!nzp)
      k_enc_zero<<<(unsigned)(sms * 4), 256, 0, st>>>(lengths, words, R, n, out, cap_bytes / 4,
                                                      ctl, bit_base);
    const auto *s16 = reinterpret_cast<const uint16_t *>(src);
    if (nzp) {
      const u64 nsc = (n + NZ_SC - 1) / NZ_SC;
      const unsigned nb = (unsigned)((nsc + NZ_FW - 1) / NZ_FW);
      k_enc_nz_count<<<nb, NZ_FW * 32, 0, st>>>(s16, nzmap, n, R, lengths, words, S, nsc, ctl,
                                                 out, cap_bytes / 4, bit_base);
      k_scan_pair<<<(unsigned)((nsc + PS_TILE - 1) / PS_TILE), PS_NT, 0, st>>>(
          S, nsc, mode, out, cap_bytes / 4, ctl, bit_base, lengths, words, R, n, 2);
      k_enc_nz_emit<<<nb, NZ_FW * 32, 0, st>>>(s16, nzmap, n, R, lengths, words, out,
                                               cap_bytes / 4, xval, o_idx, o_val, o_cap, S, nsc,
                                               idx_offset, ctl, bit_base);
      // o_val is not filled on this path: the caller gathers x[o_idx] (k_assemble)
      note_launch(2);
    } else {
      const size_t smem_s = sizeof(uint2) * (nbins + 2) + 16;
      ensure_smem((const void *)k_enc_sparse, smem_s);
      per_sm = occupancy((const void *)k_enc_sparse, ENC_NT, smem_s);
      blocks = (u64)sms * (per_sm < 1 ? 1 : per_sm);
      if (blocks > wblocks) blocks = wblocks;
      k_enc_sparse<<<(unsigned)blocks, ENC_NT, smem_s, st>>>(
          s16, n, R, lengths, words, out, cap_bytes / 4, xval, o_idx, o_val, o_cap, S, nch,
          idx_offset, ctl, bit_base);
    }
    note_launch(2);
  }
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

u64 scan_scratch_bytes(u64 m);
int launch_excl_scan_u32(const uint32_t *in, u64 m, u64 *out, u64 *total, void *scratch,
                         cudaStream_t st);
u64 chain_scratch_bytes(u64 M, int D);
int launch_chain_resolve(const uint8_t *tab, u64 M, int D, int e0, uint8_t *entries,
                         void *scratch, cudaStream_t st);

static u64 dec_chunks(u64 nbytes) { return nbytes ? (nbytes * 8 + DEC_C - 1) / DEC_C : 1; }
// bytes of the speculative / synchronisation scratch over M chunks (SyncScratch)
static u64 sync_scratch_bytes(u64 M) { return M * (8 + 8 + 4 + 3) + 64 + 16 + 8 * 16; }  // nchg: 16 u32

u64 dec_scratch_bytes(u64 nbytes, int table_mode) {
  const u64 M = dec_chunks(nbytes);
  u64 b = M * (8 + 4 + 1) + 3 * 16 + sync_scratch_bytes(M) + M * 8 + 64 + scan_scratch_bytes(M) +
          256;
  if (table_mode) b += M * 32 * (1 + 4 + 1) + M + chain_scratch_bytes(M, 32) + 256;
  return b;
}

static unsigned char *carve(unsigned char *&p, u64 bytes) {
  unsigned char *r = p;
  p += (bytes + 15) & ~(u64)15;
  return r;
}

// Decode exactly n symbols.  out_kind 0: uint16 symbols, 1: int32 codes.
// table_mode != 0 selects the exact transfer-table path (lmax = longest code
// length), used when the speculative path reports non-convergence.
__global__ void k_set_u64(u64 *p, u64 v) { *p = v; }

static Stream make_stream(const uint8_t *bytes, u64 nbytes) {
  Stream s;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(bytes);
  s.w = reinterpret_cast<const uint32_t *>(addr & ~(uintptr_t)3);
  s.b0 = 8 * (addr & 3);
  s.nb = nbytes * 8;
  s.nwords = (s.b0 + s.nb + 31) / 32;
  return s;
}

// Scratch of the speculative / synchronisation phases over M chunks.
struct SyncScratch {
  u64 *spec_exit, *X1, *entry;
  uint32_t *spec_cnt, *nchg;
  uint8_t *spec_dead, *chg0, *chg1;
};
static SyncScratch carve_sync(unsigned char *&p, u64 M) {
  SyncScratch S;
  S.spec_exit = reinterpret_cast<u64 *>(carve(p, M * 8));
  S.X1 = reinterpret_cast<u64 *>(carve(p, M * 8));
  S.spec_cnt = reinterpret_cast<uint32_t *>(carve(p, M * 4));
  S.nchg = reinterpret_cast<uint32_t *>(carve(p, 64));
  S.entry = reinterpret_cast<u64 *>(carve(p, 16));
  S.spec_dead = carve(p, M);
  S.chg0 = carve(p, M);
  S.chg1 = carve(p, M);
  return S;
}

// Phases 1-2 over the chunk range [h0, h1) of a stream of M chunks: the
// speculative decode (of h0 - 1 as well, whose exit is the range's assumed
// entry unless `entry` is given) and three synchronisation iterations.
// X / K / D (full-length arrays) receive the range's true exits, symbol
// counts and dead flags; *entry_used the entry the range assumed;
// ctl->scratch[1] the number of chains still moving (0: converged).
static void huff_sync_range(const Stream &s, const DecTables *G, const uint16_t *sorted, u64 M,
                            u64 h0, u64 h1, u64 entry, u64 *X, uint32_t *K, uint8_t *D,
                            u64 *entry_used, const SyncScratch &S, cszi_ctl *ctl,
                            cudaStream_t st, int iters = 3, u64 *fd_init = nullptr) {
  // iters is odd: the last iteration writes X (even iterations write X,
  // odd ones the scratch copy)
  launch_zero16(S.nchg, 64, st);
  if (h1 <= h0) {
    cudaMemcpyAsync(&ctl->scratch[1], S.nchg, 4, cudaMemcpyDeviceToDevice, st);
    if (fd_init) {
      k_set_u64<<<1, 1, 0, st>>>(fd_init, ~0ull);
      note_launch();
    }
    return;
  }
  const u64 sb = (h0 > 0 && entry == ~0ull) ? h0 - 1 : h0;  // speculate h0 - 1 for the entry
  k_dec_spec<<<(unsigned)((h1 - sb + DEC_NT - 1) / DEC_NT), DEC_NT, 0, st>>>(
      s, G, sorted, h1, S.spec_exit, S.spec_cnt, S.spec_dead, sb, fd_init);
  note_launch();
  // the range's entry: 0 at the stream start, else the given one, else the
  // speculative exit of chunk h0 - 1 (device-resident: read by k_dec_sync)
  const u64 e0 = (h0 == 0) ? 0ull : entry;  // ~0: k_dec_sync takes spec_exit[h0 - 1]
  const unsigned blocks = (unsigned)((h1 - h0 + 255) / 256);
  // iteration 0 verifies every chunk; later iterations repair chunks whose
  // predecessor did not synchronise (blocks without one exit at once)
  for (int it = 0; it < iters; ++it) {
    u64 *Xo = (it & 1) ? S.X1 : X;
    const u64 *Xp = it ? ((it & 1) ? X : S.X1) : nullptr;
    uint8_t *co = (it & 1) ? S.chg1 : S.chg0;
    const uint8_t *cp = it ? ((it & 1) ? S.chg0 : S.chg1) : nullptr;
    k_dec_sync<<<blocks, 256, 0, st>>>(s, G, sorted, h1, it, S.spec_exit, S.spec_cnt,
                                       S.spec_dead, Xp, cp, Xo, K, D, co, S.nchg + it, h0,
                                       S.entry, e0);
    note_launch();
  }
  if (entry_used) cudaMemcpyAsync(entry_used, S.entry, 8, cudaMemcpyDeviceToDevice, st);
  // (fd_init: the whole-stream decode, whose write phase copies the count)
  if (!fd_init)
    cudaMemcpyAsync(&ctl->scratch[1], S.nchg + iters - 1, 4, cudaMemcpyDeviceToDevice, st);
}

// Phase 3-4 over all M chunks: exclusive scan of the symbol counts,
// truncation check, and the write of the symbol window [w0, w1).
// first_dead of huff_write's scratch starting at p (the same carving)
static u64 *write_first_dead(unsigned char *p, u64 M) {
  carve(p, M * 8);
  return reinterpret_cast<u64 *>(carve(p, 64)) + 2;
}

// fd_ready: first_dead was set by the speculative decode and the sync's
// moving-chain count (*nchg_last) goes to ctl->scratch[1] here
static void huff_write(const Stream &s, const DecTables *G, const uint16_t *sorted, u64 M,
                       const u64 *X, uint32_t *K, const uint8_t *D, u64 n, int R, void *out,
                       int out_kind, u64 w0, u64 w1, unsigned char *p, cszi_ctl *ctl,
                       cudaStream_t st, bool fd_ready = false,
                       const uint32_t *nchg_last = nullptr) {
  u64 *off = reinterpret_cast<u64 *>(carve(p, M * 8));
  u64 *misc = reinterpret_cast<u64 *>(carve(p, 64));
  u64 *first_dead = misc + 2;
  u64 *total = misc + 3;
  void *scan_ws = carve(p, scan_scratch_bytes(M));
  if (!fd_ready) {
    k_set_u64<<<1, 1, 0, st>>>(first_dead, ~0ull);  // (a kernel: no memset node)
    note_launch();
  }
  const unsigned blocks = (unsigned)((M + 255) / 256);
  const unsigned dblocks = (unsigned)((M + DEC_NT - 1) / DEC_NT);
  launch_excl_scan_u32(K, M, off, total, scan_ws, st);
  k_dec_first_dead<<<blocks, 256, 0, st>>>(M, D, first_dead, nchg_last,
                                           nchg_last ? reinterpret_cast<u64 *>(&ctl->scratch[1])
                                                     : nullptr);
  note_launch();
  const DecCheck C{first_dead, total, ctl};
  if (out_kind == 0) {
    k_dec_write<uint16_t><<<dblocks, DEC_NT, 0, st>>>(s, G, sorted, M, X, off, K, n, R,
                                                      reinterpret_cast<uint16_t *>(out), w0, w1,
                                                      C);
    k_dec_write_zr<uint16_t><<<dblocks, DEC_NT, 0, st>>>(
        s, G, sorted, M, X, off, K, n, R, reinterpret_cast<uint16_t *>(out), w0, w1, C);
  } else {
    k_dec_write<int32_t><<<dblocks, DEC_NT, 0, st>>>(s, G, sorted, M, X, off, K, n, R,
                                                     reinterpret_cast<int32_t *>(out), w0, w1, C);
    k_dec_write_zr<int32_t><<<dblocks, DEC_NT, 0, st>>>(
        s, G, sorted, M, X, off, K, n, R, reinterpret_cast<int32_t *>(out), w0, w1, C);
  }
  note_launch(2);
}

u64 huff_split_scratch_bytes(u64 nbytes) {
  const u64 M = dec_chunks(nbytes);
  return sync_scratch_bytes(M) + M * 8 + 64 + scan_scratch_bytes(M) + 1024;
}

// table_mode != 0 selects the exact transfer-table path (lmax = longest code
// length), used when the speculative path reports non-convergence.
int launch_decode(const uint8_t *bytes, u64 nbytes, u64 n, int R, const void *dec_tables,
                  void *out, int out_kind, void *scratch, cszi_ctl *ctl, cudaStream_t st,
                  int table_mode, int lmax, u64 w0, u64 w1) {
  if (n == 0) return CSZI_OK;
  const Stream s = make_stream(bytes, nbytes);
  const DecTables *G = reinterpret_cast<const DecTables *>(dec_tables);
  const uint16_t *sorted = reinterpret_cast<const uint16_t *>(G + 1);
  const u64 M = dec_chunks(nbytes);
  unsigned char *p = reinterpret_cast<unsigned char *>(scratch);
  u64 *X0 = reinterpret_cast<u64 *>(carve(p, M * 8));
  uint32_t *K = reinterpret_cast<uint32_t *>(carve(p, M * 4));
  uint8_t *D = carve(p, M);
  const uint32_t *nchg_last = nullptr;
  if (!table_mode) {
    const SyncScratch S = carve_sync(p, M);
    // the whole stream is one range entering at bit 0; a chain still moving
    // after three iterations is reported in ctl->scratch[1] and the caller
    // reruns in table mode
    huff_sync_range(s, G, sorted, M, 0, M, 0, X0, K, D, nullptr, S, ctl, st, 3,
                    write_first_dead(p, M));
    nchg_last = S.nchg + 2;
  } else {
    if (lmax < 1 || lmax > 32) lmax = 32;
    uint8_t *tab = carve(p, M * lmax);
    uint32_t *ktab = reinterpret_cast<uint32_t *>(carve(p, M * lmax * 4));
    uint8_t *dtab = carve(p, M * lmax);
    uint8_t *E = carve(p, M);
    void *chain_ws = carve(p, chain_scratch_bytes(M, lmax));
    const u64 work = M * (u64)lmax;
    const unsigned blocks = (unsigned)((M + 255) / 256);
    k_dec_table<<<(unsigned)((work + 255) / 256), 256, 0, st>>>(s, G, sorted, M, lmax, tab,
                                                               ktab, dtab);
    note_launch();
    launch_chain_resolve(tab, M, lmax, 0, E, chain_ws, st);
    k_dec_from_tab<<<blocks, 256, 0, st>>>(M, lmax, E, ktab, dtab, X0, K, D);
    note_launch();
  }
  huff_write(s, G, sorted, M, X0, K, D, n, R, out, out_kind, w0, w1, p, ctl, st,
             nchg_last != nullptr, nchg_last);
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

// ---- split decode (sharded decompress): ranges of chunks per rank --------
u64 huff_chunks(u64 nbytes) { return dec_chunks(nbytes); }

int launch_huff_sync_range(const uint8_t *bytes, u64 nbytes, const void *dec_tables, u64 h0,
                           u64 h1, u64 entry, u64 *X, uint32_t *K, uint8_t *D, u64 *entry_used,
                           void *scratch, cszi_ctl *ctl, cudaStream_t st) {
  const Stream s = make_stream(bytes, nbytes);
  const DecTables *G = reinterpret_cast<const DecTables *>(dec_tables);
  const uint16_t *sorted = reinterpret_cast<const uint16_t *>(G + 1);
  const u64 M = dec_chunks(nbytes);
  if (h1 > M) h1 = M;
  unsigned char *p = reinterpret_cast<unsigned char *>(scratch);
  const SyncScratch S = carve_sync(p, M);
  // more repair iterations than the whole-stream decode (which falls back to
  // the exact table path): a range has no second chance at that
  huff_sync_range(s, G, sorted, M, h0, h1, entry, X, K, D, entry_used, S, ctl, st, 11);
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

int launch_huff_write_window(const uint8_t *bytes, u64 nbytes, u64 n, int R,
                             const void *dec_tables, const u64 *X, uint32_t *K, const uint8_t *D,
                             u64 w0, u64 w1, uint16_t *out, void *scratch, cszi_ctl *ctl,
                             cudaStream_t st) {
  if (n == 0) return CSZI_OK;
  const Stream s = make_stream(bytes, nbytes);
  const DecTables *G = reinterpret_cast<const DecTables *>(dec_tables);
  const uint16_t *sorted = reinterpret_cast<const uint16_t *>(G + 1);
  const u64 M = dec_chunks(nbytes);
  unsigned char *p = reinterpret_cast<unsigned char *>(scratch);
  carve_sync(p, M);  // (the same scratch block as the range phase)
  huff_write(s, G, sorted, M, X, K, D, n, R, out, 0, w0, w1, p, ctl, st);
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

}  // namespace cszi
