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
                                                    cszi_ctl *ctl) {
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
  for (int s = threadIdx.x; s < npow2; s += blockDim.x) {
    u64 k = ~0ull;
    if (s < nbins) {
      const u64 f = hist[s];
      len_s[s] = 0;
      if (f) {
        k = (f << 16) | (u64)s;
        atomicAdd(&alive, 1);
      }
    }
    keys[s] = k;
  }
  __syncthreads();
  const int m = alive;
  if (m == 0) {
    if (threadIdx.x == 0) ctl->flags |= CSZI_F_EMPTY_HISTOGRAM;
    for (int s = threadIdx.x; s < nbins; s += blockDim.x) {
      lengths[s] = 0;
      words[s] = 0;
    }
    return;
  }
  bitonic_sort_u64(keys, npow2);
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
  for (int s = threadIdx.x; s < nbins; s += blockDim.x) lengths[s] = len_s[s];
  __syncthreads();
  canonical_block(len_s, nbins, words, nullptr, nullptr, ctl);
}

__global__ void __launch_bounds__(CB_NT) k_canonical(const uint8_t *__restrict__ lengths,
                                                     int nbins, uint32_t *words,
                                                     DecTables *dec, cszi_ctl *ctl) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  uint8_t *len_s = sm_raw;
  for (int s = threadIdx.x; s < nbins; s += blockDim.x) len_s[s] = lengths[s];
  __syncthreads();
  uint16_t *sorted = dec ? reinterpret_cast<uint16_t *>(dec + 1) : nullptr;
  canonical_block(len_s, nbins, words, dec, sorted, ctl);
}

// ---------------------------------------------------------------------------
// encode: one MSB-first stream; tile offsets by decoupled look-back
// ---------------------------------------------------------------------------
// Each persistent block owns a contiguous range of tiles (ENC_SPT symbols
// per thread per tile).  Pass 1 sums the code lengths (and outliers) of the
// whole range; ONE decoupled look-back across blocks gives the range its
// global bit / outlier offsets.  Pass 2 re-reads the range tile by tile:
// a block scan gives every thread its bit offset, codes are packed MSB-first
// in a 64-bit register accumulator and written as whole 32-bit words to a
// shared staging buffer (atomicOr only on the <= 2 words a thread shares
// with its neighbours); the partial last word of a tile is carried into the
// next tile.  The two words a range shares with its neighbour ranges are
// merged by whichever block arrives second.
constexpr int ENC_NT = 256;
constexpr int ENC_SPT = 32;
constexpr int ENC_TILE = ENC_NT * ENC_SPT;

struct EncScratch {  // zeroed before each launch (except head/tail)
  u64 *st_bits;
  u64 *st_out;
  uint32_t *bflag;
  uint32_t *bhead;
  uint32_t *btail;
  uint32_t *ticket;
};

template <int MODE>
DEV void enc_load(const void *src, u64 n, int R, int nbins, u64 base, uint32_t (&sy)[ENC_SPT]) {
  if (MODE == 0) {
    const uint16_t *sp = reinterpret_cast<const uint16_t *>(src) + base;
    if (base + ENC_SPT <= n && (((uintptr_t)sp) & 15) == 0) {
#pragma unroll
      for (int q = 0; q < ENC_SPT / 8; ++q) {
        const uint4 a = __ldcs(reinterpret_cast<const uint4 *>(sp) + q);
        const uint32_t w4[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          sy[8 * q + 2 * j] = w4[j] & 0xffffu;
          sy[8 * q + 2 * j + 1] = w4[j] >> 16;
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < ENC_SPT; ++j) sy[j] = (base + j < n) ? sp[j] : 0xffffffffu;
    }
  } else {
    const int32_t *cp = reinterpret_cast<const int32_t *>(src) + base;
#pragma unroll
    for (int j = 0; j < ENC_SPT; ++j) {
      if (base + j < n) {
        const int64_t v = (int64_t)cp[j] + R;
        sy[j] = (v >= 0 && v < nbins) ? (uint32_t)v : 0xfffffffeu;
      } else {
        sy[j] = 0xffffffffu;
      }
    }
  }
}

// classify + count: returns bits; marks invalid symbols 0xffffffff
template <int MODE>
DEV uint32_t enc_count(uint32_t (&sy)[ENC_SPT], const uint2 *lut, int R, uint32_t &nout,
                       uint32_t &outmask, bool &unknown) {
  uint32_t nbits = 0;
  nout = 0;
  outmask = 0;
#pragma unroll
  for (int j = 0; j < ENC_SPT; ++j) {
    uint32_t s = sy[j];
    if (s == 0xffffffffu) continue;
    if (s == 0xfffffffeu) {
      unknown = true;
      sy[j] = 0xffffffffu;
      continue;
    }
    if (MODE == 0 && s == 0) {
      nout++;
      outmask |= 1u << j;
      s = (uint32_t)R;
      sy[j] = s;
    }
    const uint32_t l = lut[s].y;
    if (l == 0) {
      unknown = true;
      sy[j] = 0xffffffffu;
      continue;
    }
    nbits += l;
  }
  return nbits;
}

// merge a word shared with the neighbouring range (second arriver writes)
DEV void enc_boundary(uint32_t *out, u64 gw, uint32_t val, uint32_t *mine, uint32_t *other,
                      uint32_t *flag) {
  *mine = val;
  __threadfence();
  if (atomicAdd(flag, 1u) == 1u) {
    __threadfence();
    out[gw] = bswap32(val | ld_volatile_u32(other));
  }
}

template <int MODE>
__global__ void __launch_bounds__(ENC_NT) k_encode(const void *__restrict__ src, u64 n, int R,
                                                  const uint8_t *__restrict__ lengths,
                                                  const uint32_t *__restrict__ words,
                                                  uint32_t *__restrict__ out, u64 cap_words,
                                                  const float *__restrict__ xval, u64 *o_idx,
                                                  float *o_val, u64 o_cap, EncScratch S,
                                                  u64 ntiles, u64 tiles_per_block, u64 nranges,
                                                  u64 idx_offset, cszi_ctl *ctl) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  const int nbins = 2 * R;
  uint2 *lut = reinterpret_cast<uint2 *>(sm_raw);  // (word, length)
  uint32_t *stage = reinterpret_cast<uint32_t *>(lut + nbins);  // ENC_TILE + 2 words
  __shared__ uint32_t scan_ws32[ENC_NT / 32 + 1];
  __shared__ u64 red_ws[ENC_NT / 32 + 1];
  __shared__ u64 s_r, s_B, s_O;
  const int tid = threadIdx.x;
  for (int i = tid; i < nbins; i += ENC_NT) lut[i] = make_uint2(words[i], lengths[i]);
  if (tid == 0) s_r = atomicAdd(S.ticket, 1u);  // ranges in ticket order
  __syncthreads();
  const u64 r = s_r;
  if (r >= nranges) return;
  const u64 t0 = r * tiles_per_block;
  const u64 t1 = min(t0 + tiles_per_block, ntiles);
  // ---- pass 1: range totals ----
  u64 my_bits = 0, my_out = 0;
  bool unknown = false;
  for (u64 t = t0; t < t1; ++t) {
    uint32_t sy[ENC_SPT];
    enc_load<MODE>(src, n, R, nbins, t * ENC_TILE + (u64)tid * ENC_SPT, sy);
    uint32_t nout, outmask;
    my_bits += enc_count<MODE>(sy, lut, R, nout, outmask, unknown);
    my_out += nout;
  }
  if (unknown) atomicOr(&ctl->flags, (uint32_t)CSZI_F_UNKNOWN_SYMBOL);
  u64 range_bits, range_out;
  block_excl_scan<ENC_NT, u64>(my_bits, red_ws, range_bits);
  block_excl_scan<ENC_NT, u64>(my_out, red_ws, range_out);
  if (tid < 32) {
    const u64 B = lookback_exclusive(S.st_bits, r, range_bits);
    const u64 O = (MODE == 0) ? lookback_exclusive(S.st_out, r, range_out) : 0;
    if (tid == 0) {
      s_B = B;
      s_O = O;
    }
  }
  __syncthreads();
  const u64 RB = s_B, RO = s_O;  // range offsets
  const bool last_range = (r + 1 == nranges);
  // ---- pass 2: pack ----
  u64 tb = RB;  // global bit offset of the current tile
  u64 to = RO;
  uint32_t carry = 0;  // partial last word carried from the previous tile
  for (u64 t = t0; t < t1; ++t) {
    const u64 base = t * ENC_TILE + (u64)tid * ENC_SPT;
    uint32_t sy[ENC_SPT];
    enc_load<MODE>(src, n, R, nbins, base, sy);
    uint32_t nout, outmask;
    bool unk2 = false;
    const uint32_t nbits = enc_count<MODE>(sy, lut, R, nout, outmask, unk2);
    uint32_t tot_bits, tot_out = 0;
    const uint32_t bexcl = block_excl_scan<ENC_NT, uint32_t>(nbits, scan_ws32, tot_bits);
    uint32_t oexcl = 0;
    if (MODE == 0) oexcl = block_excl_scan<ENC_NT, uint32_t>(nout, scan_ws32, tot_out);
    const uint32_t off0 = (uint32_t)(tb & 31);
    const uint32_t nw = (off0 + tot_bits + 31) >> 5;
    for (uint32_t i = tid; i < nw + 1; i += ENC_NT) stage[i] = (i == 0) ? carry : 0u;
    __syncthreads();
    if (MODE == 0 && outmask) {
      u64 k = to + oexcl;
      uint32_t m = outmask;
      while (m) {
        const int j = __ffs(m) - 1;
        m &= m - 1;
        const u64 gi = base + j;
        if (k < o_cap) {
          o_idx[k] = gi + idx_offset;
          o_val[k] = xval[gi];
        } else {
          atomicOr(&ctl->flags, (uint32_t)CSZI_F_CAPACITY);
        }
        k++;
      }
    }
    {
      const uint32_t pos = off0 + bexcl;
      uint32_t w = pos >> 5;
      const uint32_t fill = pos & 31;
      u64 acc = 0;
      uint32_t nb = fill;
      bool shared_head = fill != 0;
#pragma unroll
      for (int j = 0; j < ENC_SPT; ++j) {
        const uint32_t s = sy[j];
        if (s == 0xffffffffu) continue;
        const uint2 e = lut[s];
        acc = (acc << e.y) | (u64)e.x;
        nb += e.y;
        if (nb >= 32) {
          const uint32_t v = (uint32_t)(acc >> (nb - 32));
          if (shared_head) atomicOr(&stage[w], v);
          else stage[w] = v;
          shared_head = false;
          ++w;
          nb -= 32;
          acc &= (nb ? ((1ull << nb) - 1) : 0ull);
        }
      }
      if (nb > 0 && (nb > fill || !shared_head)) atomicOr(&stage[w], (uint32_t)(acc << (32 - nb)));
    }
    __syncthreads();
    const u64 gw0 = tb >> 5;
    const u64 end_bits = tb + tot_bits;
    const bool tail_partial = (end_bits & 31) != 0;
    const bool is_range_last_tile = (t + 1 == t1);
    // words [0, nw): word 0 is the range head when t == t0 and unaligned;
    // the last partial word is carried to the next tile, or is the range
    // tail (merged with the next range) on the range's last tile.
    for (uint32_t i = tid; i < nw; i += ENC_NT) {
      const u64 gw = gw0 + i;
      const uint32_t val = stage[i];
      const bool last_w = (i == nw - 1) && tail_partial;
      if (last_w && !is_range_last_tile) continue;  // carried
      if (gw >= cap_words) {
        atomicOr(&ctl->flags, (uint32_t)CSZI_F_CAPACITY);
        continue;
      }
      const bool head_w = (t == t0) && (i == 0) && (RB & 31) != 0;
      if (head_w && last_w && !last_range) {
        // the whole range fits inside one word shared on both sides: merge
        // with the previous range first (as head) and the next (as tail)
        enc_boundary(out, gw, val, &S.bhead[r], &S.btail[r], &S.bflag[r]);
      } else if (head_w) {
        enc_boundary(out, gw, val, &S.bhead[r], &S.btail[r], &S.bflag[r]);
      } else if (last_w && !last_range) {
        enc_boundary(out, gw, val, &S.btail[r + 1], &S.bhead[r + 1], &S.bflag[r + 1]);
      } else {
        out[gw] = bswap32(val);
      }
    }
    carry = (tail_partial && !is_range_last_tile) ? stage[nw - 1] : 0u;
    tb = end_bits;
    to += tot_out;
    __syncthreads();
  }
  if (last_range && tid == 0) {
    ctl->bits = RB + range_bits;
    if (MODE == 0) ctl->n_outliers = RO + range_out;
  }
}

// ---------------------------------------------------------------------------
// decode: self-synchronising chunked decode of one stream
// ---------------------------------------------------------------------------
constexpr u64 DEC_C = 1024;  // bits per chunk (32 words)

struct DecSmem {
  uint32_t lut[4096];
  u64 first_code[33];
  uint32_t first_index[33];
  uint32_t counts[33];
};

DEV void load_dec_smem(DecSmem &T, const DecTables *G) {
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) T.lut[i] = G->lut[i];
  for (int i = threadIdx.x; i < 33; i += blockDim.x) {
    T.first_code[i] = G->first_code[i];
    T.first_index[i] = G->first_index[i];
    T.counts[i] = G->counts[i];
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
  const uint32_t e = T.lut[win >> 20];
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

// Phase 1: speculative decode of chunk j from its first bit.
__global__ void __launch_bounds__(DEC_NT) k_dec_spec(Stream s, const DecTables *G,
                                                    const uint16_t *sorted, u64 M, u64 *spec_exit,
                                                    uint32_t *spec_cnt, uint8_t *spec_dead) {
  __shared__ DecSmem T;
  __shared__ uint32_t sw[DEC_SW];
  const u64 j0 = (u64)blockIdx.x * DEC_NT;
  SmemStream ss;
  stage_words(sw, s, j0, ss);
  load_dec_smem(T, G);  // ends with __syncthreads()
  const u64 j = j0 + threadIdx.x;
  if (j >= M) return;
  SmemReader br;
  br.init();
  u64 pos = j * DEC_C;
  const u64 end = min((j + 1) * DEC_C, s.nb);
  uint32_t cnt = 0;
  uint8_t dead = 0;
  while (pos < end) {
    uint32_t len;
    decode_at(T, sorted, br.peek(ss, pos), len);
    if (len == 0 || pos + len > s.nb) {
      dead = 1;
      break;
    }
    pos += len;
    cnt++;
  }
  spec_exit[j] = pos;
  spec_cnt[j] = cnt;
  spec_dead[j] = dead;
}

// Phase 2 (iteration `it`): chunk j decoded from its current entry estimate,
// walked in lockstep with its speculative decode until both chains meet.
// it == 0: entry = 0 (j == 0) or spec_exit[j-1]; it > 0: entry = X_prev[j-1]
// for chunks whose entry changed in the previous iteration.
__global__ void __launch_bounds__(256) k_dec_sync(Stream s, const DecTables *G,
                                                 const uint16_t *sorted, u64 M, int it,
                                                 const u64 *spec_exit, const uint32_t *spec_cnt,
                                                 const uint8_t *spec_dead, const u64 *X_prev,
                                                 const uint8_t *chg_prev, u64 *X, uint32_t *K,
                                                 uint8_t *D, uint8_t *chg, uint32_t *nchg) {
  __shared__ DecSmem T;
  load_dec_smem(T, G);
  const u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  if (j >= M) return;
  u64 e;
  if (it == 0) {
    e = (j == 0) ? 0 : spec_exit[j - 1];
  } else {
    if (j == 0 || !chg_prev[j - 1]) {
      X[j] = X_prev[j];
      chg[j] = 0;
      return;
    }
    e = X_prev[j - 1];
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
      uint32_t len;
      decode_at(T, sorted, ba.peek(s, a), len);
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
      uint32_t len;
      decode_at(T, sorted, bb.peek(s, b), len);
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
  if (c && j + 1 < M) atomicAdd(nchg, 1u);
}

// Phase 3 (after the generic exclusive scan of K into off): truncation
// check.  Decodable symbols = offset + count of the first chunk whose chain
// dies (invalid code / exhausted stream), or the total when none dies.
__global__ void k_dec_first_dead(u64 M, const uint8_t *D, u64 *first_dead) {
  const u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  if (j < M && D[j]) atomicMin(first_dead, j);
}
__global__ void k_dec_check(const u64 *off, const uint32_t *K, const u64 *first_dead,
                            const u64 *total, u64 n, cszi_ctl *ctl) {
  const u64 fd = *first_dead;
  const u64 avail = (fd != ~0ull) ? off[fd] + K[fd] : *total;
  ctl->decoded_symbols = avail;
  if (avail < n) ctl->flags |= CSZI_F_TRUNCATED;
}

// Fallback for streams whose chunks do not self-synchronise (e.g. codebooks
// with all lengths equal): exact per-chunk transfer tables over every entry
// offset 0 <= d < lmax, composed by the chain resolver.
__global__ void __launch_bounds__(256) k_dec_table(Stream s, const DecTables *G,
                                                  const uint16_t *sorted, u64 M, int lmax,
                                                  uint8_t *tab, uint32_t *ktab, uint8_t *dtab) {
  __shared__ DecSmem T;
  load_dec_smem(T, G);
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

template <typename OutT>
__global__ void __launch_bounds__(DEC_NT) k_dec_write(Stream s, const DecTables *G,
                                                     const uint16_t *sorted, u64 M, const u64 *X,
                                                     const u64 *off, u64 n, int R,
                                                     OutT *__restrict__ out) {
  __shared__ DecSmem T;
  __shared__ uint32_t sw[DEC_SW];
  constexpr int K = (sizeof(OutT) == 2) ? DEC_K : DEC_K / 2;
  __shared__ OutT ob[DEC_NT / 32][32][K + 1];
  const u64 j0 = (u64)blockIdx.x * DEC_NT;
  SmemStream ss;
  stage_words(sw, s, j0, ss);
  load_dec_smem(T, G);
  const u64 j = j0 + threadIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  u64 k = (j < M) ? off[j] : n;
  u64 pos = (j < M) ? ((j == 0) ? 0 : X[j - 1]) : 0;
  const u64 end = (j < M) ? min((j + 1) * DEC_C, s.nb) : 0;
  bool active = j < M && k < n;
  SmemReader br;
  br.init();
  while (__any_sync(CSZI_FULL, active)) {
    int cnt = 0;
    if (active) {
      while (cnt < K && pos < end && k + cnt < n) {
        uint32_t len;
        const uint32_t sym = decode_at(T, sorted, br.peek(ss, pos), len);
        if (len == 0 || pos + len > s.nb) {
          pos = end;  // dead chain: truncation is reported by k_dec_check
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
      if (lane < ci) out[ki + lane] = ob[warp][i][lane];
    }
    __syncwarp();
    k += cnt;
    active = active && cnt == K && pos < end && k < n;
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
                    cszi_ctl *ctl, cudaStream_t st) {
  if (nbins > 16384 || nbins < 1) return CSZI_E_UNSUPPORTED;
  int npow2 = 1;
  while (npow2 < nbins) npow2 <<= 1;
  // keys[npow2] + parent[2*nbins] + len[nbins] + internal keys / depths
  const size_t smem = sizeof(u64) * (npow2 + nbins) + sizeof(int32_t) * 3 * nbins + nbins + 16;
  cudaFuncSetAttribute(k_codebook, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_codebook<<<1, CB_NT, smem, st>>>(hist, nbins, lengths, words, ctl);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

size_t dec_tables_bytes(int nbins) { return sizeof(DecTables) + sizeof(uint16_t) * nbins + 16; }

int launch_canonical(const uint8_t *lengths, int nbins, uint32_t *words, void *dec_tables,
                     cszi_ctl *ctl, cudaStream_t st) {
  if (nbins > 65536 || nbins < 1) return CSZI_E_UNSUPPORTED;
  const size_t smem = nbins + 16;
  cudaFuncSetAttribute(k_canonical, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_canonical<<<1, CB_NT, smem, st>>>(lengths, nbins, words,
                                      reinterpret_cast<DecTables *>(dec_tables), ctl);
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
  const u64 nt = (n + ENC_TILE - 1) / ENC_TILE + 2;
  return nt * (8 + 8 + 4 + 4 + 4) + 64;
}

// mode 0: uint16 symbols with outlier sentinel; mode 1: int32 codes
int launch_encode(int mode, const void *src, u64 n, int R, const uint8_t *lengths,
                  const uint32_t *words, uint32_t *out, u64 cap_bytes, const float *xval,
                  u64 *o_idx, float *o_val, u64 o_cap, void *scratch, cszi_ctl *ctl,
                  cudaStream_t st, u64 idx_offset) {
  if (n == 0) return CSZI_OK;
  const u64 ntiles = (n + ENC_TILE - 1) / ENC_TILE;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const u64 want = (u64)sms * 4;
  const u64 tpb = (ntiles + want - 1) / want;
  const u64 nranges = (ntiles + tpb - 1) / tpb;
  const u64 nt = nranges + 2;
  unsigned char *p = reinterpret_cast<unsigned char *>(scratch);
  EncScratch S;
  S.st_bits = reinterpret_cast<u64 *>(p);
  S.st_out = S.st_bits + nt;
  S.bflag = reinterpret_cast<uint32_t *>(S.st_out + nt);
  S.ticket = S.bflag + nt;
  S.bhead = S.ticket + 4;
  S.btail = S.bhead + nt;
  cudaMemsetAsync(p, 0, (size_t)(nt * 8 * 2 + nt * 4 + 16), st);
  const int nbins = 2 * R;
  const size_t smem = sizeof(uint2) * nbins + sizeof(uint32_t) * (ENC_TILE + 2) + 16;
  if (mode == 0) {
    cudaFuncSetAttribute(k_encode<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_encode<0><<<(unsigned)nranges, ENC_NT, smem, st>>>(src, n, R, lengths, words, out,
                                                        cap_bytes / 4, xval, o_idx, o_val, o_cap,
                                                        S, ntiles, tpb, nranges, idx_offset,
                                                        ctl);
  } else {
    cudaFuncSetAttribute(k_encode<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_encode<1><<<(unsigned)nranges, ENC_NT, smem, st>>>(src, n, R, lengths, words, out,
                                                        cap_bytes / 4, xval, o_idx, o_val, o_cap,
                                                        S, ntiles, tpb, nranges, idx_offset,
                                                        ctl);
  }
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

u64 scan_scratch_bytes(u64 m);
int launch_excl_scan_u32(const uint32_t *in, u64 m, u64 *out, u64 *total, void *scratch,
                         cudaStream_t st);
u64 chain_scratch_bytes(u64 M, int D);
int launch_chain_resolve(const uint8_t *tab, u64 M, int D, int e0, uint8_t *entries,
                         void *scratch, cudaStream_t st);

static u64 dec_chunks(u64 nbytes) { return nbytes ? (nbytes * 8 + DEC_C - 1) / DEC_C : 1; }

u64 dec_scratch_bytes(u64 nbytes, int table_mode) {
  const u64 M = dec_chunks(nbytes);
  u64 b = M * (8 * 4 + 4 * 2 + 4) + 256 + scan_scratch_bytes(M) + 64;
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
int launch_decode(const uint8_t *bytes, u64 nbytes, u64 n, int R, const void *dec_tables,
                  void *out, int out_kind, void *scratch, cszi_ctl *ctl, cudaStream_t st,
                  int table_mode, int lmax) {
  if (n == 0) return CSZI_OK;
  Stream s;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(bytes);
  s.w = reinterpret_cast<const uint32_t *>(addr & ~(uintptr_t)3);
  s.b0 = 8 * (addr & 3);
  s.nb = nbytes * 8;
  s.nwords = (s.b0 + s.nb + 31) / 32;
  const DecTables *G = reinterpret_cast<const DecTables *>(dec_tables);
  const uint16_t *sorted = reinterpret_cast<const uint16_t *>(G + 1);
  const u64 M = dec_chunks(nbytes);
  unsigned char *p = reinterpret_cast<unsigned char *>(scratch);
  u64 *spec_exit = reinterpret_cast<u64 *>(carve(p, M * 8));
  u64 *X0 = reinterpret_cast<u64 *>(carve(p, M * 8));
  u64 *X1 = reinterpret_cast<u64 *>(carve(p, M * 8));
  u64 *off = reinterpret_cast<u64 *>(carve(p, M * 8));
  uint32_t *spec_cnt = reinterpret_cast<uint32_t *>(carve(p, M * 4));
  uint32_t *K = reinterpret_cast<uint32_t *>(carve(p, M * 4));
  u64 *misc = reinterpret_cast<u64 *>(carve(p, 64));  // nchg[4] (u32), first_dead, total
  uint32_t *nchg = reinterpret_cast<uint32_t *>(misc);
  u64 *first_dead = misc + 2;
  u64 *total = misc + 3;
  uint8_t *spec_dead = carve(p, M);
  uint8_t *D = carve(p, M);
  uint8_t *chg0 = carve(p, M);
  uint8_t *chg1 = carve(p, M);
  void *scan_ws = carve(p, scan_scratch_bytes(M));
  cudaMemsetAsync(misc, 0, 16, st);
  cudaMemsetAsync(first_dead, 0xff, 8, st);
  const unsigned blocks = (unsigned)((M + 255) / 256);
  const unsigned dblocks = (unsigned)((M + DEC_NT - 1) / DEC_NT);
  if (!table_mode) {
    k_dec_spec<<<dblocks, DEC_NT, 0, st>>>(s, G, sorted, M, spec_exit, spec_cnt, spec_dead);
    note_launch();
    // iteration 0 verifies every chunk; two more iterations repair chunks
    // whose predecessor did not synchronise.  A chain still moving after
    // that is reported in ctl->scratch[1]; the caller reruns in table mode.
    k_dec_sync<<<blocks, 256, 0, st>>>(s, G, sorted, M, 0, spec_exit, spec_cnt, spec_dead,
                                       nullptr, nullptr, X0, K, D, chg0, nchg + 0);
    note_launch();
    k_dec_sync<<<blocks, 256, 0, st>>>(s, G, sorted, M, 1, spec_exit, spec_cnt, spec_dead, X0,
                                       chg0, X1, K, D, chg1, nchg + 1);
    note_launch();
    k_dec_sync<<<blocks, 256, 0, st>>>(s, G, sorted, M, 2, spec_exit, spec_cnt, spec_dead, X1,
                                       chg1, X0, K, D, chg0, nchg + 2);
    note_launch();
    cudaMemcpyAsync(&ctl->scratch[1], nchg + 2, 4, cudaMemcpyDeviceToDevice, st);
  } else {
    if (lmax < 1 || lmax > 32) lmax = 32;
    uint8_t *tab = carve(p, M * lmax);
    uint32_t *ktab = reinterpret_cast<uint32_t *>(carve(p, M * lmax * 4));
    uint8_t *dtab = carve(p, M * lmax);
    uint8_t *E = carve(p, M);
    void *chain_ws = carve(p, chain_scratch_bytes(M, lmax));
    const u64 work = M * (u64)lmax;
    k_dec_table<<<(unsigned)((work + 255) / 256), 256, 0, st>>>(s, G, sorted, M, lmax, tab,
                                                               ktab, dtab);
    note_launch();
    launch_chain_resolve(tab, M, lmax, 0, E, chain_ws, st);
    k_dec_from_tab<<<blocks, 256, 0, st>>>(M, lmax, E, ktab, dtab, X0, K, D);
    note_launch();
  }
  launch_excl_scan_u32(K, M, off, total, scan_ws, st);
  k_dec_first_dead<<<blocks, 256, 0, st>>>(M, D, first_dead);
  note_launch();
  k_dec_check<<<1, 1, 0, st>>>(off, K, first_dead, total, n, ctl);
  note_launch();
  if (out_kind == 0)
    k_dec_write<uint16_t><<<dblocks, DEC_NT, 0, st>>>(s, G, sorted, M, X0, off, n, R,
                                                      reinterpret_cast<uint16_t *>(out));
  else
    k_dec_write<int32_t><<<dblocks, DEC_NT, 0, st>>>(s, G, sorted, M, X0, off, n, R,
                                                     reinterpret_cast<int32_t *>(out));
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

}  // namespace cszi
