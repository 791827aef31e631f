// Pass-2 zero-run codec (codec id 0) for sm_100a.
//
// Reference semantics: pass2.py:10-16 (grammar), :30-37 (_zero_runs: runs of
// >= 2 zero bytes), :40-47 (_emit_literals: chunks of <= 128 bytes from the
// start of each literal stretch), :50-67 (encode), :70-86 (decode, Corrupt on
// a literal run that overruns the stream).
//
// Encode = a parallel segmentation: every byte is classified RUN (a zero
// with a zero neighbour) or LIT; maximal same-class stretches are segments.
// Segment starts are compacted in order (decoupled look-back), segment output
// sizes scanned (look-back), then every byte writes its output independently.
//
// Decode = exact per-chunk transfer tables: for each entry offset e in
// [0, 128] into a 256-byte chunk (a literal run spills at most 128 bytes into
// the next chunk) one backward pass gives the exit offset and output count;
// the chain resolver composes the tables; each chunk then walks its true
// control chain and expands it cooperatively.
#include "common.cuh"

namespace cszi {
void launch_zero16(void *p, u64 bytes, cudaStream_t st);

u64 scan_scratch_bytes(u64 m);
int launch_excl_scan_u32(const uint32_t *in, u64 m, u64 *out, u64 *total, void *scratch,
                         cudaStream_t st);
u64 chain_scratch_bytes(u64 M, int D);
int launch_chain_resolve(const uint8_t *tab, u64 M, int D, int e0, uint8_t *entries,
                         void *scratch, cudaStream_t st);

// Encoder (pass2.py:30-67) in three launches, warp-granular (a warp chunk is
// P2_CH = 1024 bytes, 32 per lane) and bit-parallel (a lane classifies its
// 32 bytes with a handful of 64-bit mask operations).  Every byte is RUN (a
// zero with a zero neighbour) or LIT; a byte whose class differs from its
// predecessor's starts a segment.  A byte's output depends on its distance j
// from its segment start: LIT emits itself plus a control byte when
// j % 128 == 0, RUN only the control at j % 128 == 0; a control's value needs
// the distance to the segment end, capped at 128 (and at n).
//   k_p2_summary  per chunk: last segment start, first segment start, class
//                 of the carried-in segment, output bytes from the first
//                 start on;
//   k_p2_scan     max-scan of starts -> carried-in phase -> chunk output
//                 sizes -> sum-scan (both by decoupled look-back);
//   k_p2_emit     per chunk: output assembled in a per-warp shared buffer,
//                 copied out coalesced (each output byte has one writer).
constexpr int P2_NT = 256;
constexpr int P2_NW = P2_NT / 32;
constexpr int P2_BPL = 32;                 // bytes per lane
constexpr int P2_CH = 32 * P2_BPL;         // bytes per warp chunk
constexpr int P2_OB = P2_CH + P2_CH / 128 + 32;  // max output of one chunk
constexpr uint32_t P2_NONE = 0xffffffffu;

struct P2EncScratch {
  u64 *last1;     // per chunk: last segment start + 1 (0: none)
  uint32_t *fs;   // per chunk: first segment start (local), P2_NONE if none
  uint32_t *rest; // per chunk: output bytes from the first start on
  uint8_t *lit0;  // per chunk: class of its first byte (1: literal)
  u64 *prev1;     // per chunk: last start before the chunk + 1
  u64 *out_off;   // per chunk: output offset
  u64 *st_max, *st_sum;  // look-back status of the scan tiles
  uint32_t *ticket;
};

// 4-bit mask of the zero bytes of w
DEV uint32_t zero_nibble(uint32_t w) {
  const uint32_t t = __vcmpeq4(w, 0u);
  return ((t & 0x08040201u) * 0x01010101u) >> 24;
}

struct P2Lane {
  uint32_t w[8];   // the lane's 32 bytes (past n read as 1)
  uint32_t zmask;  // RUN class per position
  uint32_t smask;  // segment starts
  uint32_t valid;  // positions < n
  u64 p0;
};

// Load and classify the 32 bytes of one lane of chunk c.
DEV void p2_lane(const uint8_t *__restrict__ in, u64 n, u64 c, P2Lane &L) {
  const int lane = threadIdx.x & 31;
  const u64 p0 = c * P2_CH + (u64)lane * P2_BPL;
  L.p0 = p0;
  if (p0 + P2_BPL <= n && ((reinterpret_cast<uintptr_t>(in + p0) & 15) == 0)) {
    const uint4 a = __ldcs(reinterpret_cast<const uint4 *>(in + p0));
    const uint4 b = __ldcs(reinterpret_cast<const uint4 *>(in + p0) + 1);
    L.w[0] = a.x; L.w[1] = a.y; L.w[2] = a.z; L.w[3] = a.w;
    L.w[4] = b.x; L.w[5] = b.y; L.w[6] = b.z; L.w[7] = b.w;
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint32_t x = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const u64 i = p0 + 4 * q + k;
        x |= (uint32_t)(i < n ? __ldg(in + i) : 1) << (8 * k);
      }
      L.w[q] = x;
    }
  }
  uint32_t zb = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) zb |= zero_nibble(L.w[q]) << (4 * q);
  // neighbours: 2 bytes before (previous lane), 1 after (next lane)
  const uint32_t prevw = __shfl_up_sync(CSZI_FULL, L.w[7], 1);
  const uint32_t nextw = __shfl_down_sync(CSZI_FULL, L.w[0], 1);
  uint32_t zlo, zhi;
  if (lane == 0) {
    const uint32_t b2 = (p0 >= 2) ? __ldg(in + p0 - 2) : 1u;
    const uint32_t b1 = (p0 >= 1) ? __ldg(in + p0 - 1) : 1u;
    zlo = (b2 == 0 ? 1u : 0u) | (b1 == 0 ? 2u : 0u);
  } else {
    zlo = zero_nibble(prevw) >> 2;  // bytes 2, 3 of the previous lane
  }
  if (lane == 31) {
    const u64 pn = p0 + P2_BPL;
    zhi = (pn < n && __ldg(in + pn) == 0) ? 1u : 0u;
  } else {
    zhi = zero_nibble(nextw) & 1u;
  }
  // bit i <-> position p0 - 2 + i
  const u64 Zb = (u64)zlo | ((u64)zb << 2) | ((u64)zhi << 34);
  const u64 Z = Zb & ((Zb << 1) | (Zb >> 1));
  const u64 S = Z ^ (Z << 1);
  L.valid = (p0 >= n) ? 0u : (n - p0 >= 32 ? 0xffffffffu : ((1u << (n - p0)) - 1u));
  L.zmask = (uint32_t)(Z >> 2) & L.valid;
  L.smask = ((uint32_t)(S >> 2) | (p0 == 0 ? 1u : 0u)) & L.valid;
}

// heads and output bytes of a lane whose carried-in segment started at
// cs (< p0); positions before `from` are excluded.
DEV uint32_t p2_heads(const P2Lane &L, u64 cs) {
  uint32_t heads = L.smask;
  const uint32_t kh = (uint32_t)((128 - ((L.p0 - cs) & 127)) & 127);
  const uint32_t fsl = L.smask ? (uint32_t)(__ffs(L.smask) - 1) : 32u;
  if (kh < fsl) heads |= (1u << kh);  // kh < 32 here
  return heads & L.valid;
}

__global__ void __launch_bounds__(P2_NT) k_p2_summary(const uint8_t *__restrict__ in,
                                                      const u64 *Np, P2EncScratch S) {
  const int lane = threadIdx.x & 31;
  const u64 n = *Np;
  const u64 nch = (n + P2_CH - 1) / P2_CH;
  const u64 stride = (u64)gridDim.x * P2_NW;
  for (u64 c = (u64)blockIdx.x * P2_NW + (threadIdx.x >> 5); c < nch; c += stride) {
    P2Lane L;
    p2_lane(in, n, c, L);
    const u64 mylast = L.smask ? L.p0 + (31 - __clz(L.smask)) + 1 : 0;
    u64 incl = warp_incl_max(mylast);
    u64 cs1 = __shfl_up_sync(CSZI_FULL, incl, 1);
    if (lane == 0) cs1 = 0;
    const u64 last1 = __shfl_sync(CSZI_FULL, incl, 31);
    const uint32_t myfirst = L.smask ? lane * P2_BPL + (__ffs(L.smask) - 1) : P2_NONE;
    uint32_t fs = myfirst;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) fs = min(fs, __shfl_xor_sync(CSZI_FULL, fs, o));
    uint32_t cnt;
    const uint32_t lit = ~L.zmask & L.valid;
    if (cs1) {
      cnt = __popc(lit) + __popc(p2_heads(L, cs1 - 1));
    } else if (L.smask) {
      const uint32_t from = ~((1u << (__ffs(L.smask) - 1)) - 1u);
      cnt = __popc(lit & from) + __popc(L.smask);
    } else {
      cnt = 0;
    }
    cnt = warp_sum(cnt);
    if (lane == 0) {
      S.last1[c] = last1;
      S.fs[c] = fs;
      S.rest[c] = cnt;
      S.lit0[c] = (L.valid & ~L.zmask & 1u) ? 1 : 0;
    }
  }
}

// 2 chunks per thread: 4x the tiles of the first version, so more SMs share
// the dependent summary loads (512^3: -2 us, RTM / 256x384x384 -3 us)
constexpr int P2S_NT = 256, P2S_IPT = 2, P2S_TILE = P2S_NT * P2S_IPT;
__global__ void __launch_bounds__(P2S_NT) k_p2_scan(const u64 *Np, P2EncScratch S,
                                                    cszi_ctl *ctl) {
  __shared__ u64 ws[P2S_NT / 32 + 1];
  __shared__ u64 s_t, s_pmax, s_psum;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u64 n = *Np;
  const u64 nch = (n + P2_CH - 1) / P2_CH;
  const u64 ntiles = (nch + P2S_TILE - 1) / P2S_TILE;
  if (threadIdx.x == 0) s_t = atomicAdd(S.ticket, 1u);
  __syncthreads();
  const u64 t = s_t;
  if (t >= ntiles) {
    if (t == 0 && threadIdx.x == 0) ctl->payload_len = 0;  // n == 0
    return;
  }
  const u64 c0 = t * P2S_TILE + (u64)threadIdx.x * P2S_IPT;
  // max-scan of last1 (inclusive within the thread's items)
  u64 lm = 0;
#pragma unroll
  for (int i = 0; i < P2S_IPT; ++i)
    if (c0 + i < nch) lm = max(lm, S.last1[c0 + i]);
  u64 incl = warp_incl_max(lm);
  if (lane == 31) ws[warp] = incl;
  __syncthreads();
  u64 tile_max = 0, wpre = 0;
#pragma unroll
  for (int w = 0; w < P2S_NT / 32; ++w) {
    if (w < warp) wpre = max(wpre, ws[w]);
    tile_max = max(tile_max, ws[w]);
  }
  u64 ex = __shfl_up_sync(CSZI_FULL, incl, 1);
  if (lane == 0) ex = 0;
  ex = max(ex, wpre);
  if (warp == 0) {
    const u64 pm = lookback_exclusive<true>(S.st_max, t, tile_max);
    if (lane == 0) s_pmax = pm;
  }
  __syncthreads();
  u64 run = max(ex, s_pmax);  // last start + 1 before item c0
  u64 cnt[P2S_IPT];
  u64 sum = 0;
#pragma unroll
  for (int i = 0; i < P2S_IPT; ++i) {
    const u64 c = c0 + i;
    cnt[i] = 0;
    if (c < nch) {
      const uint32_t fs = S.fs[c];
      const u64 len = min((u64)P2_CH, n - c * P2_CH);
      const u64 l0 = (fs == P2_NONE) ? len : fs;
      u64 k = S.rest[c];
      if (l0 > 0) {  // run >= 1: position 0 starts a segment
        const u64 d = c * P2_CH - (run - 1);
        k += (S.lit0[c] ? l0 : 0) + ((d + l0 - 1) / 128 - (d - 1) / 128);
      }
      S.prev1[c] = run;
      run = max(run, S.last1[c]);
      cnt[i] = k;
      sum += k;
    }
  }
  __syncthreads();
  u64 tot;
  const u64 so = block_excl_scan<P2S_NT, u64>(sum, ws, tot);
  if (warp == 0) {
    const u64 ps = lookback_exclusive<false>(S.st_sum, t, tot);
    if (lane == 0) s_psum = ps;
  }
  __syncthreads();
  u64 o = s_psum + so;
#pragma unroll
  for (int i = 0; i < P2S_IPT; ++i) {
    if (c0 + i < nch) S.out_off[c0 + i] = o;
    o += cnt[i];
  }
  if (t + 1 == ntiles && threadIdx.x == 0) ctl->payload_len = s_psum + tot;
}

__global__ void __launch_bounds__(P2_NT) k_p2_emit(const uint8_t *__restrict__ in, const u64 *Np,
                                                   P2EncScratch S, uint8_t *__restrict__ out) {
  __shared__ uint8_t obuf[P2_NW][P2_OB];
  __shared__ uint32_t ibuf[P2_NW][P2_CH / 4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t *ob = obuf[warp];
  uint32_t *iw = ibuf[warp] + lane * (P2_BPL / 4);
  const uint8_t *ib = reinterpret_cast<const uint8_t *>(iw);
  const u64 n = *Np;
  const u64 nch = (n + P2_CH - 1) / P2_CH;
  const u64 stride = (u64)gridDim.x * P2_NW;
  for (u64 c = (u64)blockIdx.x * P2_NW + warp; c < nch; c += stride) {
    const u64 prev1 = S.prev1[c];
    const u64 O = S.out_off[c];
    const uint32_t fsn = (c + 1 < nch) ? S.fs[c + 1] : P2_NONE;
    P2Lane L;
    p2_lane(in, n, c, L);
    const u64 mylast = L.smask ? L.p0 + (31 - __clz(L.smask)) + 1 : 0;
    u64 incl = warp_incl_max(mylast);
    u64 cs1 = __shfl_up_sync(CSZI_FULL, incl, 1);
    if (lane == 0) cs1 = 0;
    cs1 = max(cs1, prev1);  // >= 1
    const uint32_t heads = p2_heads(L, cs1 - 1);
    const uint32_t lit = ~L.zmask & L.valid;
#pragma unroll
    for (int q = 0; q < P2_BPL / 4; ++q) iw[q] = L.w[q];
    const uint32_t cnt = __popc(lit) + __popc(heads);
    const uint32_t incl_cnt = warp_incl_scan(cnt);
    const uint32_t tot = __shfl_sync(CSZI_FULL, incl_cnt, 31);
    uint32_t o = incl_cnt - cnt;
    // first start after this lane: suffix minimum over later lanes, then the
    // next chunk's first start
    u64 nxt = L.smask ? L.p0 + (__ffs(L.smask) - 1) : ~0ull;
    if (lane == 31) {
      const u64 fn = (fsn == P2_NONE) ? ~0ull : (c + 1) * P2_CH + fsn;
      nxt = min(nxt, fn);
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u64 x = __shfl_down_sync(CSZI_FULL, nxt, d);
      if (lane + d < 32) nxt = min(nxt, x);
    }
    u64 after = __shfl_down_sync(CSZI_FULL, nxt, 1);
    if (lane == 31) after = (fsn == P2_NONE) ? ~0ull : (c + 1) * P2_CH + fsn;
    for (uint32_t m = lit | heads; m; m &= m - 1) {
      const int k = __ffs(m) - 1;
      const u64 p = L.p0 + k;
      const uint32_t byte = ib[k];
      const bool z = (L.zmask >> k) & 1u;
      if ((heads >> k) & 1u) {
        const uint32_t later = L.smask & ~((2u << k) - 1u);  // k = 31: (2u << 31) == 0
        const u64 ns = later ? L.p0 + (__ffs(later) - 1) : after;
        u64 len = min((u64)128, n - p);
        if (ns != ~0ull) len = min(len, ns - p);
        if (z) {
          ob[o++] = (uint8_t)(127 + len);
        } else {
          ob[o++] = (uint8_t)(len - 1);
          ob[o++] = (uint8_t)byte;
        }
      } else {
        ob[o++] = (uint8_t)byte;
      }
    }
    __syncwarp();
    for (uint32_t i = lane; i < tot; i += 32) out[O + i] = ob[i];
    __syncwarp();
  }
}

u64 p2enc_scratch_bytes(u64 n) {
  const u64 nc = (n + P2_CH - 1) / P2_CH + 2;
  const u64 nt = (nc + P2S_TILE - 1) / P2S_TILE + 2;
  return nc * (8 + 4 + 4 + 1 + 8 + 8) + nt * 16 + 256;
}

// in: device bytes; Np: device pointer to the byte count (<= cap_n)
int launch_pass2_encode(const uint8_t *in, const u64 *Np, u64 cap_n, uint8_t *out,
                        void *scratch, cszi_ctl *ctl, cudaStream_t st) {
  const u64 nc = (cap_n + P2_CH - 1) / P2_CH + 2;
  const u64 ntm = (nc + P2S_TILE - 1) / P2S_TILE;
  const u64 nt = ntm + 2;
  unsigned char *p = reinterpret_cast<unsigned char *>(scratch);
  P2EncScratch S;
  S.st_max = reinterpret_cast<u64 *>(p);  // zeroed: st_max, st_sum, ticket
  S.st_sum = S.st_max + nt;
  S.ticket = reinterpret_cast<uint32_t *>(S.st_sum + nt);
  S.last1 = reinterpret_cast<u64 *>(S.ticket + 4);
  S.prev1 = S.last1 + nc;
  S.out_off = S.prev1 + nc;
  S.fs = reinterpret_cast<uint32_t *>(S.out_off + nc);
  S.rest = S.fs + nc;
  S.lit0 = reinterpret_cast<uint8_t *>(S.rest + nc);
  launch_zero16(p, (u64)(nt * 16 + 16), st);  // (a kernel: no memset node in the graph)
  int sms = sm_count(), per_sm = 1;
  per_sm = occupancy((const void *)k_p2_emit, P2_NT, 0);
  if (per_sm < 1) per_sm = 1;
  u64 grid = (u64)sms * per_sm;
  const u64 wb = (nc + P2_NW - 1) / P2_NW;
  if (grid > wb) grid = wb;
  if (grid < 1) grid = 1;
  k_p2_summary<<<(unsigned)grid, P2_NT, 0, st>>>(in, Np, S);
  k_p2_scan<<<(unsigned)(ntm < 1 ? 1 : ntm), P2S_NT, 0, st>>>(Np, S, ctl);
  k_p2_emit<<<(unsigned)grid, P2_NT, 0, st>>>(in, Np, S, out);
  note_launch(3);
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

// ---------------------------------------------------------------------------
// decode
// ---------------------------------------------------------------------------
#ifndef P2D_CHUNK
#define P2D_CHUNK 256
#endif
constexpr int P2D_C = P2D_CHUNK;  // bytes of the stream per decode chunk
constexpr int P2D_D = 129;           // entry offsets 0..128
constexpr int P2D_P = P2D_C + 130;   // local positions incl. spill
constexpr uint32_t OVR = 0x80000000u;

// Transfer tables by a backward pass over the chunk, one warp per chunk.
// Every control's successor lies at most 129 bytes ahead (a literal header
// p jumps to p + b + 2 <= p + 129), so (exit, count) of a position follows
// from its successor's: X[p] = X[next(p)], C[p] = c(p) + C[next(p)], with
// positions >= clen terminal (X = p, C = 0).  The warp walks the chunk in
// 32-byte windows from its end: successors past the window are read from a
// 256-entry ring in shared memory (they are at most 160 positions ahead),
// successors inside the window are resolved by pointer jumping over the
// lanes (<= 5 shuffle rounds).  The windows over positions 0..128 are the
// table.  (Replaces pointer doubling over all 1154 positions: 4x fewer
// instructions.)
constexpr int P2T_WPB = 8;    // warps (chunks) per block
constexpr int P2T_RING = 256;
// chunks [jbase, jend) of the stream
__global__ void __launch_bounds__(P2T_WPB * 32) k_p2d_tables(const uint8_t *__restrict__ in,
                                                            u64 n, uint8_t *tab, uint32_t *ctab,
                                                            u64 jbase, u64 jend) {
  __shared__ uint16_t rx[P2T_WPB][P2T_RING];
  __shared__ uint32_t rc[P2T_WPB][P2T_RING];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const u64 jb = jbase + (u64)blockIdx.x * P2T_WPB + w;
  if (jb >= jend) return;
  const u64 c0 = jb * P2D_C;
  const int clen = (int)min((u64)P2D_C, n - c0);
  uint16_t *RX = rx[w];
  uint32_t *RC = rc[w];
  const int wtop = ((clen - 1) >> 5) << 5;  // window holding the last control
  uint32_t bnext = (c0 + wtop + lane < n) ? (uint32_t)__ldg(in + c0 + wtop + lane) : 0u;
  for (int w0 = wtop; w0 >= 0; w0 -= 32) {
    const int p = w0 + lane;
    const uint32_t b = bnext;
    if (w0 >= 32) bnext = __ldg(in + c0 + w0 - 32 + lane);  // prefetch (always in range)
    int X;
    uint32_t acc;
    int ptr = lane;
    bool res = true;
    if (p >= clen) {
      X = p;
      acc = 0;
    } else {
      int nx;
      if (b < 128) {
        nx = p + (int)b + 2;
        acc = b + 1;
        if (c0 + p + 1 + b + 1 > n) acc |= OVR;  // literal overruns the stream
      } else {
        nx = p + 1;
        acc = b - 127;
      }
      if (nx >= clen) {
        X = nx;
      } else if (nx >= w0 + 32) {
        X = RX[nx & (P2T_RING - 1)];
        const uint32_t c2 = RC[nx & (P2T_RING - 1)];
        acc = ((acc & ~OVR) + (c2 & ~OVR)) | ((acc | c2) & OVR);
      } else {
        X = 0;
        ptr = nx - w0;
        res = false;
      }
    }
    while (!__all_sync(CSZI_FULL, res)) {
      // (exit | lane pointer | resolved) in one word: two shuffles a round
      const int q = ptr;
      const uint32_t pk = ((uint32_t)X << 6) | ((uint32_t)ptr << 1) | (res ? 1u : 0u);
      const uint32_t tpk = __shfl_sync(CSZI_FULL, pk, q);
      const uint32_t ta = __shfl_sync(CSZI_FULL, acc, q);
      const bool tr = tpk & 1u;
      const int tx = (int)(tpk >> 6);
      const int tp = (int)((tpk >> 1) & 31u);
      if (!res) {
        acc = ((acc & ~OVR) + (ta & ~OVR)) | ((acc | ta) & OVR);
        if (tr) {
          X = tx;
          res = true;
        } else {
          ptr = tp;
        }
      }
    }
    RX[p & (P2T_RING - 1)] = (uint16_t)X;
    RC[p & (P2T_RING - 1)] = acc;
    if (p < P2D_D) {
      tab[jb * P2D_D + p] = (uint8_t)(X >= P2D_C ? X - P2D_C : 0);
      ctab[jb * P2D_D + p] = acc;
    }
    __syncwarp();
  }
  // entries past the last window (clen < 129: the stream's short tail)
  for (int e = wtop + 32 + lane; e < P2D_D; e += 32) {
    tab[jb * P2D_D + e] = (uint8_t)(e >= P2D_C ? e - P2D_C : 0);
    ctab[jb * P2D_D + e] = 0;
  }
}

__global__ void k_p2d_counts(u64 M, const uint8_t *E, const uint32_t *ctab, uint32_t *cnt,
                             cszi_ctl *ctl) {
  const u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  if (j >= M) return;
  const uint32_t c = ctab[j * P2D_D + E[j]];
  if (c & OVR) atomicOr(&ctl->flags, (uint32_t)CSZI_F_P2_CORRUPT);
  cnt[j] = c & ~OVR;
}

// Expand: one warp per chunk.  The chunk's output range [off, off + cnt)
// is zero-filled with coalesced 16-byte stores; the control chain is then
// walked 32 bytes at a time: lane l holds byte l of the window, the chain
// positions inside the window come from pointer jumping over the lanes
// (5 shuffle rounds for the 1..16-step successors, 5 OR-reductions to mark
// the positions reachable from the window's entry), a warp scan gives each
// control its output offset, and only literal payload bytes are stored
// (consecutive lanes -> consecutive output bytes).  A literal payload that
// runs past the window (or past the chunk, <= 128 bytes) is carried.
constexpr int P2X_WPB = 8;  // warps (chunks) per block
__global__ void __launch_bounds__(P2X_WPB * 32) k_p2d_expand(const uint8_t *__restrict__ in,
                                                            u64 n, const uint8_t *E,
                                                            const u64 *off,
                                                            const uint32_t *cnt,
                                                            uint8_t *__restrict__ out, u64 cap,
                                                            u64 M, cszi_ctl *ctl, u64 jbase) {
  const int lane = threadIdx.x & 31;
  const u64 j = jbase + (u64)blockIdx.x * P2X_WPB + (threadIdx.x >> 5);
  if (j >= M) return;
  const u64 c0 = j * P2D_C;
  const u64 cend = min(c0 + P2D_C, n);  // controls start below cend
  u64 obase = off[j];
  const u64 oend = obase + cnt[j];
  if (oend > cap) {
    if (lane == 0) atomicOr(&ctl->flags, (uint32_t)CSZI_F_CAPACITY);
    return;
  }
  {  // zero fill
    const u64 va = (obase + 15) / 16, vb = oend / 16;
    if (va <= vb) {
      for (u64 f = obase + lane; f < va * 16; f += 32) out[f] = 0;
      for (u64 v = va + lane; v < vb; v += 32)
        __stcs(reinterpret_cast<uint4 *>(out) + v, make_uint4(0, 0, 0, 0));
      for (u64 f = vb * 16 + lane; f < oend; f += 32) out[f] = 0;
    } else {
      for (u64 f = obase + lane; f < oend; f += 32) out[f] = 0;
    }
  }
  __syncwarp();
  int cur = E[j];                 // next control, relative to the window start
  u64 lit_lo = 0, lit_hi = 0;     // carried literal payload [lo, hi) (absolute)
  u64 lit_dst = 0;                // output position of lit_lo
  const u64 wend = min(c0 + P2D_C + 130, n);
  for (u64 w0 = c0; w0 < wend; w0 += 32) {
    if (cur >= 32 && lit_hi <= w0) {  // entry beyond this window and no payload:
      cur -= 32;                     // (the previous chunk's spill) skip it
      continue;
    }
    const u64 i = w0 + lane;
    const uint32_t b = (i < n) ? (uint32_t)__ldg(in + i) : 0u;
    const bool can_ctrl = i < cend;
    // successor of a control at this lane (32 = leaves the window)
    int nx = can_ctrl ? lane + (b < 128 ? (int)b + 2 : 1) : 32;
    if (nx > 32) nx = 32;
    int J[5];
    J[0] = nx;
#pragma unroll
    for (int r = 1; r < 5; ++r) {
      const int t = __shfl_sync(CSZI_FULL, J[r - 1], J[r - 1] & 31);
      J[r] = (J[r - 1] < 32) ? t : 32;
    }
    uint32_t on = 0;
    if (cur < 32) {
      on = 1u << cur;
#pragma unroll
      for (int r = 4; r >= 0; --r) {
        const uint32_t c = ((on >> lane) & 1u) && J[r] < 32 ? (1u << J[r]) : 0u;
        on |= __reduce_or_sync(CSZI_FULL, c);
      }
      on &= __ballot_sync(CSZI_FULL, can_ctrl);
    }
    const bool is_ctrl = (on >> lane) & 1u;
    const uint32_t o = is_ctrl ? (b < 128 ? b + 1 : b - 127) : 0u;
    // exclusive scan of output counts
    uint32_t inc = o;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(CSZI_FULL, inc, d);
      if (lane >= d) inc += t;
    }
    const uint32_t excl = inc - o;
    const uint32_t wtot = __shfl_sync(CSZI_FULL, inc, 31);
    // literal payload bytes: governed by the last control before the lane
    const uint32_t before = on & ((1u << lane) - 1u);
    u64 dst = ~0ull;
    const int cl = before ? 31 - __clz(before) : 0;
    const uint32_t bcl = __shfl_sync(CSZI_FULL, b, cl);
    const uint32_t excl_cl = __shfl_sync(CSZI_FULL, excl, cl);
    if (!is_ctrl && i < n) {
      if (before) {
        if (bcl < 128 && (uint32_t)(lane - cl) <= bcl + 1u)
          dst = obase + excl_cl + (u64)(lane - cl - 1);
      } else if (i >= lit_lo && i < lit_hi) {
        dst = lit_dst + (i - lit_lo);
      }
    }
    if (dst != ~0ull && dst < oend) out[dst] = (uint8_t)b;
    // carry: the window's last control
    u64 nabs;  // absolute position of the next control
    if (on) {
      const int L = 31 - __clz(on);
      const uint32_t bL = __shfl_sync(CSZI_FULL, b, L);
      const uint32_t exL = __shfl_sync(CSZI_FULL, excl, L);
      if (bL < 128) {
        lit_lo = w0 + L + 1;
        lit_hi = w0 + L + 2 + bL;
        lit_dst = obase + exL;
      } else {
        lit_lo = lit_hi = 0;
      }
      nabs = w0 + L + (bL < 128 ? bL + 2 : 1);
    } else {
      nabs = (cur >= (1 << 20)) ? cend : w0 + cur;
    }
    obase += wtot;
    if (nabs >= cend) {  // the chain left the chunk: finish the carried payload
      if (lit_hi <= w0 + 32) break;
      cur = 1 << 20;     // no more controls; keep storing payload bytes
    } else {
      cur = (int)(nabs - (w0 + 32));
    }
  }
}

static unsigned char *carve2(unsigned char *&p, u64 bytes) {
  unsigned char *r = p;
  p += (bytes + 15) & ~(u64)15;
  return r;
}

u64 p2dec_scratch_bytes(u64 n) {
  const u64 M = (n + P2D_C - 1) / P2D_C + 1;
  return M * (P2D_D * 5 + 1 + 4 + 8) + chain_scratch_bytes(M, P2D_D) + scan_scratch_bytes(M) +
         512;
}

// Phase A: sizes (tables, chain, counts, scan).  ctl->raw_len <- total.
// Phase B (expand) writes `out` (cap bytes).  expand == 0 stops after A.
int launch_pass2_decode(const uint8_t *in, u64 n, uint8_t *out, u64 cap, void *scratch,
                        cszi_ctl *ctl, cudaStream_t st, int expand) {
  if (n == 0) {
    cudaMemsetAsync(&ctl->raw_len, 0, 8, st);
    return CSZI_OK;
  }
  const u64 M = (n + P2D_C - 1) / P2D_C;
  unsigned char *p = reinterpret_cast<unsigned char *>(scratch);
  uint8_t *tab = carve2(p, M * P2D_D);
  uint32_t *ctab = reinterpret_cast<uint32_t *>(carve2(p, M * P2D_D * 4));
  uint8_t *E = carve2(p, M);
  uint32_t *cnt = reinterpret_cast<uint32_t *>(carve2(p, M * 4));
  u64 *off = reinterpret_cast<u64 *>(carve2(p, M * 8));
  void *chain_ws = carve2(p, chain_scratch_bytes(M, P2D_D));
  void *scan_ws = carve2(p, scan_scratch_bytes(M));
  k_p2d_tables<<<(unsigned)((M + P2T_WPB - 1) / P2T_WPB), P2T_WPB * 32, 0, st>>>(in, n, tab,
                                                                                 ctab, 0, M);
  note_launch();
  launch_chain_resolve(tab, M, P2D_D, 0, E, chain_ws, st);
  k_p2d_counts<<<(unsigned)((M + 255) / 256), 256, 0, st>>>(M, E, ctab, cnt, ctl);
  note_launch();
  launch_excl_scan_u32(cnt, M, off, reinterpret_cast<u64 *>(&ctl->raw_len), scan_ws, st);
  if (expand) {
    k_p2d_expand<<<(unsigned)((M + P2X_WPB - 1) / P2X_WPB), P2X_WPB * 32, 0, st>>>(
        in, n, E, off, cnt, out, cap, M, ctl, 0);
    note_launch();
  }
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

// ---- split decode (sharded decompress): chunk ranges per rank -------------
u64 p2d_chunks(u64 n) { return n ? (n + P2D_C - 1) / P2D_C : 0; }
u64 p2d_resolve_scratch_bytes(u64 n) {
  const u64 M = p2d_chunks(n) + 1;
  return chain_scratch_bytes(M, P2D_D) + scan_scratch_bytes(M) + 512;
}

int launch_p2d_tables_range(const uint8_t *in, u64 n, u64 c0, u64 c1, uint8_t *tab,
                            uint32_t *ctab, cudaStream_t st) {
  const u64 M = p2d_chunks(n);
  if (c1 > M) c1 = M;
  if (c1 > c0) {
    k_p2d_tables<<<(unsigned)((c1 - c0 + P2T_WPB - 1) / P2T_WPB), P2T_WPB * 32, 0, st>>>(
        in, n, tab, ctab, c0, c1);
    note_launch();
  }
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

int launch_p2d_resolve(const uint8_t *tab, const uint32_t *ctab, u64 n, uint8_t *E,
                       uint32_t *cnt, u64 *off, void *scratch, cszi_ctl *ctl, cudaStream_t st) {
  const u64 M = p2d_chunks(n);
  if (M == 0) {
    cudaMemsetAsync(&ctl->raw_len, 0, 8, st);
    return CSZI_OK;
  }
  unsigned char *p = reinterpret_cast<unsigned char *>(scratch);
  void *chain_ws = carve2(p, chain_scratch_bytes(M, P2D_D));
  void *scan_ws = carve2(p, scan_scratch_bytes(M));
  launch_chain_resolve(tab, M, P2D_D, 0, E, chain_ws, st);
  k_p2d_counts<<<(unsigned)((M + 255) / 256), 256, 0, st>>>(M, E, ctab, cnt, ctl);
  note_launch();
  launch_excl_scan_u32(cnt, M, off, reinterpret_cast<u64 *>(&ctl->raw_len), scan_ws, st);
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

int launch_p2d_expand_range(const uint8_t *in, u64 n, const uint8_t *E, const u64 *off,
                            const uint32_t *cnt, u64 c0, u64 c1, uint8_t *out, u64 cap,
                            cszi_ctl *ctl, cudaStream_t st) {
  const u64 M = p2d_chunks(n);
  if (c1 > M) c1 = M;
  if (c1 > c0) {
    k_p2d_expand<<<(unsigned)((c1 - c0 + P2X_WPB - 1) / P2X_WPB), P2X_WPB * 32, 0, st>>>(
        in, n, E, off, cnt, out, cap, c1, ctl, c0);
    note_launch();
  }
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

}  // namespace cszi
