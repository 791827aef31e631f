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
// [0, 128] into a 2 KiB chunk (a literal run spills at most 128 bytes into
// the next chunk) pointer jumping gives the exit offset and output count;
// the chain resolver composes the tables; each chunk then walks its true
// control chain and expands it cooperatively.
#include "common.cuh"

namespace cszi {

u64 scan_scratch_bytes(u64 m);
int launch_excl_scan_u32(const uint32_t *in, u64 m, u64 *out, u64 *total, void *scratch,
                         cudaStream_t st);
u64 chain_scratch_bytes(u64 M, int D);
int launch_chain_resolve(const uint8_t *tab, u64 M, int D, int e0, uint8_t *entries,
                         void *scratch, cudaStream_t st);

constexpr int P2_NT = 256;
constexpr int P2_BPT = 16;
constexpr int P2_TILE = P2_NT * P2_BPT;
constexpr u64 RUNBIT = 1ull << 63;

struct P2EncScratch {
  u64 *st_seg;      // look-back status, byte tiles
  u64 *st_out;      // look-back status, segment tiles
  u64 *tile_base;   // segments starting before each byte tile
  u64 *seg_start;   // start | RUNBIT
  u64 *seg_out;     // output offset per segment
  uint32_t *tickets;  // [0] byte tiles (pass a), [1] segment tiles, [2] emit
  u64 *nseg;
};

DEV uint8_t ldb(const uint8_t *in, int64_t i, u64 n) {
  return (i >= 0 && (u64)i < n) ? __ldg(in + i) : (uint8_t)1;
}

// classification of 16 bytes [i0, i0+16) plus start flags
DEV uint32_t classify(const uint8_t *in, u64 n, u64 i0, uint32_t &runmask) {
  uint8_t b[P2_BPT + 4];
#pragma unroll
  for (int k = 0; k < P2_BPT + 4; ++k) b[k] = ldb(in, (int64_t)i0 + k - 2, n);
  // z at local k (position i0+k-2), valid for k in [1, P2_BPT+2]
  bool z[P2_BPT + 4];
#pragma unroll
  for (int k = 1; k < P2_BPT + 3; ++k) z[k] = b[k] == 0 && (b[k - 1] == 0 || b[k + 1] == 0);
  uint32_t starts = 0;
  runmask = 0;
#pragma unroll
  for (int k = 0; k < P2_BPT; ++k) {
    const u64 i = i0 + k;
    if (i >= n) break;
    const bool zc = z[k + 2];
    const bool zp = z[k + 1];
    if (i == 0 || zc != zp) starts |= 1u << k;
    if (zc) runmask |= 1u << k;
  }
  return starts;
}

__global__ void __launch_bounds__(P2_NT) k_p2_segments(const uint8_t *__restrict__ in,
                                                       const u64 *Np, P2EncScratch S) {
  __shared__ u64 ws[P2_NT / 32 + 1];
  __shared__ u64 s_t, s_pre;
  const u64 n = *Np;
  const u64 ntiles = (n + P2_TILE - 1) / P2_TILE;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_t = atomicAdd(&S.tickets[0], 1u);
    __syncthreads();
    const u64 t = s_t;
    if (t >= ntiles) break;
    const u64 i0 = t * P2_TILE + (u64)threadIdx.x * P2_BPT;
    uint32_t runmask;
    const uint32_t starts = classify(in, n, i0, runmask);
    u64 tot;
    const u64 ex = block_excl_scan<P2_NT, u64>((u64)__popc(starts), ws, tot);
    if (threadIdx.x < 32) {
      const u64 p = lookback_exclusive(S.st_seg, t, tot);
      if (threadIdx.x == 0) s_pre = p;
    }
    __syncthreads();
    u64 g = s_pre + ex;
    uint32_t m = starts;
    while (m) {
      const int k = __ffs(m) - 1;
      m &= m - 1;
      S.seg_start[g++] = (i0 + k) | (((runmask >> k) & 1u) ? RUNBIT : 0ull);
    }
    if (threadIdx.x == 0) {
      S.tile_base[t] = s_pre;
      if (t + 1 == ntiles) *S.nseg = s_pre + tot;
    }
  }
}

DEV u64 seg_size(u64 L, bool run) { return run ? (L + 127) / 128 : L + (L + 127) / 128; }

__global__ void __launch_bounds__(P2_NT) k_p2_sizes(const u64 *Np, P2EncScratch S,
                                                    cszi_ctl *ctl) {
  __shared__ u64 ws[P2_NT / 32 + 1];
  __shared__ u64 s_t, s_pre;
  const u64 n = *Np;
  const u64 nseg = (n == 0) ? 0 : *S.nseg;
  const u64 ntiles = (nseg + P2_TILE - 1) / P2_TILE;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_t = atomicAdd(&S.tickets[1], 1u);
    __syncthreads();
    const u64 t = s_t;
    if (t >= ntiles) break;
    const u64 g0 = t * P2_TILE + (u64)threadIdx.x * P2_BPT;
    u64 sz[P2_BPT];
    u64 sum = 0;
#pragma unroll
    for (int k = 0; k < P2_BPT; ++k) {
      const u64 g = g0 + k;
      sz[k] = 0;
      if (g < nseg) {
        const u64 a = S.seg_start[g];
        const u64 st = a & ~RUNBIT;
        const u64 en = (g + 1 < nseg) ? (S.seg_start[g + 1] & ~RUNBIT) : n;
        sz[k] = seg_size(en - st, (a & RUNBIT) != 0);
      }
      sum += sz[k];
    }
    u64 tot;
    const u64 ex = block_excl_scan<P2_NT, u64>(sum, ws, tot);
    if (threadIdx.x < 32) {
      const u64 p = lookback_exclusive(S.st_out, t, tot);
      if (threadIdx.x == 0) s_pre = p;
    }
    __syncthreads();
    u64 o = s_pre + ex;
#pragma unroll
    for (int k = 0; k < P2_BPT; ++k) {
      if (g0 + k < nseg) S.seg_out[g0 + k] = o;
      o += sz[k];
    }
    if (t + 1 == ntiles && threadIdx.x == 0) ctl->payload_len = s_pre + tot;
  }
}

__global__ void __launch_bounds__(P2_NT) k_p2_emit(const uint8_t *__restrict__ in, const u64 *Np,
                                                   P2EncScratch S, uint8_t *__restrict__ out) {
  __shared__ u64 ws[P2_NT / 32 + 1];
  const u64 n = *Np;
  const u64 nseg = (n == 0) ? 0 : *S.nseg;
  const u64 ntiles = (n + P2_TILE - 1) / P2_TILE;
  for (u64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const u64 i0 = t * P2_TILE + (u64)threadIdx.x * P2_BPT;
    uint32_t runmask;
    const uint32_t starts = classify(in, n, i0, runmask);
    u64 tot;
    const u64 ex = block_excl_scan<P2_NT, u64>((u64)__popc(starts), ws, tot);
    long long g = (long long)(S.tile_base[t] + ex) - 1;  // segment of byte i0-1
    u64 sst = 0, len = 0, O = 0;
    bool run = false;
    long long cur = -2;
#pragma unroll 1
    for (int k = 0; k < P2_BPT; ++k) {
      const u64 i = i0 + k;
      if (i >= n) break;
      if ((starts >> k) & 1u) g++;
      if (g != cur) {
        cur = g;
        const u64 a = S.seg_start[g];
        sst = a & ~RUNBIT;
        run = (a & RUNBIT) != 0;
        const u64 en = ((u64)g + 1 < nseg) ? (S.seg_start[g + 1] & ~RUNBIT) : n;
        len = en - sst;
        O = S.seg_out[g];
      }
      const u64 j = i - sst;
      const u64 jm = j & 127;
      if (run) {
        if (jm == 0) out[O + j / 128] = (uint8_t)(127 + min((u64)128, len - j));
      } else {
        const u64 c = j / 128;
        out[O + c * 129 + 1 + jm] = __ldg(in + i);
        if (jm == 0) out[O + c * 129] = (uint8_t)(min((u64)128, len - j) - 1);
      }
    }
    __syncthreads();
  }
}

u64 p2enc_scratch_bytes(u64 n) {
  const u64 nt = (n + P2_TILE - 1) / P2_TILE + 2;
  return nt * 8 * 3 + (n + 2) * 8 * 2 + nt * 8 + 256;
}

// in: device bytes; Np: device pointer to the byte count (<= cap_n)
int launch_pass2_encode(const uint8_t *in, const u64 *Np, u64 cap_n, uint8_t *out,
                        void *scratch, cszi_ctl *ctl, cudaStream_t st) {
  const u64 nt = (cap_n + P2_TILE - 1) / P2_TILE + 2;
  unsigned char *p = reinterpret_cast<unsigned char *>(scratch);
  P2EncScratch S;
  S.st_seg = reinterpret_cast<u64 *>(p);
  S.st_out = S.st_seg + nt;
  S.tickets = reinterpret_cast<uint32_t *>(S.st_out + nt);
  S.nseg = reinterpret_cast<u64 *>(S.tickets + 4);
  S.tile_base = S.nseg + 2;
  S.seg_start = S.tile_base + nt;
  S.seg_out = S.seg_start + cap_n + 2;
  cudaMemsetAsync(p, 0, (size_t)(nt * 16 + 16 + 16), st);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  u64 grid = (u64)sms * 4;
  const u64 tiles_max = (cap_n + P2_TILE - 1) / P2_TILE;
  if (grid > tiles_max) grid = tiles_max;
  if (grid < 1) grid = 1;
  k_p2_segments<<<(unsigned)grid, P2_NT, 0, st>>>(in, Np, S);
  note_launch();
  k_p2_sizes<<<(unsigned)grid, P2_NT, 0, st>>>(Np, S, ctl);
  note_launch();
  k_p2_emit<<<(unsigned)grid, P2_NT, 0, st>>>(in, Np, S, out);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

// ---------------------------------------------------------------------------
// decode
// ---------------------------------------------------------------------------
constexpr int P2D_C = 2048;
constexpr int P2D_D = 129;           // entry offsets 0..128
constexpr int P2D_P = P2D_C + 130;   // local positions incl. spill
constexpr uint32_t OVR = 0x80000000u;

__global__ void __launch_bounds__(256) k_p2d_tables(const uint8_t *__restrict__ in, u64 n,
                                                    uint8_t *tab, uint32_t *ctab) {
  __shared__ uint16_t nx[2][P2D_P];
  __shared__ uint32_t ct[2][P2D_P];
  const u64 c0 = (u64)blockIdx.x * P2D_C;
  const int clen = (int)min((u64)P2D_C, n - c0);
  for (int p = threadIdx.x; p < P2D_P; p += blockDim.x) {
    uint16_t x;
    uint32_t c;
    if (p < clen) {
      const uint32_t b = __ldg(in + c0 + p);
      if (b < 128) {
        x = (uint16_t)min(p + (int)b + 2, P2D_P - 1);
        c = b + 1;
        if (c0 + p + 1 + b + 1 > n) c |= OVR;  // literal overruns the stream
      } else {
        x = (uint16_t)(p + 1);
        c = b - 127;
      }
    } else {
      x = (uint16_t)p;
      c = 0;
    }
    nx[0][p] = x;
    ct[0][p] = c;
  }
  __syncthreads();
  int cur = 0;
  for (int r = 0; r < 12; ++r) {
    for (int p = threadIdx.x; p < P2D_P; p += blockDim.x) {
      const int a = nx[cur][p];
      nx[cur ^ 1][p] = nx[cur][a];
      const uint32_t c1 = ct[cur][p], c2 = ct[cur][a];
      ct[cur ^ 1][p] = ((c1 & ~OVR) + (c2 & ~OVR)) | ((c1 | c2) & OVR);
    }
    __syncthreads();
    cur ^= 1;
  }
  for (int e = threadIdx.x; e < P2D_D; e += blockDim.x) {
    const int x = nx[cur][e];
    tab[(u64)blockIdx.x * P2D_D + e] = (uint8_t)(x >= P2D_C ? x - P2D_C : 0);
    ctab[(u64)blockIdx.x * P2D_D + e] = ct[cur][e];
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

__global__ void __launch_bounds__(256) k_p2d_expand(const uint8_t *__restrict__ in, u64 n,
                                                    const uint8_t *E, const u64 *off,
                                                    uint8_t *__restrict__ out, u64 cap,
                                                    cszi_ctl *ctl) {
  __shared__ uint16_t ctrl[P2D_C];
  __shared__ uint32_t cout_[P2D_C];
  __shared__ int nctrl;
  __shared__ u64 ws[9];
  const u64 c0 = (u64)blockIdx.x * P2D_C;
  const u64 cend = min(c0 + P2D_C, n);
  if (threadIdx.x == 0) {
    int k = 0;
    u64 p = c0 + E[blockIdx.x];
    while (p < cend) {
      const uint32_t b = in[p];
      ctrl[k] = (uint16_t)(p - c0);
      const uint32_t o = b < 128 ? b + 1 : b - 127;
      cout_[k] = o;
      k++;
      p += (b < 128) ? b + 2 : 1;
    }
    nctrl = k;
  }
  __syncthreads();
  const int nc = nctrl;
  u64 carry = off[blockIdx.x];
  for (int base = 0; base < nc; base += blockDim.x) {
    const int k = base + threadIdx.x;
    const u64 o = (k < nc) ? cout_[k] : 0;
    u64 tot;
    const u64 ex = block_excl_scan<256, u64>(o, ws, tot);
    if (k < nc) {
      const u64 dst = carry + ex;
      const u64 src = c0 + ctrl[k];
      const uint32_t b = in[src];
      if (dst + o > cap) {
        atomicOr(&ctl->flags, (uint32_t)CSZI_F_CAPACITY);
      } else if (b < 128) {
        const u64 avail = (src + 1 < n) ? n - (src + 1) : 0;
        const u64 m = min((u64)o, avail);  // overrun already flagged Corrupt
        for (u64 q = 0; q < m; ++q) out[dst + q] = in[src + 1 + q];
      } else {
        for (u64 q = 0; q < o; ++q) out[dst + q] = 0;
      }
    }
    carry += tot;
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
  k_p2d_tables<<<(unsigned)M, 256, 0, st>>>(in, n, tab, ctab);
  note_launch();
  launch_chain_resolve(tab, M, P2D_D, 0, E, chain_ws, st);
  k_p2d_counts<<<(unsigned)((M + 255) / 256), 256, 0, st>>>(M, E, ctab, cnt, ctl);
  note_launch();
  launch_excl_scan_u32(cnt, M, off, reinterpret_cast<u64 *>(&ctl->raw_len), scan_ws, st);
  if (expand) { k_p2d_expand<<<(unsigned)M, 256, 0, st>>>(in, n, E, off, out, cap, ctl); note_launch(); }
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

}  // namespace cszi
