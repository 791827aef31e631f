// Generic single-pass scans and the chunk-chain resolver.
//
// * excl_scan_u32: u32 values -> u64 exclusive prefix (decoupled look-back).
// * chain resolve: chunk j maps an entry state e (0 <= e < D) to the entry
//   state of chunk j+1 through a table tab[j][e].  Entries E[0] = e0,
//   E[j+1] = tab[j][E[j]] are resolved by a hierarchical composition of the
//   tables (groups of G chunks), which turns an M-step dependent walk into
//   ~G * log_G(M) dependent shared-memory lookups.  Used for the pass-2
//   control-byte chain (pass2.py:75-85: where a control byte sits depends on
//   every control before it) and for the Huffman self-sync fallback.
#include "common.cuh"

namespace cszi {

constexpr int SCAN_NT = 256;
constexpr int SCAN_IPT = 8;
constexpr int SCAN_TILE = SCAN_NT * SCAN_IPT;

__global__ void __launch_bounds__(SCAN_NT) k_excl_scan_u32(const uint32_t *__restrict__ in,
                                                         u64 m, u64 *__restrict__ out,
                                                         u64 *total, u64 *status,
                                                         uint32_t *ticket, u64 ntiles) {
  __shared__ u64 ws[SCAN_NT / 32 + 1];
  __shared__ u64 s_tile, s_pre;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const u64 t = s_tile;
  const u64 base = t * SCAN_TILE + (u64)threadIdx.x * SCAN_IPT;
  u64 v[SCAN_IPT];
  u64 sum = 0;
#pragma unroll
  for (int i = 0; i < SCAN_IPT; ++i) {
    v[i] = (base + i < m) ? in[base + i] : 0;
    sum += v[i];
  }
  u64 tot;
  const u64 ex = block_excl_scan<SCAN_NT, u64>(sum, ws, tot);
  if (threadIdx.x < 32) {
    const u64 p = lookback_exclusive(status, t, tot);
    if (threadIdx.x == 0) s_pre = p;
  }
  __syncthreads();
  u64 run = s_pre + ex;
#pragma unroll
  for (int i = 0; i < SCAN_IPT; ++i) {
    if (base + i < m) out[base + i] = run;
    run += v[i];
  }
  if (t + 1 == ntiles && threadIdx.x == 0 && total) *total = s_pre + tot;
}

u64 scan_scratch_bytes(u64 m) { return ((m + SCAN_TILE - 1) / SCAN_TILE + 1) * 8 + 16; }

// Zero a small 16-byte-aligned scratch block with a kernel: inside the
// captured graphs a memset node costs a 3-4 us gap on each side (the
// look-back tile states of the encoder and the pass-2 encoder).
__global__ void k_zero16(uint4 *p, u64 n16) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n16; i += (u64)gridDim.x * blockDim.x)
    p[i] = make_uint4(0, 0, 0, 0);
}
void launch_zero16(void *p, u64 bytes, cudaStream_t st) {
  const u64 n16 = (bytes + 15) / 16;
  u64 blocks = (n16 + 255) / 256;
  if (blocks > 1024) blocks = 1024;
  if (blocks < 1) blocks = 1;
  k_zero16<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<uint4 *>(p), n16);
  note_launch();
}

int launch_excl_scan_u32(const uint32_t *in, u64 m, u64 *out, u64 *total, void *scratch,
                         cudaStream_t st) {
  if (m == 0) {
    if (total) cudaMemsetAsync(total, 0, 8, st);
    return CSZI_OK;
  }
  const u64 ntiles = (m + SCAN_TILE - 1) / SCAN_TILE;
  u64 *status = reinterpret_cast<u64 *>(scratch);
  uint32_t *ticket = reinterpret_cast<uint32_t *>(status + ntiles);
  launch_zero16(scratch, ntiles * 8 + 16, st);
  k_excl_scan_u32<<<(unsigned)ntiles, SCAN_NT, 0, st>>>(in, m, out, total, status, ticket,
                                                        ntiles);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

// ---------------------------------------------------------------------------
// chain resolver
// ---------------------------------------------------------------------------
constexpr int CH_G = 64;  // chunks per group

// Stage a group's tables (bytes) in shared memory with 16-byte loads, all
// issued before the stores (a byte loop paid one L2 round trip per
// iteration: ~10 us per launch for 8 KB).
DEV void stage_tables(uint8_t *st, const uint8_t *__restrict__ src, int bytes) {
  const bool al = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(st)) & 15) == 0;
  const int nv = al ? bytes / 16 : 0;
  const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
  uint4 *d4 = reinterpret_cast<uint4 *>(st);
  constexpr int U = 4;
  for (int i0 = threadIdx.x; i0 < nv; i0 += U * blockDim.x) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < nv) v[u] = __ldg(s4 + i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < nv) d4[i] = v[u];
    }
  }
  for (int i = nv * 16 + threadIdx.x; i < bytes; i += blockDim.x) st[i] = src[i];
}

// up-sweep: group table out[g][e] = composition of the member tables
__global__ void __launch_bounds__(256) k_chain_up(const uint8_t *__restrict__ tab, u64 M, int D,
                                                  uint8_t *__restrict__ out) {
  extern __shared__ __align__(16) uint8_t st_[];
  const u64 g = blockIdx.x;
  const u64 c0 = g * CH_G;
  const int cnt = (int)min((u64)CH_G, M - c0);
  stage_tables(st_, tab + c0 * D, cnt * D);
  __syncthreads();
  for (int e = threadIdx.x; e < D; e += blockDim.x) {
    int x = e;
    for (int c = 0; c < cnt; ++c) x = st_[c * D + x];
    out[g * D + e] = (uint8_t)x;
  }
}

// down-sweep: member entries from the group entry (gentry == nullptr: e0)
__global__ void __launch_bounds__(256) k_chain_down(const uint8_t *__restrict__ tab, u64 M, int D,
                                                    const uint8_t *__restrict__ gentry, int e0,
                                                    uint8_t *__restrict__ entry) {
  extern __shared__ __align__(16) uint8_t st_[];
  const u64 g = blockIdx.x;
  const u64 c0 = g * CH_G;
  const int cnt = (int)min((u64)CH_G, M - c0);
  stage_tables(st_, tab + c0 * D, cnt * D);
  __syncthreads();
  if (threadIdx.x == 0) {
    int x = gentry ? gentry[g] : e0;
    for (int c = 0; c < cnt; ++c) {
      entry[c0 + c] = (uint8_t)x;
      x = st_[c * D + x];
    }
  }
}

u64 chain_scratch_bytes(u64 M, int D) {
  u64 total = 0;
  u64 m = M;
  while (m > (u64)CH_G) {
    m = (m + CH_G - 1) / CH_G;
    total += m * (u64)D + m + 64;
  }
  return total + 256;
}

// entries[j] for j < M (entry state of chunk j)
int launch_chain_resolve(const uint8_t *tab, u64 M, int D, int e0, uint8_t *entries,
                         void *scratch, cudaStream_t st) {
  if (M == 0) return CSZI_OK;
  // level tables and level entries live in scratch
  const int MAXL = 8;
  const uint8_t *ltab[MAXL];
  uint8_t *lent[MAXL];
  u64 lM[MAXL];
  int L = 0;
  ltab[0] = tab;
  lent[0] = entries;
  lM[0] = M;
  unsigned char *p = reinterpret_cast<unsigned char *>(scratch);
  const size_t smem = (size_t)CH_G * D;
  while (lM[L] > (u64)CH_G) {
    if (L + 1 >= MAXL) return CSZI_E_UNSUPPORTED;
    const u64 mg = (lM[L] + CH_G - 1) / CH_G;
    uint8_t *gt = p;
    p += mg * D;
    uint8_t *ge = p;
    p += mg + 64;
    k_chain_up<<<(unsigned)mg, 256, smem, st>>>(ltab[L], lM[L], D, gt);
    note_launch();
    ++L;
    ltab[L] = gt;
    lent[L] = ge;
    lM[L] = mg;
  }
  k_chain_down<<<1, 256, smem, st>>>(ltab[L], lM[L], D, nullptr, e0, lent[L]);
  note_launch();
  for (int l = L - 1; l >= 0; --l) {
    const u64 mg = (lM[l] + CH_G - 1) / CH_G;
    k_chain_down<<<(unsigned)mg, 256, smem, st>>>(ltab[l], lM[l], D, lent[l + 1], e0, lent[l]);
    note_launch();
  }
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

}  // namespace cszi
