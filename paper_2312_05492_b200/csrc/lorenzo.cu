// First-order Lorenzo predictor (the reference's baseline predictor,
// lorenzo.py:22-53 with the numba kernels of _kernels.py:104-215) for
// sm_100a: compress (predict + quantize against reconstructed neighbours)
// and decompress (replay), bit-exact with the reference.
//
// The reference is a raster-order recurrence: point (z, y, x) is predicted
// from the signed corner sum of the seven reconstructed points behind it,
//   pred = ((((((a1 + a2) + a3) - a4) - a5) - a6) + a7)        (float64)
// (a1 = r[z-1,y,x], a2 = r[z,y-1,x], a3 = r[z,y,x-1], a4 = r[z,y-1,x-1],
// a5 = r[z-1,y,x-1], a6 = r[z-1,y-1,x], a7 = r[z-1,y-1,x-1]; out-of-grid
// neighbours are 0), so each point depends on its own row's left
// neighbour.  Rank 2 and 1 are the same sum with the missing axes' terms
// 0 (adding / subtracting +0 only changes the sign of a zero prediction,
// which never reaches q, the reconstruction or the guard).
//
// GPU schedule: the grid is cut into tiles (TZ x TY x 32; 8 x 8 x 32 for
// rank 3, 1 x 32 x 32 for rank 2) that form a dependency DAG along the
// three axes; all tiles on one anti-diagonal wavefront tz + ty + tx = w are
// independent and run in one launch (one warp per tile), wavefront after
// wavefront.  Inside a tile lane l owns column x = l and processes row
// r = (z, y) at step k = r + l: its left neighbour (lane l - 1) finished the
// same row one step earlier, its own previous rows are older still, so a
// __syncwarp per step orders every read after the write it needs.  Tile
// halos (the plane / row / column behind the tile) come from the global
// reconstruction written by earlier wavefronts.  Rank 1 is a single
// sequential chain (no parallelism exists in the reference recurrence) and
// runs on one thread.
//
// Quantiser: predictor.py's rules with one global bound (eb, e2 = 2 eb):
// the shared fast / exact quantize<> (interp_common.cuh) -- identical to
// the reference's |t| < R - 0.5, |q| < R and |f64(r) - o| <= eb tests.
#include "common.cuh"
#include "interp_common.cuh"

namespace cszi {

struct LzGeo {
  int64_t ext[3];  // z, y, x (padded with leading 1s)
  int64_t nt[3];   // tiles per axis
};

struct LzQ {
  double eb, e2, inv;  // compress: from ctl (device), decompress: e2 only
  int R;
};

constexpr int LZ_TX = 32;
constexpr int LZ_NW = 4;  // warps (tiles) per CTA

template <int TZ, int TY>
struct LzTile {
  static constexpr int PX = LZ_TX + 1;                // x in [-1, 31]
  static constexpr int PY = TY + 1, PZ = TZ + 1;
  static constexpr int NB = PZ * PY * PX;             // recon + halo
  static constexpr int NO = TZ * TY * LZ_TX;          // owned
  static constexpr int BYTES = 4 * NB + 4 * NO + 2 * NO + 16;
};

// number of (ty, tx) with ty + tx = s, 0 <= ty < ny, 0 <= tx < nx
DEV int64_t diag_count(int64_t s, int64_t ny, int64_t nx) {
  if (s < 0) return 0;
  const int64_t lo = s - (nx - 1) > 0 ? s - (nx - 1) : 0;
  const int64_t hi = s < ny - 1 ? s : ny - 1;
  return hi >= lo ? hi - lo + 1 : 0;
}
static int64_t diag_count_h(int64_t s, int64_t ny, int64_t nx) {
  if (s < 0) return 0;
  const int64_t lo = s - (nx - 1) > 0 ? s - (nx - 1) : 0;
  const int64_t hi = s < ny - 1 ? s : ny - 1;
  return hi >= lo ? hi - lo + 1 : 0;
}

// i-th tile of wavefront w (tz ascending, then ty ascending)
DEV bool wave_tile(const LzGeo &G, int64_t w, int64_t i, int64_t t[3]) {
  for (int64_t tz = 0; tz < G.nt[0] && tz <= w; ++tz) {
    const int64_t c = diag_count(w - tz, G.nt[1], G.nt[2]);
    if (i < c) {
      const int64_t s = w - tz;
      const int64_t ty = (s - (G.nt[2] - 1) > 0 ? s - (G.nt[2] - 1) : 0) + i;
      t[0] = tz;
      t[1] = ty;
      t[2] = s - ty;
      return true;
    }
    i -= c;
  }
  return false;
}

DEV double lz_pred(const float *b, int i, int PX, int PZS) {
  // b[i] is the point; neighbours at -1 (x), -PX (y), -PZS (z)
  const double a1 = (double)b[i - PZS], a2 = (double)b[i - PX], a3 = (double)b[i - 1];
  const double a4 = (double)b[i - PX - 1], a5 = (double)b[i - PZS - 1];
  const double a6 = (double)b[i - PZS - PX], a7 = (double)b[i - PZS - PX - 1];
  return dadd(dsub(dsub(dsub(dadd(dadd(a1, a2), a3), a4), a5), a6), a7);
}

// One wavefront.  MODE 0: x (original) -> rec (reconstruction scratch) +
// sym (q + R, 0 for an outlier).  MODE 1: sym (0xFFFF at outliers) -> rec.
template <int TZ, int TY, int MODE>
__global__ void __launch_bounds__(LZ_NW * 32)
    k_lorenzo_wave(const float *__restrict__ x, float *rec, uint16_t *sym, LzGeo G, int64_t w,
                   int64_t count, const cszi_ctl *ctl, double e2_host, int R, const u64 *oidx,
                   const float *oval, const u64 *nout_dev, u64 nout_host) {
  using TL = LzTile<TZ, TY>;
  constexpr int PX = TL::PX, PZS = TL::PY * TL::PX;
  extern __shared__ __align__(16) unsigned char lz_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ti = (int64_t)blockIdx.x * LZ_NW + warp;
  if (ti >= count) return;
  int64_t t[3];
  if (!wave_tile(G, w, ti, t)) return;
  unsigned char *base = lz_smem + (size_t)warp * TL::BYTES;
  float *b = reinterpret_cast<float *>(base);
  float *orig = b + TL::NB;
  uint16_t *cs = reinterpret_cast<uint16_t *>(orig + TL::NO);
  const int64_t o0 = t[0] * TZ, o1 = t[1] * TY, o2 = t[2] * LZ_TX;
  const int64_t sz = G.ext[1] * G.ext[2], sy = G.ext[2];
  const int e0 = (int)min((int64_t)TZ, G.ext[0] - o0), e1 = (int)min((int64_t)TY, G.ext[1] - o1);
  const int e2x = (int)min((int64_t)LZ_TX, G.ext[2] - o2);
  double e2, inv = 0.0, eb = 0.0;
  if (MODE == 0) {
    eb = ctl->level_eb[0];
    e2 = dmul(2.0, eb);
    inv = ctl->inv_e2[0];
  } else {
    e2 = e2_host;
  }
  // halo: the plane z = -1, rows y = -1 and the column x = -1 (global
  // reconstruction of earlier wavefronts; 0 outside the grid)
  for (int i = lane; i < TL::NB; i += 32) {
    const int lz = i / PZS, r = i - lz * PZS, ly = r / PX, lx = r - ly * PX;
    if (lz > 0 && ly > 0 && lx > 0) continue;
    const int64_t gz = o0 + lz - 1, gy = o1 + ly - 1, gx = o2 + lx - 1;
    float v = 0.f;
    if (gz >= 0 && gy >= 0 && gx >= 0 && gz < G.ext[0] && gy < G.ext[1] && gx < G.ext[2])
      v = rec[gz * sz + gy * sy + gx];
    b[i] = v;
  }
  // the tile's inputs, row by row (coalesced)
  for (int r = 0; r < TZ * TY; ++r) {
    const int lz = r / TY, ly = r - lz * TY;
    if (lz >= e0 || ly >= e1 || lane >= e2x) continue;
    const int64_t g = (o0 + lz) * sz + (o1 + ly) * sy + o2 + lane;
    if (MODE == 0) orig[r * LZ_TX + lane] = x[g];
    else cs[r * LZ_TX + lane] = sym[g];
  }
  const u64 nout = MODE == 1 ? (nout_dev ? *nout_dev : nout_host) : 0;
  __syncwarp();
  // skewed sweep: lane l handles row r = k - l
  for (int k = 0; k < TZ * TY + 31; ++k) {
    const int r = k - lane;
    if (r >= 0 && r < TZ * TY) {
      const int lz = r / TY, ly = r - lz * TY;
      if (lz < e0 && ly < e1 && lane < e2x) {
        const int i = (lz + 1) * PZS + (ly + 1) * PX + lane + 1;
        const double pred = lz_pred(b, i, PX, PZS);
        float v;
        if (MODE == 0) {
          const uint32_t s = quantize<false>(pred, orig[r * LZ_TX + lane], eb, e2, inv, R, v);
          cs[r * LZ_TX + lane] = (uint16_t)s;
        } else {
          const uint32_t s = cs[r * LZ_TX + lane];
          if (s == 0xFFFFu) {
            const u64 flat = (u64)((o0 + lz) * sz + (o1 + ly) * sy + o2 + lane);
            v = outlier_value(oidx, oval, nout, flat);
          } else {
            const int q = (int)s - R;
            v = __double2float_rn(dadd(pred, dmul(e2, (double)q)));
          }
        }
        b[i] = v;
      }
    }
    __syncwarp();
  }
  // results out (coalesced rows)
  for (int r = 0; r < TZ * TY; ++r) {
    const int lz = r / TY, ly = r - lz * TY;
    if (lz >= e0 || ly >= e1 || lane >= e2x) continue;
    const int64_t g = (o0 + lz) * sz + (o1 + ly) * sy + o2 + lane;
    rec[g] = b[(lz + 1) * PZS + (ly + 1) * PX + lane + 1];
    if (MODE == 0) sym[g] = cs[r * LZ_TX + lane];
  }
}

// Rank 1: one sequential chain (lorenzo_1d, _kernels.py:113-141).
template <int MODE>
__global__ void k_lorenzo_1d(const float *__restrict__ x, float *rec, uint16_t *sym, int64_t n,
                             const cszi_ctl *ctl, double e2_host, int R, const u64 *oidx,
                             const float *oval, const u64 *nout_dev, u64 nout_host) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  double e2, inv = 0.0, eb = 0.0;
  if (MODE == 0) {
    eb = ctl->level_eb[0];
    e2 = dmul(2.0, eb);
    inv = ctl->inv_e2[0];
  } else {
    e2 = e2_host;
  }
  const u64 nout = MODE == 1 ? (nout_dev ? *nout_dev : nout_host) : 0;
  u64 next_out = 0;
  float prev = 0.f;
  for (int64_t i = 0; i < n; ++i) {
    const double pred = (i > 0) ? (double)prev : 0.0;
    float v;
    if (MODE == 0) {
      sym[i] = (uint16_t)quantize<false>(pred, x[i], eb, e2, inv, R, v);
    } else {
      const uint32_t s = sym[i];
      if (s == 0xFFFFu) {
        // outliers are strictly increasing: walk the list with the scan
        while (next_out < nout && oidx[next_out] < (u64)i) ++next_out;
        v = (next_out < nout) ? oval[next_out] : 0.f;
      } else {
        v = __double2float_rn(dadd(pred, dmul(e2, (double)((int)s - R))));
      }
    }
    rec[i] = v;
    prev = v;
  }
}

// eb_abs for the Lorenzo path (pipeline.py:123-128): rel -> eb * range when
// the range is positive, else eb; stored as level 0 with e2 and RN(1/e2).
__global__ void k_lorenzo_eb(cszi_ctl *ctl, double eb, int rel, int R) {
  if (ctl->first_nonfinite != ~0ull) ctl->flags |= CSZI_F_NONFINITE;
  double eab = eb;
  if (rel) {
    const double rng = dsub((double)key_float(ctl->vmax_key), (double)key_float(ctl->vmin_key));
    eab = rng > 0.0 ? dmul(eb, rng) : eb;
  }
  ctl->eb_abs = eab;
  ctl->alpha = 1.0;
  ctl->nlev = 1;
  ctl->radius = R;
  ctl->level_eb[0] = eab;
  ctl->inv_e2[0] = ddiv(1.0, dmul(2.0, eab));
  for (int a = 0; a < 3; ++a) {
    ctl->variant[a] = 0;
    ctl->order[a] = a;
  }
}

// symbol histogram (u16 symbols; the outlier sentinel 0 counts as R,
// huffman.py:60-74 on codes holding 0 there)
__global__ void k_hist_sym(const uint16_t *__restrict__ sym, u64 n, int R, u64 *hist) {
  extern __shared__ unsigned int hs[];
  for (int i = threadIdx.x; i < 2 * R; i += blockDim.x) hs[i] = 0;
  __syncthreads();
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
       i += (u64)gridDim.x * blockDim.x) {
    const uint32_t s = sym[i];
    atomicAdd(&hs[s == 0 ? R : s], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * R; i += blockDim.x)
    if (hs[i]) atomicAdd(&hist[i], (u64)hs[i]);
}

static LzGeo lz_geo(const cszi_geom *g, int &tz, int &ty) {
  LzGeo G;
  for (int a = 0; a < 3; ++a) G.ext[a] = g->ext[a];
  if (g->rank == 3) {
    tz = 8;
    ty = 8;
  } else {
    tz = 1;
    ty = 32;
  }
  G.nt[0] = (G.ext[0] + tz - 1) / tz;
  G.nt[1] = (G.ext[1] + ty - 1) / ty;
  G.nt[2] = (G.ext[2] + LZ_TX - 1) / LZ_TX;
  return G;
}

template <int TZ, int TY, int MODE>
static int lz_waves(const float *x, float *rec, uint16_t *sym, const LzGeo &G,
                    const cszi_ctl *ctl, double e2, int R, const u64 *oidx, const float *oval,
                    const u64 *nout_dev, u64 nout_host, cudaStream_t st) {
  using TL = LzTile<TZ, TY>;
  const size_t smem = (size_t)LZ_NW * TL::BYTES;
  auto k = k_lorenzo_wave<TZ, TY, MODE>;
  ensure_smem((const void *)k, smem);
  const int64_t nw = G.nt[0] + G.nt[1] + G.nt[2] - 2;
  for (int64_t w = 0; w < nw; ++w) {
    int64_t count = 0;
    for (int64_t tz = 0; tz < G.nt[0] && tz <= w; ++tz) count += diag_count_h(w - tz, G.nt[1], G.nt[2]);
    if (!count) continue;
    const unsigned grid = (unsigned)((count + LZ_NW - 1) / LZ_NW);
    k<<<grid, LZ_NW * 32, smem, st>>>(x, rec, sym, G, w, count, ctl, e2, R, oidx, oval, nout_dev,
                                      nout_host);
    note_launch();
  }
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

// mode 0: x -> sym (+ rec scratch); mode 1: sym -> rec
int launch_lorenzo(int mode, const float *x, float *rec, uint16_t *sym, const cszi_geom *g,
                   const cszi_ctl *ctl, double e2, int R, const u64 *oidx, const float *oval,
                   const u64 *nout_dev, u64 nout_host, cudaStream_t st) {
  if (g->rank == 1) {
    const int64_t n = g->ext[0] * g->ext[1] * g->ext[2];
    if (mode == 0) k_lorenzo_1d<0><<<1, 32, 0, st>>>(x, rec, sym, n, ctl, e2, R, oidx, oval, nout_dev, nout_host);
    else k_lorenzo_1d<1><<<1, 32, 0, st>>>(x, rec, sym, n, ctl, e2, R, oidx, oval, nout_dev, nout_host);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
  }
  int tz, ty;
  const LzGeo G = lz_geo(g, tz, ty);
  if (g->rank == 3) {
    return mode == 0 ? lz_waves<8, 8, 0>(x, rec, sym, G, ctl, e2, R, oidx, oval, nout_dev, nout_host, st)
                     : lz_waves<8, 8, 1>(x, rec, sym, G, ctl, e2, R, oidx, oval, nout_dev, nout_host, st);
  }
  return mode == 0 ? lz_waves<1, 32, 0>(x, rec, sym, G, ctl, e2, R, oidx, oval, nout_dev, nout_host, st)
                   : lz_waves<1, 32, 1>(x, rec, sym, G, ctl, e2, R, oidx, oval, nout_dev, nout_host, st);
}

int launch_lorenzo_eb(cszi_ctl *ctl, double eb, int rel, int R, cudaStream_t st) {
  k_lorenzo_eb<<<1, 1, 0, st>>>(ctl, eb, rel, R);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

int launch_hist_sym(const uint16_t *sym, u64 n, int R, u64 *hist, cudaStream_t st) {
  cudaMemsetAsync(hist, 0, 8 * 2 * (size_t)R, st);
  const size_t smem = 4 * 2 * (size_t)R;
  ensure_smem((const void *)k_hist_sym, smem);
  u64 blocks = (n + 255) / 256;
  const u64 cap = (u64)sm_count() * 4;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  k_hist_sym<<<(unsigned)blocks, 256, smem, st>>>(sym, n, R, hist);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

}  // namespace cszi
