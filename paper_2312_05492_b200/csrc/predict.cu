// G-Interp predictor + synchronized quantizer (compress) and the inverse
// interpolation (decompress) for sm_100a.
//
// Reference semantics: predictor.py:283-344 (_run_pass), :367-392
// (interpolate_level), :395-465 (compress_predict / decompress_predict).
//
// Design: neighbour reads are confined to a
// super-chunk tile plus one closing plane per axis, so any tile-aligned
// block plus its closing planes reproduces the global result.  One CTA owns
// a BZ x BY x BX block, stages the closed block (+1 plane per axis) in shared
// memory, and runs every (level, dimension) pass in place with a
// __syncthreads() between passes.  Closing-plane points are recomputed
// redundantly (bit-identical to their owner).  Anchors are skipped (the
// reference predicts them transiently and restores them after each pass).
//
// Arithmetic is float64 with explicit round-to-nearest intrinsics (no FMA
// contraction) in the reference's expression order.  The division
// t = r / e2 runs as r * (1/e2) with an exact-division fallback whenever the
// rounded quotient could land on the other side of a half-integer (see
// quantize()).  Zero-weight spline terms are dropped: they can only change
// the sign of a zero prediction, which never reaches q, rec or the guard
// because the reconstruction always adds e2*q with q == +0.0.
#include "common.cuh"

namespace cszi {

struct InterpParams {
  int64_t ext[3];
  int64_t tile[3];
  int64_t stride;
  int32_t rank;
  int32_t radius;
  int32_t nb[3];  // blocks per axis
};

// ---------------------------------------------------------------------------
// per-point arithmetic
// ---------------------------------------------------------------------------
constexpr double NAK_O = -1.0 / 16.0, NAK_I = 9.0 / 16.0;
constexpr double NAT_O = -3.0 / 40.0, NAT_I = 23.0 / 40.0;
constexpr double QO = -1.0 / 8.0, QN = 6.0 / 8.0, QF = 3.0 / 8.0;
constexpr double MAGIC = 6755399441055744.0;  // 1.5 * 2^52

// predictor.py:297-306 case table; returns the prediction in float64.
// vm3, vm1, vp1, vp3: neighbours at -3s, -s, +s, +3s (only read if used).
DEV double spline(int cs, int variant, const float *p, int step) {
  // cs: 0 cubic, 1 quad-left, 2 quad-right, 3 linear, 4 copy
  const double v1 = f2d(p[-step]);
  if (cs == 4) return v1;
  const double v2 = f2d(p[step]);
  if (cs == 3) return dadd(dmul(0.5, v1), dmul(0.5, v2));
  if (cs == 1) {
    const double v0 = f2d(p[-3 * step]);
    return dadd(dadd(dmul(QO, v0), dmul(QN, v1)), dmul(QF, v2));
  }
  const double v3 = f2d(p[3 * step]);
  if (cs == 2) return dadd(dadd(dmul(QF, v1), dmul(QN, v2)), dmul(QO, v3));
  const double v0 = f2d(p[-3 * step]);
  const double wo = variant ? NAT_O : NAK_O;
  const double wi = variant ? NAT_I : NAK_I;
  return dadd(dadd(dadd(dmul(wo, v0), dmul(wi, v1)), dmul(wi, v2)), dmul(wo, v3));
}

DEV int spline_case(int64_t pd, int64_t s, int64_t tile, int64_t extent) {
  const int64_t offset = pd & (tile - 1);
  const bool m3 = offset >= 3 * s;
  const bool p1 = pd + s <= extent - 1;
  const bool p3 = (offset <= tile - 3 * s) && (pd + 3 * s <= extent - 1);
  if (!p1) return 4;
  if (m3) return p3 ? 0 : 1;
  return p3 ? 2 : 3;
}

// predictor.py:327-339.  Returns the symbol (q + R, or 0 for an outlier)
// and the value stored in the reconstruction buffer.
template <bool EXACT>
DEV uint32_t quantize(double pred, float o32, double leb, double e2, double inv, int R,
                      float &recon) {
  const double o = f2d(o32);
  const double r = dsub(o, pred);
  int q = 0;
  double qd = 0.0;
  bool big = false, fast = false;
  if (!EXACT) {
    // t' = r * RN(1/e2) is within 3 ulp of RN(r/e2).  Away from a
    // half-integer, rint(t') == trunc(t + copysign(.5, t)) exactly.
    const double t = dmul(r, inv);
    if (fabs(t) < 1073741824.0) {
      const double m = dadd(t, MAGIC);
      const double rq = dsub(m, MAGIC);
      if (fabs(dsub(t, rq)) <= 0.49999904632568359375) {
        fast = true;
        q = __double2loint(m);
        big = (q >= R) || (q <= -R);
        qd = big ? 0.0 : rq;
      }
    }
  }
  if (!fast) {
    const double t = ddiv(r, e2);
    const double qf = trunc(dadd(t, copysign(0.5, t)));
    big = fabs(qf) >= (double)R;
    q = big ? 0 : (int)qf;
    qd = (double)q;
  }
  const float rec = __double2float_rn(dadd(pred, dmul(e2, qd)));
  const bool bad = big || (fabs(dsub(f2d(rec), o)) > leb);
  recon = bad ? o32 : rec;
  return bad ? 0u : (uint32_t)(q + R);
}

DEV bool is_anchor(const InterpParams &P, int64_t g0, int64_t g1, int64_t g2) {
  const int64_t m = P.stride - 1;
  return ((g0 & m) == 0 || g0 == P.ext[0] - 1) && ((g1 & m) == 0 || g1 == P.ext[1] - 1) &&
         ((g2 & m) == 0 || g2 == P.ext[2] - 1);
}

// quotient for k < 2^22 via float reciprocal + one correction
DEV int fdiv(int k, int d, float rd) {
  int q = __float2int_rz(__int2float_rz(k) * rd);
  if (q * d > k) q--;
  else if ((q + 1) * d <= k) q++;
  return q;
}

struct PassShape {
  int lo[3], st[3], cnt[3];
  int total;
};

DEV PassShape pass_shape(int d, int s, const bool passed[3], const int L[3]) {
  PassShape ps;
  for (int a = 0; a < 3; ++a) {
    ps.lo[a] = (a == d) ? s : 0;
    ps.st[a] = (a == d || !passed[a]) ? 2 * s : s;
    ps.cnt[a] = (L[a] - 1 >= ps.lo[a]) ? (L[a] - 1 - ps.lo[a]) / ps.st[a] + 1 : 0;
  }
  ps.total = ps.cnt[0] * ps.cnt[1] * ps.cnt[2];
  return ps;
}

struct LevelCfg {
  double leb[CSZI_MAX_LEVELS];
  double inv[CSZI_MAX_LEVELS];
  int order[3];
  int variant[3];
  int nlev;
};

// ---------------------------------------------------------------------------
// compress: predict + quantize + histogram
// ---------------------------------------------------------------------------
template <int BZ, int BY, int BX, int NT, bool EXACT>
__global__ void __launch_bounds__(NT) k_predict(const float *__restrict__ x, InterpParams P,
                                                const cszi_ctl *__restrict__ ctl,
                                                uint16_t *__restrict__ sym,
                                                u64 *__restrict__ hist, int hist_in_smem) {
  constexpr int CZ = BZ == 1 ? 1 : BZ + 1, CY = BY == 1 ? 1 : BY + 1, CX = BX + 1;
  constexpr int PX = CX, PY = CY;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float *buf = reinterpret_cast<float *>(smem_raw);
  uint16_t *codes = reinterpret_cast<uint16_t *>(buf + CZ * CY * CX);
  uint32_t *hs = reinterpret_cast<uint32_t *>(codes + ((BZ * BY * BX + 1) & ~1));
  __shared__ LevelCfg cfg;
  __shared__ uint32_t zero_ws[NT / 32];

  const int R = P.radius;
  const int nbins = 2 * R;
  const int tid = threadIdx.x;
  int b = blockIdx.x;
  const int bx = b % P.nb[2];
  b /= P.nb[2];
  const int by = b % P.nb[1];
  const int bz = b / P.nb[1];
  const int64_t o0 = (int64_t)bz * BZ, o1 = (int64_t)by * BY, o2 = (int64_t)bx * BX;
  int L[3];
  L[0] = (int)min((int64_t)CZ, P.ext[0] - o0);
  L[1] = (int)min((int64_t)CY, P.ext[1] - o1);
  L[2] = (int)min((int64_t)CX, P.ext[2] - o2);
  const int O0 = min(BZ, L[0]), O1 = min(BY, L[1]), O2 = min(BX, L[2]);

  if (tid == 0) {
    cfg.nlev = ctl->nlev;
    for (int a = 0; a < 3; ++a) {
      cfg.order[a] = ctl->order[a];
      cfg.variant[a] = ctl->variant[a];
    }
  }
  if (tid < CSZI_MAX_LEVELS) {
    cfg.leb[tid] = ctl->level_eb[tid];
    cfg.inv[tid] = ctl->inv_e2[tid];
  }
  if (hist_in_smem)
    for (int i = tid; i < nbins; i += NT) hs[i] = 0;
  // stage the closed block
  const int warp = tid >> 5, lane = tid & 31;
  for (int row = warp; row < L[0] * L[1]; row += NT / 32) {
    const int lz = row / L[1], ly = row - lz * L[1];
    const float *src = x + ((o0 + lz) * P.ext[1] + (o1 + ly)) * P.ext[2] + o2;
    float *dst = buf + (lz * PY + ly) * PX;
    for (int lx = lane; lx < L[2]; lx += 32) dst[lx] = __ldg(src + lx);
  }
  for (int i = tid; i < BZ * BY * BX; i += NT) codes[i] = (uint16_t)R;
  __syncthreads();

  const int rank = P.rank;
  const int S = (int)P.stride;
  for (int lv = 0; lv < cfg.nlev; ++lv) {
    const int s = S >> (lv + 1);
    const double leb = cfg.leb[lv];
    const double e2 = dmul(2.0, leb);
    const double inv = cfg.inv[lv];
    bool passed[3] = {false, false, false};
    for (int oi = 0; oi < rank; ++oi) {
      const int d = cfg.order[oi];
      if (s < P.ext[d]) {
        const PassShape ps = pass_shape(d, s, passed, L);
        const int pitch = (d == 0) ? PY * PX : (d == 1 ? PX : 1);
        const int step = s * pitch;
        const int variant = cfg.variant[d];
        const float r2 = 1.0f / (float)max(ps.cnt[2], 1), r1 = 1.0f / (float)max(ps.cnt[1], 1);
        for (int k = tid; k < ps.total; k += NT) {
          const int t = fdiv(k, ps.cnt[2], r2);
          const int i2 = k - t * ps.cnt[2];
          const int i0 = fdiv(t, ps.cnt[1], r1);
          const int i1 = t - i0 * ps.cnt[1];
          const int l0 = ps.lo[0] + i0 * ps.st[0];
          const int l1 = ps.lo[1] + i1 * ps.st[1];
          const int l2 = ps.lo[2] + i2 * ps.st[2];
          const int64_t g0 = o0 + l0, g1 = o1 + l1, g2 = o2 + l2;
          if (is_anchor(P, g0, g1, g2)) continue;
          const int64_t pd = (d == 0) ? g0 : (d == 1 ? g1 : g2);
          const int cs = spline_case(pd, s, P.tile[d], P.ext[d]);
          float *p = buf + (l0 * PY + l1) * PX + l2;
          const double pred = spline(cs, variant, p, step);
          float rec;
          const uint32_t sy = quantize<EXACT>(pred, *p, leb, e2, inv, R, rec);
          *p = rec;
          if (l0 < BZ && l1 < BY && l2 < BX) codes[(l0 * BY + l1) * BX + l2] = (uint16_t)sy;
        }
      }
      passed[d] = true;
      __syncthreads();
    }
  }

  // codes out (coalesced rows) + histogram; outliers (symbol 0) count as R
  uint32_t zeros = 0;
  for (int row = warp; row < O0 * O1; row += NT / 32) {
    const int lz = row / O1, ly = row - lz * O1;
    uint16_t *dst = sym + ((o0 + lz) * P.ext[1] + (o1 + ly)) * P.ext[2] + o2;
    const uint16_t *srow = codes + (lz * BY + ly) * BX;
    for (int lx = lane; lx < O2; lx += 32) {
      const uint32_t sy = srow[lx];
      dst[lx] = (uint16_t)sy;
      if (sy == (uint32_t)R || sy == 0) {
        zeros++;
      } else if (hist_in_smem) {
        atomicAdd(&hs[sy], 1u);
      } else {
        atomicAdd(&hist[sy], 1ull);
      }
    }
  }
  zeros = warp_sum(zeros);
  if (lane == 0) zero_ws[warp] = zeros;
  __syncthreads();
  if (tid == 0) {
    uint32_t z = 0;
    for (int w = 0; w < NT / 32; ++w) z += zero_ws[w];
    if (z) atomicAdd(&hist[R], (u64)z);
  }
  if (hist_in_smem) {
    for (int i = tid; i < nbins; i += NT)
      if (hs[i]) atomicAdd(&hist[i], (u64)hs[i]);
  }
}

// ---------------------------------------------------------------------------
// decompress: inverse interpolation from symbols
// ---------------------------------------------------------------------------
// Outlier values: symbols hold 0xFFFF at outlier points; the value is found
// by binary search in the (strictly increasing) outlier index list.
DEV float outlier_value(const u64 *idx, const float *val, u64 k, u64 target) {
  u64 lo = 0, hi = k;
  while (lo < hi) {
    const u64 mid = (lo + hi) >> 1;
    if (idx[mid] < target) lo = mid + 1;
    else hi = mid;
  }
  return val[lo];
}

DEV int64_t anchor_index_axis(int64_t c, int64_t S, int64_t ext) {
  // position of coordinate c in predictor.py:230-235's closed axis
  return ((c & (S - 1)) == 0) ? (c / S) : ((ext - 1) / S + 1);
}

template <int BZ, int BY, int BX, int NT>
__global__ void __launch_bounds__(NT) k_reconstruct(
    const uint16_t *__restrict__ sym, const float *__restrict__ anchors, const u64 *out_idx,
    const float *out_val, u64 n_out, const u64 *nout_dev, InterpParams P, LevelCfg lc,
    float *__restrict__ y) {
  constexpr int CZ = BZ == 1 ? 1 : BZ + 1, CY = BY == 1 ? 1 : BY + 1, CX = BX + 1;
  constexpr int PX = CX, PY = CY;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float *buf = reinterpret_cast<float *>(smem_raw);
  uint16_t *cs_ = reinterpret_cast<uint16_t *>(buf + CZ * CY * CX);

  const int R = P.radius;
  const int tid = threadIdx.x;
  if (nout_dev) n_out = *nout_dev;
  int b = blockIdx.x;
  const int bx = b % P.nb[2];
  b /= P.nb[2];
  const int by = b % P.nb[1];
  const int bz = b / P.nb[1];
  const int64_t o0 = (int64_t)bz * BZ, o1 = (int64_t)by * BY, o2 = (int64_t)bx * BX;
  int L[3];
  L[0] = (int)min((int64_t)CZ, P.ext[0] - o0);
  L[1] = (int)min((int64_t)CY, P.ext[1] - o1);
  L[2] = (int)min((int64_t)CX, P.ext[2] - o2);
  const int O0 = min(BZ, L[0]), O1 = min(BY, L[1]), O2 = min(BX, L[2]);
  const int64_t S = P.stride;
  const int64_t na1 = (P.ext[1] - 1) / S + 1 + (((P.ext[1] - 1) & (S - 1)) ? 1 : 0);
  const int64_t na2 = (P.ext[2] - 1) / S + 1 + (((P.ext[2] - 1) & (S - 1)) ? 1 : 0);

  const int warp = tid >> 5, lane = tid & 31;
  for (int row = warp; row < L[0] * L[1]; row += NT / 32) {
    const int lz = row / L[1], ly = row - lz * L[1];
    const int64_t g0 = o0 + lz, g1 = o1 + ly;
    const uint16_t *src = sym + (g0 * P.ext[1] + g1) * P.ext[2] + o2;
    uint16_t *dst = cs_ + (lz * PY + ly) * PX;
    float *bd = buf + (lz * PY + ly) * PX;
    const bool a01 = ((g0 & (S - 1)) == 0 || g0 == P.ext[0] - 1) &&
                     ((g1 & (S - 1)) == 0 || g1 == P.ext[1] - 1);
    for (int lx = lane; lx < L[2]; lx += 32) {
      dst[lx] = src[lx];
      const int64_t g2 = o2 + lx;
      if (a01 && ((g2 & (S - 1)) == 0 || g2 == P.ext[2] - 1)) {
        const int64_t ai = (anchor_index_axis(g0, S, P.ext[0]) * na1 +
                            anchor_index_axis(g1, S, P.ext[1])) * na2 +
                           anchor_index_axis(g2, S, P.ext[2]);
        bd[lx] = anchors[ai];
      }
    }
  }
  __syncthreads();

  const int rank = P.rank;
  for (int lv = 0; lv < lc.nlev; ++lv) {
    const int s = (int)(S >> (lv + 1));
    const double e2 = dmul(2.0, lc.leb[lv]);
    bool passed[3] = {false, false, false};
    for (int oi = 0; oi < rank; ++oi) {
      const int d = lc.order[oi];
      if (s < P.ext[d]) {
        const PassShape ps = pass_shape(d, s, passed, L);
        const int pitch = (d == 0) ? PY * PX : (d == 1 ? PX : 1);
        const int step = s * pitch;
        const int variant = lc.variant[d];
        const float r2 = 1.0f / (float)max(ps.cnt[2], 1), r1 = 1.0f / (float)max(ps.cnt[1], 1);
        for (int k = tid; k < ps.total; k += NT) {
          const int t = fdiv(k, ps.cnt[2], r2);
          const int i2 = k - t * ps.cnt[2];
          const int i0 = fdiv(t, ps.cnt[1], r1);
          const int i1 = t - i0 * ps.cnt[1];
          const int l0 = ps.lo[0] + i0 * ps.st[0];
          const int l1 = ps.lo[1] + i1 * ps.st[1];
          const int l2 = ps.lo[2] + i2 * ps.st[2];
          const int64_t g0 = o0 + l0, g1 = o1 + l1, g2 = o2 + l2;
          if (is_anchor(P, g0, g1, g2)) continue;
          const int64_t pd = (d == 0) ? g0 : (d == 1 ? g1 : g2);
          const int csx = spline_case(pd, s, P.tile[d], P.ext[d]);
          const int li = (l0 * PY + l1) * PX + l2;
          float *p = buf + li;
          const uint32_t code = cs_[li];
          float v;
          if (code == 0xFFFFu) {
            v = outlier_value(out_idx, out_val, n_out, (u64)((g0 * P.ext[1] + g1) * P.ext[2] + g2));
          } else {
            const double pred = spline(csx, variant, p, step);
            // predictor.py:341-342: rec = f32(pred + e2 * float64(q))
            const int q = (int)code - R;
            const double qd =
                dsub(__hiloint2double(0x43300000, (int)((uint32_t)q ^ 0x80000000u)),
                     4503601774854144.0);  // 2^52 + 2^31
            v = __double2float_rn(dadd(pred, dmul(e2, qd)));
          }
          *p = v;
        }
      }
      passed[d] = true;
      __syncthreads();
    }
  }
  for (int row = warp; row < O0 * O1; row += NT / 32) {
    const int lz = row / O1, ly = row - lz * O1;
    float *dst = y + ((o0 + lz) * P.ext[1] + (o1 + ly)) * P.ext[2] + o2;
    const float *srow = buf + (lz * PY + ly) * PX;
    for (int lx = lane; lx < O2; lx += 32) dst[lx] = srow[lx];
  }
}

// ---------------------------------------------------------------------------
// anchors: gather_anchors (predictor.py:250-256) / lattice row-major order
// ---------------------------------------------------------------------------
__global__ void k_gather_anchors(const float *__restrict__ x, InterpParams P, int64_t na0,
                                 int64_t na1, int64_t na2, float *__restrict__ out) {
  const int64_t total = na0 * na1 * na2;
  const int64_t S = P.stride;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i2 = i % na2, t = i / na2, i1 = t % na1, i0 = t / na1;
    const int64_t c0 = min(i0 * S, P.ext[0] - 1), c1 = min(i1 * S, P.ext[1] - 1),
                  c2 = min(i2 * S, P.ext[2] - 1);
    out[i] = x[(c0 * P.ext[1] + c1) * P.ext[2] + c2];
  }
}

// ---------------------------------------------------------------------------
// host-side launchers
// ---------------------------------------------------------------------------
template <int BZ, int BY, int BX>
static size_t predict_smem(int radius, bool hist_smem) {
  constexpr int CZ = BZ == 1 ? 1 : BZ + 1, CY = BY == 1 ? 1 : BY + 1, CX = BX + 1;
  size_t s = sizeof(float) * CZ * CY * CX + sizeof(uint16_t) * ((BZ * BY * BX + 1) & ~1);
  if (hist_smem) s += sizeof(uint32_t) * 2 * (size_t)radius;
  return s;
}
template <int BZ, int BY, int BX>
static size_t recon_smem() {
  constexpr int CZ = BZ == 1 ? 1 : BZ + 1, CY = BY == 1 ? 1 : BY + 1, CX = BX + 1;
  return (sizeof(float) + sizeof(uint16_t)) * CZ * CY * CX + 16;
}

static bool fill_params(const cszi_geom *g, int32_t radius, int bz, int by, int bx,
                        InterpParams &P) {
  for (int a = 0; a < 3; ++a) {
    P.ext[a] = g->ext[a];
    P.tile[a] = g->tile[a];
  }
  P.stride = g->stride;
  P.rank = g->rank;
  P.radius = radius;
  const int B[3] = {bz, by, bx};
  for (int a = 0; a < 3; ++a) {
    if (B[a] == 1) {
      if (g->ext[a] != 1) return false;
    } else if (B[a] % g->tile[a] != 0 || g->tile[a] % g->stride != 0) {
      return false;
    }
    if (g->tile[a] & (g->tile[a] - 1)) return false;
    P.nb[a] = (int)((g->ext[a] + B[a] - 1) / B[a]);
  }
  return true;
}

#define CSZI_NT 256

template <int BZ, int BY, int BX>
static int launch_predict_t(const float *x, const cszi_geom *g, int32_t radius,
                            const cszi_ctl *ctl, uint16_t *sym, u64 *hist, bool exact,
                            cudaStream_t st) {
  InterpParams P;
  if (!fill_params(g, radius, BZ, BY, BX, P)) return CSZI_E_UNSUPPORTED;
  const bool hsm = 2 * radius <= 8192;
  const size_t smem = predict_smem<BZ, BY, BX>(radius, hsm);
  const int64_t nblk = (int64_t)P.nb[0] * P.nb[1] * P.nb[2];
  if (nblk > 0x7fffffffLL) return CSZI_E_UNSUPPORTED;
  if (exact) {
    auto k = k_predict<BZ, BY, BX, CSZI_NT, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<(unsigned)nblk, CSZI_NT, smem, st>>>(x, P, ctl, sym, hist, hsm ? 1 : 0);
    note_launch();
  } else {
    auto k = k_predict<BZ, BY, BX, CSZI_NT, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<(unsigned)nblk, CSZI_NT, smem, st>>>(x, P, ctl, sym, hist, hsm ? 1 : 0);
    note_launch();
  }
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

template <int BZ, int BY, int BX>
static int launch_recon_t(const uint16_t *sym, const float *anchors, const u64 *oidx,
                          const float *oval, u64 nout, const u64 *nout_dev,
                          const cszi_geom *g, int32_t radius,
                          const LevelCfg &lc, float *y, cudaStream_t st) {
  InterpParams P;
  if (!fill_params(g, radius, BZ, BY, BX, P)) return CSZI_E_UNSUPPORTED;
  const size_t smem = recon_smem<BZ, BY, BX>();
  const int64_t nblk = (int64_t)P.nb[0] * P.nb[1] * P.nb[2];
  if (nblk > 0x7fffffffLL) return CSZI_E_UNSUPPORTED;
  auto k = k_reconstruct<BZ, BY, BX, CSZI_NT>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<(unsigned)nblk, CSZI_NT, smem, st>>>(sym, anchors, oidx, oval, nout, nout_dev, P, lc, y);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

// Block shapes per layout: 3-D default (8,8,32) tiles -> 8x16x32 blocks;
// 2-D (16,16) tiles -> 1x32x64; 1-D 512 tile -> 1x1x1024.  Non-default
// strides (decode of archives with anchor_stride != default) use the shape
// whose extents are multiples of (stride,)*rank when one exists.
int launch_predict(const float *x, const cszi_geom *g, int32_t radius, const cszi_ctl *ctl,
                   uint16_t *sym, u64 *hist, bool exact, cudaStream_t st) {
  if (g->rank == 3) return launch_predict_t<8, 16, 32>(x, g, radius, ctl, sym, hist, exact, st);
  if (g->rank == 2) return launch_predict_t<1, 32, 64>(x, g, radius, ctl, sym, hist, exact, st);
  return launch_predict_t<1, 1, 1024>(x, g, radius, ctl, sym, hist, exact, st);
}

int launch_reconstruct(const uint16_t *sym, const float *anchors, const u64 *oidx,
                       const float *oval, u64 nout, const u64 *nout_dev, const cszi_geom *g,
                       int32_t radius,
                       const double *leb, int nlev, const int32_t variant[3],
                       const int32_t order[3], float *y, cudaStream_t st) {
  LevelCfg lc;
  lc.nlev = nlev;
  for (int i = 0; i < CSZI_MAX_LEVELS; ++i) {
    lc.leb[i] = i < nlev ? leb[i] : 0.0;
    lc.inv[i] = 0.0;
  }
  for (int a = 0; a < 3; ++a) {
    lc.order[a] = order[a];
    lc.variant[a] = variant[a];
  }
  int rc = CSZI_E_UNSUPPORTED;
  if (g->rank == 3) {
    rc = launch_recon_t<8, 16, 32>(sym, anchors, oidx, oval, nout, nout_dev, g, radius, lc, y, st);
    if (rc == CSZI_E_UNSUPPORTED)
      rc = launch_recon_t<16, 16, 32>(sym, anchors, oidx, oval, nout, nout_dev, g, radius, lc, y, st);
  } else if (g->rank == 2) {
    rc = launch_recon_t<1, 32, 64>(sym, anchors, oidx, oval, nout, nout_dev, g, radius, lc, y, st);
  } else {
    rc = launch_recon_t<1, 1, 1024>(sym, anchors, oidx, oval, nout, nout_dev, g, radius, lc, y, st);
  }
  return rc;
}

int launch_gather_anchors(const float *x, const cszi_geom *g, float *out, cudaStream_t st) {
  InterpParams P;
  for (int a = 0; a < 3; ++a) {
    P.ext[a] = g->ext[a];
    P.tile[a] = g->tile[a];
  }
  P.stride = g->stride;
  int64_t na[3];
  for (int a = 0; a < 3; ++a) {
    const int64_t e = g->ext[a], S = g->stride;
    na[a] = (e - 1) / S + 1 + (((e - 1) % S) ? 1 : 0);
  }
  const int64_t total = na[0] * na[1] * na[2];
  const int threads = 256;
  int64_t blocks = (total + threads - 1) / threads;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  k_gather_anchors<<<(unsigned)blocks, threads, 0, st>>>(x, P, na[0], na[1], na[2], out);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

}  // namespace cszi
