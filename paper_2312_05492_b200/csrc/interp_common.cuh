// Per-point G-Interp arithmetic shared by the generic / rank-1-2 kernels
// (predict.cu) and the 3-D tile kernels (t3.cu): spline weights, the
// reference quantiser, outlier lookup, spline cases (predictor.py:59-69,
// 187-223, 293-339).
#pragma once

#include "common.cuh"

namespace cszi {

// ---------------------------------------------------------------------------
// per-point arithmetic
// ---------------------------------------------------------------------------
constexpr double NAK_O = -1.0 / 16.0, NAK_I = 9.0 / 16.0;
constexpr double NAT_O = -3.0 / 40.0, NAT_I = 23.0 / 40.0;
constexpr double QO = -1.0 / 8.0, QN = 6.0 / 8.0, QF = 3.0 / 8.0;
constexpr double MAGIC = 6755399441055744.0;  // 1.5 * 2^52

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

// Outlier values (decompress): symbols hold 0xFFFF at outlier points; the
// value is found by binary search in the strictly increasing index list.
DEV float outlier_value(const u64 *idx, const float *val, u64 k, u64 target) {
  u64 lo = 0, hi = k;
  while (lo < hi) {
    const u64 mid = (lo + hi) >> 1;
    if (idx[mid] < target) lo = mid + 1;
    else hi = mid;
  }
  return val[lo];
}

// quotient for 0 <= k < 2^22 via float reciprocal + one correction
DEV int fdiv(int k, int d, float rd) {
  int q = __float2int_rz(__int2float_rz(k) * rd);
  if (q * d > k) q--;
  else if ((q + 1) * d <= k) q++;
  return q;
}

struct LevelCfg {
  double leb[CSZI_MAX_LEVELS];
  double inv[CSZI_MAX_LEVELS];
  int order[3];
  int variant[3];
  int nlev;
};

// spline case of the point at global coordinate pd (predictor.py:297-306)
DEV int case_of(int pd, int s, int tile, int ext_d) {
  const int offset = pd & (tile - 1);
  const bool m3 = offset >= 3 * s;
  const bool p1 = pd + s <= ext_d - 1;
  const bool p3 = (offset <= tile - 3 * s) && (pd + 3 * s <= ext_d - 1);
  if (!p1) return 4;
  if (m3) return p3 ? 0 : 1;
  return p3 ? 2 : 3;
}

// predictor.py:325 with zero-weight terms dropped (sign of zero only).
DEV double spline4(int cs, double wo, double wi, double vm3, double vm1, double vp1,
                   double vp3) {
  switch (cs) {
    case 0:
      return dadd(dadd(dadd(dmul(wo, vm3), dmul(wi, vm1)), dmul(wi, vp1)), dmul(wo, vp3));
    case 1:
      return dadd(dadd(dmul(QO, vm3), dmul(QN, vm1)), dmul(QF, vp1));
    case 2:
      return dadd(dadd(dmul(QF, vm1), dmul(QN, vp1)), dmul(QO, vp3));
    case 3:
      return dadd(dmul(0.5, vm1), dmul(0.5, vp1));
    default:
      return vm1;
  }
}

// anchor coordinate list of one axis inside a closed block of extent C
// (predictor.py:230-235: multiples of S, plus ext-1)
template <int C, int S>
DEV int anchor_axis_local(int e, int *out) {
  int n = 0;
  for (int l = 0; l < C && l < e; l += S) out[n++] = l;
  if (e - 1 < C && ((e - 1) % S) != 0) out[n++] = e - 1;
  return n;
}

}  // namespace cszi
