// Interior tiles of the 3-D tile engine (included by tile3.cuh inside
// namespace cszi::t3).
//
// An interior tile has its closing plane inside the grid on every axis, so
// every pass has a compile-time shape: (S, D, which other axes are already
// passed at this level) fixes the lattice steps, the item count and the
// spline case of every point (predictor.py:293-306 with offset = position
// inside the 8 x 8 x 32 tile).  Each pass is one instantiation of
// iwalk_x / iwalk_col; ipass() dispatches on the tuned order at run time
// (one uniform branch per pass), so the walks carry no runtime geometry,
// no divisions by runtime counts and no per-point case logic.
//
// Per point (compress) the fast path is
//   pred: the spline in the reference's operation order (predictor.py:325);
//         with the not-a-knot weights every w * v is exact, so the chain
//         folds into FMAs bit for bit;
//   q:    t' = r * RN(1/e2), rq = rint(t') by the magic-number round; the
//         point is decided only when t' is at least 2^-20 away from a
//         half-integer (then rq == trunc(t + copysign(.5, t)) of the
//         reference, predictor.py:330-331) and |rq| < R;
//   rec:  RN32(pred + RN(e2 rq)) exactly as the reference;
//   guard (predictor.py:336-337): |f64(rec) - o| > leb is decided in fp32:
//         d = RN32(rec - o32) has relative error <= 2^-24 (exact when
//         Sterbenz applies, and for subnormal results), so |d| <= a32 with
//         a32 = RD32(leb) * (1 - 2^-23) proves |rec - o| < leb and hence
//         RN64(f64(rec) - o) <= leb.
// A line with any undecided point (near half-integer, |q| >= R, guard not
// proven) is redone by fix_line() with the exact reference quantiser.  On
// decompress the outlier symbol (0xFFFF) takes the same route.

// not-a-knot cubic (predictor.py:62): ((w0 a + w1 b) + w2 c) + w3 d with
// every product exact
DEV double p_nak(double a, double b, double c, double d) {
  return __fma_rn(NAK_O, d, __fma_rn(NAK_I, c, __fma_rn(NAK_I, b, dmul(NAK_O, a))));
}

// prediction of point k of a line with NP points (case_interior pattern)
template <int NP, bool NAK>
DEV double ipred(int k, double wo, double wi, double a, double b, double c, double d) {
  if (NP == 1) return p_lin(b, c);
  if (k == 0) return p_p3(b, c, d);
  if (k == NP - 1) return p_m3(a, b, c);
  return NAK ? p_nak(a, b, c, d) : chain4(wo, wi, wi, wo, a, b, c, d);
}

// Exact-fit axes.  An edge tile whose extent along an axis is exactly the
// tile length (8 or 32: the grid ends on the tile boundary) has no closing
// plane on that axis; its lines are the interior lines with the last two
// points changed (case_of with ext = tile length): the last point has no
// right neighbour (copy, case 4), the one before it no vp3 (m3-only, or
// linear when it is also the first).  fit is warp-uniform; with k
// compile-time this is one select per changed point.
template <int NP, bool NAK>
DEV double ipred_f(int k, bool fit, double wo, double wi, double a, double b, double c,
                   double d) {
  const double p = ipred<NP, NAK>(k, wo, wi, a, b, c, d);
  if (k == NP - 1) return fit ? b : p;
  if (k == NP - 2) return fit ? (k == 0 ? p_lin(b, c) : p_m3(a, b, c)) : p;
  return p;
}

// anchor coordinate of a tile axis of length TL: multiples of 8, plus the
// closing anchor TL - 1 when the grid ends at the tile (predictor.py:230-235)
DEV bool anc(int c, bool fit, int TL) { return (c & 7) == 0 || (fit && c == TL - 1); }

// Fast quantiser (see the header); true when the point is decided.
DEV bool quant_i(double pred, float o32, const Lv &L, double Rd, int R, float &rec,
                 uint32_t &sym) {
  const double o = (double)o32;
  const double r = dsub(o, pred);
  const double t = dmul(r, L.inv);
  const double m = dadd(t, MAGIC);
  const double rq = dsub(m, MAGIC);
  const double y = dadd(pred, dmul(L.e2, rq));
  rec = __double2float_rn(y);
  sym = (uint32_t)(__double2loint(m) + R);
  const float d = __fsub_rn(rec, o32);
  return (fabs(dsub(t, rq)) <= 0.49999904632568359375) & (fabs(rq) < Rd) & (fabsf(d) <= L.a32);
}

// Exact redo of one line of an interior pass: np points at smem addresses
// a0 + 2 k stb (neighbours at +-stb, +-3 stb), spline case pattern of
// case_interior.  MODE 0: reference quantiser per point, stores rec and
// (own) the symbol at c0 + k cstb.  MODE 1: dequantise, outlier symbols
// (0xFFFF at y0 + k ystb) take their value from the outlier list (flat
// index f0 + k fst).
template <int MODE>
__device__ __noinline__ void fix_line(uint32_t a0, uint32_t stb, int np, uint32_t c0,
                                      uint32_t cstb, bool own, double wo, double wi, Lv L, int R,
                                      uint32_t y0, uint32_t ystb, u64 f0, int64_t fst, Out O) {
  for (int k = 0; k < np; ++k) {
    const uint32_t a = a0 + 2u * (uint32_t)k * stb;
    const int cs = (np == 1) ? 3 : (k == 0) ? 2 : (k == np - 1) ? 1 : 0;
    float v[4];
    v[1] = lds_f(a - stb);
    v[2] = lds_f(a + stb);
    v[0] = (cs <= 1) ? lds_f(a - 3 * stb) : 0.f;
    v[3] = (cs == 0 || cs == 2) ? lds_f(a + 3 * stb) : 0.f;
    const double pred = spline4(cs, wo, wi, (double)v[0], (double)v[1], (double)v[2], (double)v[3]);
    if (MODE == 0) {
      const QS q = quant_slow(pred, lds_f(a), L.leb, L.e2, L.inv, R);
      sts_f(a, q.rec);
      if (own) sts_u16(c0 + (uint32_t)k * cstb, q.sym);
    } else {
      const uint32_t sy = lds_u16(y0 + (uint32_t)k * ystb);
      sts_f(a, sy == 0xFFFFu ? outlier_at(O.idx, O.val, O.n, f0 + (u64)((int64_t)k * fst))
                             : dequant(pred, sy, L, R));
    }
  }
}

// fix_line_fit: the same with fl = own | fit (the line's axis ends at the
// tile: ipred_f's end cases) | keep (its last point is a closing anchor, left
// as staged / seeded, code R).  Two copies on purpose: the callers' register
// allocation depends on what the callee clobbers, and the interior walks
// keep theirs with the copy without the exact-fit cases (one shared copy
// measured 7% larger generic-walk kernels, up to 7% slower).
enum { FL_OWN = 1, FL_FIT = 2, FL_KEEP = 4 };
template <int MODE>
__device__ __noinline__ void fix_line_fit(uint32_t a0, uint32_t stb, int np, uint32_t c0,
                                          uint32_t cstb, int fl, double wo, double wi, Lv L,
                                          int R, uint32_t y0, uint32_t ystb, u64 f0, int64_t fst,
                                          Out O) {
  const bool own = fl & FL_OWN, fit = fl & FL_FIT, keep = fl & FL_KEEP;
  for (int k = 0; k < np; ++k) {
    const uint32_t a = a0 + 2u * (uint32_t)k * stb;
    int cs = (np == 1) ? 3 : (k == 0) ? 2 : (k == np - 1) ? 1 : 0;
    if (fit && k == np - 1) {
      if (keep) continue;
      cs = 4;
    } else if (fit && k == np - 2) {
      cs = (k == 0) ? 3 : 1;
    }
    float v[4];
    v[1] = lds_f(a - stb);
    v[2] = lds_f(a + stb);
    v[0] = (cs <= 1) ? lds_f(a - 3 * stb) : 0.f;
    v[3] = (cs == 0 || cs == 2) ? lds_f(a + 3 * stb) : 0.f;
    const double pred = spline4(cs, wo, wi, (double)v[0], (double)v[1], (double)v[2], (double)v[3]);
    if (MODE == 0) {
      const QS q = quant_slow(pred, lds_f(a), L.leb, L.e2, L.inv, R);
      sts_f(a, q.rec);
      if (own) sts_u16(c0 + (uint32_t)k * cstb, q.sym);
    } else {
      const uint32_t sy = lds_u16(y0 + (uint32_t)k * ystb);
      sts_f(a, sy == 0xFFFFu ? outlier_at(O.idx, O.val, O.n, f0 + (u64)((int64_t)k * fst))
                             : dequant(pred, sy, L, R));
    }
  }
}

// D = x: a lane walks one row (z, y) of the pass lattice; rows z in
// [0, 8] step STZ, y in [0, 8] step STY.
//
// Closing planes at level 1: a point on the closing plane of axis A (z = 8,
// y = 8 or x = 32) only ever feeds an A-pass, so once A has been passed at
// the finest level its closing plane is dead (compress: its codes belong to
// the next tile; decompress: it is not stored).  Level-1 passes after the
// A-pass skip it (the last pass of a tile runs 64 instead of 81 rows).
//
// FK = 1: an edge tile whose axes are each either closed (closing plane
// inside the grid) or exact-fit (fit bit a: the grid ends at the tile's end,
// no closing plane).  FK = 2: an interior tile redone with fix_line_fit (so
// that a kernel calls one redo copy).  FK = 0: an interior tile.  A fit axis holds rows 0..7 only; along x the line takes
// ipred_f's end cases, and on a closing-anchor row (z, y anchor coordinates)
// its last point (x = 31, S = 1) is an anchor: kept, code R.
template <int S, int STZ, int STY, int MODE, bool NAK, int FK = 0>
DEV void iwalk_x(const Tile &T, double wo, double wi, const Lv &L, int R, const Out &O,
                 int fit = 0) {
  constexpr int NZr = (S == 1 && STZ == 1) ? 8 : 8 / STZ + 1;
  constexpr int NYr = (S == 1 && STY == 1) ? 8 : 8 / STY + 1;
  constexpr int NP = 16 / S;
  // the last pass of a compress tile: its values are never read again
  constexpr bool LAST = MODE == 0 && S == 1 && STZ == 1 && STY == 1;
  const bool fz = FK == 1 && (fit & 1), fy = FK == 1 && (fit & 2), fx = FK == 1 && (fit & 4);
  const int nzr = fz ? 7 / STZ + 1 : NZr, nyr = fy ? 7 / STY + 1 : NYr;
  const int nl = nzr * nyr;
  const uint32_t my = (65536u + nyr - 1) / nyr;
  const int lane = threadIdx.x & 31;
  const double Rd = (double)R;
#pragma unroll 1
  for (int l = lane; l < nl; l += 32) {
    const int iz = FK == 1 ? (int)(((uint32_t)l * my) >> 16) : l / NYr;
    const int iy = l - iz * nyr;
    const int z = iz * STZ, y = iy * STY;
    const bool keep = FK == 1 && S == 1 && fx && anc(z, fz, 8) && anc(y, fy, 8);
    const uint32_t row = bufa(T, z, y, 0);
    double ev[NP + 1];
    float pt[NP];
    float4 Q[8];
    if (S <= 2) {
#pragma unroll
      for (int j = 0; j < 8; ++j) Q[j] = lds_f4(row + 16 * j);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (S == 1) {
          ev[2 * j] = (double)Q[j].x;
          ev[2 * j + 1] = (double)Q[j].z;
          pt[2 * j] = Q[j].y;
          pt[2 * j + 1] = Q[j].w;
        } else {
          ev[j] = (double)Q[j].x;
          pt[j] = Q[j].z;
        }
      }
      ev[NP] = (double)lds_f(row + 128);
    } else {
#pragma unroll
      for (int j = 0; j <= NP; ++j) ev[j] = (double)lds_f(row + 4 * 8 * j);
#pragma unroll
      for (int k = 0; k < NP; ++k) pt[k] = lds_f(row + 4 * (8 * k + 4));
    }
    uint32_t sy[NP];
    if (MODE == 1) {
      const uint32_t sr = syma(T, z, y, 0);
      if (S <= 2) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint4 w = lds_u4(sr + 16 * j);
          const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            if (S == 1) sy[4 * j + h] = ww[h] >> 16;
            else if (h & 1) sy[2 * j + (h >> 1)] = ww[h] & 0xffffu;
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < NP; ++k) sy[k] = lds_u16(sr + 2 * (8 * k + 4));
      }
    }
    float rec[NP];
    uint32_t code[NP];
    bool ok = true;
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const double pr = ipred_f<NP, NAK>(k, fx, wo, wi, k > 0 ? ev[k - 1] : 0.0, ev[k],
                                         ev[k + 1], k + 2 <= NP ? ev[k + 2] : 0.0);
      bool d;
      if (MODE == 0) {
        d = quant_i(pr, pt[k], L, Rd, R, rec[k], code[k]);
      } else {
        rec[k] = dequant(pr, sy[k], L, R);
        d = sy[k] != 0xFFFFu;
      }
      ok &= d | (keep && k == NP - 1);
    }
    if (keep) {
      rec[NP - 1] = pt[NP - 1];
      code[NP - 1] = (uint32_t)R;
    }
    const bool own = z < TZ && y < TY;
    if (!ok) {
      if constexpr (FK != 0)
        fix_line_fit<MODE>(row + 4 * S, 4 * S, NP, codea(T, z, y, S), 4 * S,
                           (own ? FL_OWN : 0) | (fx ? FL_FIT : 0) | (keep ? FL_KEEP : 0), wo, wi,
                           L, R, syma(T, z, y, S), 4 * S, flat_of(T, z, y, S), 2 * S, O);
      else
        fix_line<MODE>(row + 4 * S, 4 * S, NP, codea(T, z, y, S), 4 * S, own, wo, wi, L, R,
                       syma(T, z, y, S), 4 * S, flat_of(T, z, y, S), 2 * S, O);
      continue;
    }
    if (!LAST) {
      if (S <= 2) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (S == 1) {
            Q[j].y = rec[2 * j];
            Q[j].w = rec[2 * j + 1];
          } else {
            Q[j].z = rec[j];
          }
          sts_f4(row + 16 * j, Q[j]);
        }
      } else {
#pragma unroll
        for (int k = 0; k < NP; ++k) sts_f(row + 4 * (8 * k + 4), rec[k]);
      }
    }
    if (MODE == 0 && own) {
      const uint32_t cr = codea(T, z, y, 0);
#pragma unroll
      for (int k = 0; k < NP; ++k) sts_u16(cr + 2 * (2 * k + 1) * S, code[k]);
    }
  }
}

// D in {0 (z), 1 (y)}: lane owns the quad x in [4j, 4j + 4) at coordinate a
// of the other non-x axis A (step STA) and walks along D.  STX is the x
// lattice step: 1 -> four x-lines, 2 -> x = 4j, 4j + 2, 4 -> x = 4j,
// 8 -> x = 4j on even quads.  Quad 8 (x = 32..35) holds one real line.
// FK (see iwalk_x): a fit x axis holds quads 0..7, a fit A axis rows
// 0..7; along a fit D the lines take ipred_f's end cases, and at a closing
// anchor (a, x) the last point (D = 7, S = 1) is kept.
template <int S, int D, int STX, int STA, int MODE, bool NAK, int FK = 0>
DEV void iwalk_col(const Tile &T, double wo, double wi, const Lv &L, int R, const Out &O,
                   int fit = 0) {
  constexpr uint32_t PD4 = 4u * ((D == 0) ? PZ : PX);
  constexpr int NE = (STX == 1) ? 4 : (STX == 2) ? 2 : 1;  // x-lines per quad
  constexpr int QS_ = (STX == 8) ? 2 : 1;                   // quad step
  constexpr int NQ = (STX == 8) ? 5 : (S == 1 && STX == 1) ? 8 : 9;
  constexpr int NA = (S == 1 && STA == 1) ? 8 : 8 / STA + 1;
  constexpr int NP = 4 / S;
  constexpr int NV = NP + 1;
  // the last pass of a compress tile (x and the other axis already passed)
  constexpr bool LAST = MODE == 0 && S == 1 && STX == 1 && STA == 1;
  const bool fd = FK == 1 && ((fit >> D) & 1), fa = FK == 1 && ((fit >> (1 - D)) & 1);
  const bool fx = FK == 1 && (fit & 4);
  const int nq = fx ? (QS_ == 2 ? 4 : 8) : NQ, na = fa ? 7 / STA + 1 : NA;
  const int items = na * nq;
  const uint32_t mq = (65536u + nq - 1) / nq;
  const int lane = threadIdx.x & 31;
  const double Rd = (double)R;
#pragma unroll 1
  for (int it = lane; it < items; it += 32) {
    const int ia = FK == 1 ? (int)(((uint32_t)it * mq) >> 16) : it / NQ;
    const int jq = it - ia * nq;
    const int j = jq * QS_;
    const int a = ia * STA;
    // closing anchors on the last point, per x-line of the quad
    const bool kl = FK == 1 && S == 1 && fd && anc(a, fa, 8);
    bool keep[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) keep[e] = kl && anc(4 * j + e * STX, fx, 32);
    const uint32_t col = (D == 0) ? bufa(T, 0, a, 4 * j) : bufa(T, a, 0, 4 * j);
    double ev[NE][NV];
    float pt[NE][NP];
    float4 P4[NP];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const uint32_t ad = col + (uint32_t)(2 * v * S) * PD4;
      if (NE == 1) {
        ev[0][v] = (double)lds_f(ad);
      } else {
        const float4 q = lds_f4(ad);
        const float qq[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int e = 0; e < NE; ++e) ev[e][v] = (double)qq[e * STX];
      }
    }
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const uint32_t ad = col + (uint32_t)((2 * k + 1) * S) * PD4;
      if (NE == 1) {
        pt[0][k] = lds_f(ad);
      } else {
        P4[k] = lds_f4(ad);
        const float qq[4] = {P4[k].x, P4[k].y, P4[k].z, P4[k].w};
#pragma unroll
        for (int e = 0; e < NE; ++e) pt[e][k] = qq[e * STX];
      }
    }
    uint32_t sy[NE][NP];
    if (MODE == 1) {
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const int p = (2 * k + 1) * S;
        const uint32_t sa = (D == 0) ? syma(T, p, a, 4 * j) : syma(T, a, p, 4 * j);
        if (NE == 1) {
          sy[0][k] = lds_u16(sa);
        } else {
          const uint2 w = lds_u2(sa);
          const uint32_t h[4] = {w.x & 0xffffu, w.x >> 16, w.y & 0xffffu, w.y >> 16};
#pragma unroll
          for (int e = 0; e < NE; ++e) sy[e][k] = h[e * STX];
        }
      }
    }
    float rec[NE][NP];
    uint32_t code[NE][NP];
    bool ok = true;
#pragma unroll
    for (int k = 0; k < NP; ++k) {
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const double pr = ipred_f<NP, NAK>(k, fd, wo, wi, k > 0 ? ev[e][k - 1] : 0.0, ev[e][k],
                                           ev[e][k + 1], k + 2 <= NP ? ev[e][k + 2] : 0.0);
        // the pad lines of quad 8 (x = 33..35) compute on staged data that
        // is never read back: they cannot send the item to fix_line (nor
        // can a kept anchor)
        const bool pad = (e > 0 && STX < 4 && j == 8) || (keep[e] && k == NP - 1);
        if (MODE == 0) {
          ok &= quant_i(pr, pt[e][k], L, Rd, R, rec[e][k], code[e][k]) | pad;
        } else {
          rec[e][k] = dequant(pr, sy[e][k], L, R);
          ok &= (sy[e][k] != 0xFFFFu) | pad;
        }
      }
    }
#pragma unroll
    for (int e = 0; e < NE; ++e)
      if (keep[e]) {
        rec[e][NP - 1] = pt[e][NP - 1];
        code[e][NP - 1] = (uint32_t)R;
      }
    const bool own = a < 8 && j < 8;
    if (!ok) {
#pragma unroll 1
      for (int e = 0; e < NE; ++e) {
        const int x = 4 * j + e * STX;
        if (x > 32) continue;  // pad lines of quad 8 are never read
        const uint32_t c0 = (D == 0) ? codea(T, S, a, x) : codea(T, a, S, x);
        const uint32_t cst = 2u * 2 * S * ((D == 0) ? TY * CP : CP);
        const uint32_t y0 = (D == 0) ? syma(T, S, a, x) : syma(T, a, S, x);
        const uint32_t yst = 2u * 2 * S * ((D == 0) ? CY * SP : SP);
        const u64 f0 = (D == 0) ? flat_of(T, S, a, x) : flat_of(T, a, S, x);
        const int64_t fst = 2 * S * ((D == 0) ? T.gs0 : T.gs1);
        if constexpr (FK != 0)
          fix_line_fit<MODE>(col + (uint32_t)S * PD4 + 4u * e * STX, (uint32_t)S * PD4, NP, c0,
                             cst,
                             (own && x < TX ? FL_OWN : 0) | (fd ? FL_FIT : 0) |
                                 (keep[e] ? FL_KEEP : 0),
                             wo, wi, L, R, y0, yst, f0, fst, O);
        else
          fix_line<MODE>(col + (uint32_t)S * PD4 + 4u * e * STX, (uint32_t)S * PD4, NP, c0, cst,
                         own && x < TX, wo, wi, L, R, y0, yst, f0, fst, O);
      }
      continue;
    }
    if (!LAST) {
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const uint32_t ad = col + (uint32_t)((2 * k + 1) * S) * PD4;
        if (NE == 1) {
          sts_f(ad, rec[0][k]);
        } else {
          float qq[4] = {P4[k].x, P4[k].y, P4[k].z, P4[k].w};
#pragma unroll
          for (int e = 0; e < NE; ++e) qq[e * STX] = rec[e][k];
          sts_f4(ad, make_float4(qq[0], qq[1], qq[2], qq[3]));
        }
      }
    }
    if (MODE == 0 && own) {
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const int p = (2 * k + 1) * S;
        const uint32_t cr = (D == 0) ? codea(T, p, a, 4 * j) : codea(T, a, p, 4 * j);
        // x positions of the quad off this pass's lattice are written by a
        // later pass (odd x at level 1, x = 2 mod 4 at level 2), so packed
        // stores may carry filler there
        if (NE == 4) {
          sts_u2(cr, make_uint2(code[0][k] | (code[1][k] << 16), code[2][k] | (code[3][k] << 16)));
        } else if (NE == 2) {
          sts_u2(cr, make_uint2(code[0][k], code[1][k]));
        } else {
          sts_u16(cr, code[0][k]);
        }
      }
    }
  }
}

// Pass code of the i-th pass of a level (the same at every level): axis D,
// which other axes were passed before it, the cubic variant of D.
//   pc = 8 D + 2 sel + nak, sel = passed & 3 for D = x, else (x passed) * 2 +
//   (the other non-x axis passed).
// Computed once per CTA (pass_codes), so a pass dispatches with one shared
// load and one jump table (ipass_pc) instead of a chain of dependent tests.
DEV void pass_codes(const int order[3], const int nak[3], int pc[3]) {
  int passed = 0;
  for (int i = 0; i < 3; ++i) {
    const int D = order[i];
    int sel;
    if (D == 2) {
      sel = passed & 3;
    } else {
      const bool xp = (passed & 4) != 0;
      const bool ap = (passed & (D == 0 ? 2 : 1)) != 0;
      sel = (xp ? 2 : 0) | (ap ? 1 : 0);
    }
    pc[i] = 8 * D + 2 * sel + (nak[D] ? 1 : 0);
    passed |= 1 << D;
  }
}

// One interior pass by pass code.  (wo, wi) are the variant's cubic weights
// (the exact line redo, fix_line, evaluates the spline with them); below
// S = 1 the y / z lines hold no cubic point, so their variant is moot.
template <int MODE, int S, int FK>
DEV void ipass_pc(const Tile &T, int pc, const Lv &L, int R, const Out &O, int fit) {
  constexpr int S2 = 2 * S;
  constexpr bool CUBIC_ZY = (S == 1);
#define T3_X(SEL, STZ, STY)                                                                 \
  case 16 + 2 * SEL:                                                                        \
    iwalk_x<S, STZ, STY, MODE, false, FK>(T, NAT_O, NAT_I, L, R, O, fit);                  \
    break;                                                                                  \
  case 17 + 2 * SEL:                                                                        \
    iwalk_x<S, STZ, STY, MODE, true, FK>(T, NAK_O, NAK_I, L, R, O, fit);                   \
    break;
#define T3_C(DD, SEL, STX, STA)                                                             \
  case 8 * DD + 2 * SEL:                                                                    \
    iwalk_col<S, DD, STX, STA, MODE, !CUBIC_ZY, FK>(T, NAT_O, NAT_I, L, R, O, fit);        \
    break;                                                                                  \
  case 8 * DD + 2 * SEL + 1:                                                                \
    iwalk_col<S, DD, STX, STA, MODE, true, FK>(T, NAK_O, NAK_I, L, R, O, fit);             \
    break;
  switch (pc) {
    T3_X(0, S2, S2)
    T3_X(1, S, S2)
    T3_X(2, S2, S)
    T3_X(3, S, S)
    T3_C(0, 0, S2, S2)
    T3_C(0, 1, S2, S)
    T3_C(0, 2, S, S2)
    T3_C(0, 3, S, S)
    T3_C(1, 0, S2, S2)
    T3_C(1, 1, S2, S)
    T3_C(1, 2, S, S2)
    T3_C(1, 3, S, S)
    default: break;
  }
#undef T3_X
#undef T3_C
}

// One interior pass: (S, D, passed) -> walk instantiation.  passed: bit a
// set when axis a was passed earlier at this level.
#define T3_NAKSEL(CALL_T, CALL_F) \
  do {                            \
    if (nak) CALL_T;              \
    else CALL_F;                  \
  } while (0)

template <int MODE, int S, int FK>
DEV void ipass(const Tile &T, int D, int passed, bool nak, double wo, double wi, const Lv &L,
               int R, const Out &O, int fit) {
  constexpr int S2 = 2 * S;
  // the cubic case only exists along x at S = 4, 2 and everywhere at S = 1
  constexpr bool CUBIC_ZY = (S == 1);
#define T3_WX(STZ, STY)                                                              \
  T3_NAKSEL((iwalk_x<S, STZ, STY, MODE, true, FK>(T, wo, wi, L, R, O, fit)),         \
            (iwalk_x<S, STZ, STY, MODE, false, FK>(T, wo, wi, L, R, O, fit)))
  if (D == 2) {
    switch (passed & 3) {
      case 0: T3_WX(S2, S2); break;
      case 1: T3_WX(S, S2); break;
      case 2: T3_WX(S2, S); break;
      default: T3_WX(S, S); break;
    }
    return;
  }
#undef T3_WX
  const bool xp = (passed & 4) != 0;
  const bool ap = (passed & (D == 0 ? 2 : 1)) != 0;
  const int sel = (xp ? 2 : 0) | (ap ? 1 : 0);
#define T3_COL(DD, STX, STA)                                                              \
  do {                                                                                    \
    if (CUBIC_ZY)                                                                         \
      T3_NAKSEL((iwalk_col<S, DD, STX, STA, MODE, true, FK>(T, wo, wi, L, R, O, fit)),    \
                (iwalk_col<S, DD, STX, STA, MODE, false, FK>(T, wo, wi, L, R, O, fit)));  \
    else                                                                                  \
      iwalk_col<S, DD, STX, STA, MODE, true, FK>(T, wo, wi, L, R, O, fit);                \
  } while (0)
  if (D == 0) {
    switch (sel) {
      case 0: T3_COL(0, S2, S2); break;
      case 1: T3_COL(0, S2, S); break;
      case 2: T3_COL(0, S, S2); break;
      default: T3_COL(0, S, S); break;
    }
  } else {
    switch (sel) {
      case 0: T3_COL(1, S2, S2); break;
      case 1: T3_COL(1, S2, S); break;
      case 2: T3_COL(1, S, S2); break;
      default: T3_COL(1, S, S); break;
    }
  }
#undef T3_COL
}
#undef T3_NAKSEL

// Compress dispatches by pass code (measured: predict 535 -> 525 us on
// 512^3); the reconstructor keeps the test chain (its jump-table variant
// measured 20 us slower).
template <int MODE, int S, int FK>
DEV void ilevel(const Tile &T, const Cfg &C, int lv, int R, const Out &O, int fit) {
  const Lv L = C.lv[lv];
  int passed = 0;
#pragma unroll 1
  for (int i = 0; i < 3; ++i) {
#ifdef T3_PROF
    const long long q0 = clock64();
#endif
    if (MODE == 0) {
      ipass_pc<MODE, S, FK>(T, C.pc[i], L, R, O, fit);
    } else {
      const int D = C.order[i];
      const bool nak = C.nak[D] != 0;
      ipass<MODE, S, FK>(T, D, passed, nak, nak ? NAK_O : NAT_O, nak ? NAK_I : NAT_I, L, R, O,
                         fit);
      passed |= 1 << D;
    }
    __syncwarp();
#ifdef T3_PROF
    if (MODE == 0 && FK != 1 && (threadIdx.x & 31) == 0)
      atomicAdd(&g_t3_prof[6 + lv * 3 + i], (unsigned long long)(clock64() - q0));
#endif
  }
}

// FK (iwalk_x): 1 an exact-fit edge tile, fit = its fit mask (fit_mask)
template <int MODE, int FK = 0>
DEV void run_levels_i(const Tile &T, const Cfg &C, int R, const Out &O, int fit = 0) {
  ilevel<MODE, 4, FK>(T, C, 0, R, O, fit);
  ilevel<MODE, 2, FK>(T, C, 1, R, O, fit);
  ilevel<MODE, 1, FK>(T, C, 2, R, O, fit);
}

// Walk kind of a tile: -1 when some axis ends inside the tile (the generic
// walks, run_levels<.., true>), else bit a set when axis a ends exactly at
// the tile's end (0: every closing plane inside the grid).
DEV int fit_mask(const Tile &T) {
  int m = 0;
  if (T.e[0] < TZ || T.e[1] < TY || T.e[2] < TX) return -1;
  if (T.e[0] == TZ) m |= 1;
  if (T.e[1] == TY) m |= 2;
  if (T.e[2] == TX) m |= 4;
  return m;
}
