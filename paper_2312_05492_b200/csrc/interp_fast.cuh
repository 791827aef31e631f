// Compile-time specialised interpolation passes for the default layouts
// (predictor.py:71-105): 3-D stride 8 / tiles (8,8,32) on 8x16x32 blocks,
// 2-D stride 16 / tiles (16,16) on 32x64 blocks, 1-D stride 512 / tile 512
// on 1024-point blocks (grids padded to 3-D with leading extent-1 axes).
//
// INTERIOR blocks (closing plane inside the grid on every axis) need no
// extent or anchor checks: pass coordinates are odd multiples of s, the
// only in-block ext-1 coordinates are multiples of the anchor stride, and
// the spline case depends only on the point's offset inside its tile (the
// first point of a tile has no -3s neighbour, the last none at +3s).
// BOUNDARY blocks use the same code with runtime extent checks: the closed
// block is padded with zeros, points beyond the grid are skipped, p1/p3 use
// the true extent and a pass point sitting on a closing anchor is skipped
// (predictor.py:367-392 restores it after the pass).
#pragma once

namespace cszi {
namespace fast {

template <int BZ_, int BY_, int BX_, int TZ_, int TY_, int TX_, int S_>
struct Lay {
  static constexpr int BZ = BZ_, BY = BY_, BX = BX_;
  static constexpr int TZ = TZ_, TY = TY_, TX = TX_, S = S_;
  static constexpr int CZ = BZ == 1 ? 1 : BZ + 1, CY = BY == 1 ? 1 : BY + 1, CX = BX + 1;
  static constexpr int PX = CX, PY = CY;
  static constexpr int NCLOSED = CZ * CY * CX;
  static constexpr int NOWNED = BZ * BY * BX;
  static constexpr int B(int a) { return a == 0 ? BZ : a == 1 ? BY : BX; }
  static constexpr int C(int a) { return a == 0 ? CZ : a == 1 ? CY : CX; }
  static constexpr int T(int a) { return a == 0 ? TZ : a == 1 ? TY : TX; }
  static constexpr int P(int a) { return a == 0 ? PY * PX : a == 1 ? PX : 1; }
  static constexpr int CS(int a) { return a == 0 ? BY * BX : a == 1 ? BX : 1; }
};

using L3 = Lay<8, 16, 32, 8, 8, 32, 8>;
using L2 = Lay<1, 32, 64, 1, 16, 16, 16>;
using L1 = Lay<1, 1, 1024, 1, 1, 512, 512>;

struct Quant {
  double leb, e2, inv, Rd;
  int R;
};

struct Blk {
  int e[3];          // grid extent minus block origin (local extent) per axis
  const u64 *idx;    // decompress outliers
  const float *val;
  u64 n;
  int64_t gs0, gs1;  // flat-index strides of axes 0, 1
  int o0, o1, o2;    // block origin
};

// predictor.py:327-339 (see predict.cu for the fast-path argument).  The
// quotient is RN(r * RN(1/e2)); whenever it lies within 2^-20 of a
// half-integer the exact division decides.
template <bool EXACT>
DEV uint32_t quant(double pred, float o32, const Quant &Q, float &recon) {
  const double o = (double)o32;
  const double r = dsub(o, pred);
  double qd;
  int q;
  bool big;
  bool fast = false;
  if (!EXACT) {
    const double t = dmul(r, Q.inv);
    const double m = dadd(t, MAGIC);
    const double rq = dsub(m, MAGIC);
    if (fabs(dsub(t, rq)) <= 0.49999904632568359375) {
      fast = true;
      big = fabs(rq) >= Q.Rd;
      q = __double2loint(m);
      qd = big ? 0.0 : rq;
    }
  }
  if (!fast) {
    const double t = ddiv(r, Q.e2);
    const double qf = trunc(dadd(t, copysign(0.5, t)));
    big = fabs(qf) >= Q.Rd;
    q = big ? 0 : (int)qf;
    qd = (double)q;
  }
  const float rec = __double2float_rn(dadd(pred, dmul(Q.e2, qd)));
  const bool bad = big || (fabs(dsub((double)rec, o)) > Q.leb);
  recon = bad ? o32 : rec;
  return bad ? 0u : (uint32_t)(q + Q.R);
}

// One (level S, dimension D) pass; PASSED = bitmask of dims already passed
// at this level.  MODE 0 compress, 1 decompress.
template <class LY, int MODE, bool EXACT, bool BND, int NT, int S, int D, int PASSED>
DEV void pass(float *buf, uint16_t *codes, const uint16_t *csym, double wo, double wi,
              const Quant &Q, const Blk &K) {
  const bool nak = wo == NAK_O;
  constexpr int A1 = (D == 0) ? 1 : 0;
  constexpr int A2 = (D == 2) ? 1 : 2;
  constexpr int ST1 = ((PASSED >> A1) & 1) ? S : 2 * S;
  constexpr int ST2 = ((PASSED >> A2) & 1) ? S : 2 * S;
  constexpr int CNT1 = (LY::C(A1) - 1) / ST1 + 1;
  constexpr int CNT2 = (LY::C(A2) - 1) / ST2 + 1;
  constexpr int NL = CNT1 * CNT2;
  constexpr int NP = LY::B(D) / (2 * S);  // points per line
  constexpr int PT = (LY::T(D) / (2 * S)) > 0 ? LY::T(D) / (2 * S) : 1;
  constexpr int SEG = PT < 4 ? PT : 4;
  constexpr int NSEG = NP / SEG;
  constexpr int GPT = PT / SEG;  // segments per tile
  constexpr int PD = LY::P(D);
  constexpr int ES = 2 * S * PD;  // smem distance of even positions
  constexpr int ITEMS = NSEG * NL;
  constexpr int AM = LY::S - 1;   // anchor-lattice mask
  const int ed = K.e[D];
  for (int it = threadIdx.x; it < ITEMS; it += NT) {
    const int sg = it / NL;
    const int line = it - sg * NL;
    const int i1 = line / CNT2;
    const int i2 = line - i1 * CNT2;
    const int l1 = i1 * ST1, l2 = i2 * ST2;
    if (BND && (l1 >= K.e[A1] || l2 >= K.e[A2])) continue;
    float *base = buf + l1 * LY::P(A1) + l2 * LY::P(A2);
    const bool owned = BND ? (l1 < min(LY::B(A1), K.e[A1]) && l2 < min(LY::B(A2), K.e[A2]))
                           : (l1 < LY::B(A1) && l2 < LY::B(A2));
    const bool line_anchor = BND && ((l1 & AM) == 0 || l1 == K.e[A1] - 1) &&
                             ((l2 & AM) == 0 || l2 == K.e[A2] - 1);
    const int k0 = sg * SEG;
    const int tpos = (GPT > 1) ? (sg % GPT) : 0;
    const bool first = tpos == 0, last = tpos == GPT - 1;
    double vm3 = (k0 >= 1) ? (double)base[(k0 - 1) * ES] : 0.0;
    double vm1 = (double)base[k0 * ES];
    double vp1 = (double)base[(k0 + 1) * ES];
    double vp3 = (k0 + 2 <= NP) ? (double)base[(k0 + 2) * ES] : 0.0;
#pragma unroll
    for (int j = 0; j < SEG; ++j) {
      const int k = k0 + j;
      const int pdl = (2 * k + 1) * S;
      bool skip = false;
      bool m3 = !(j == 0 && first);
      bool p3 = !(j == SEG - 1 && last);
      bool p1 = true;
      if (BND) {
        skip = pdl >= ed || (line_anchor && pdl == ed - 1);
        p1 = pdl + S <= ed - 1;
        p3 = p3 && (pdl + 3 * S <= ed - 1);
      }
      if (!skip) {
        // ((w0 v0 + w1 v1) + w2 v2) + w3 v3 in float64.  For the dyadic
        // weights (not-a-knot, quadratic, linear) every w*v of a float v is
        // exact, so fma(w, v, acc) == RN(RN(w*v) + acc) bit for bit; the
        // natural-spline weights (/40) are not and keep mul + add.
        double pred;
        if (!p1)
          pred = vm1;
        else if (m3 && p3)
          pred = nak ? __fma_rn(wo, vp3, __fma_rn(wi, vp1, __fma_rn(wi, vm1, dmul(wo, vm3))))
                     : dadd(dadd(dadd(dmul(wo, vm3), dmul(wi, vm1)), dmul(wi, vp1)),
                            dmul(wo, vp3));
        else if (m3)
          pred = __fma_rn(QF, vp1, __fma_rn(QN, vm1, dmul(QO, vm3)));
        else if (p3)
          pred = __fma_rn(QO, vp3, __fma_rn(QN, vp1, dmul(QF, vm1)));
        else
          pred = __fma_rn(0.5, vp1, dmul(0.5, vm1));
        float *pp = base + pdl * PD;
        if (MODE == 0) {
          float rec;
          const uint32_t sy = quant<EXACT>(pred, *pp, Q, rec);
          *pp = rec;
          if (owned && (!BND || pdl < LY::B(D)))
            codes[pdl * LY::CS(D) + l1 * LY::CS(A1) + l2 * LY::CS(A2)] = (uint16_t)sy;
        } else {
          const uint32_t code = csym[pp - buf];
          float v;
          if (code == 0xFFFFu) {
            int c[3];
            c[D] = pdl;
            c[A1] = l1;
            c[A2] = l2;
            const u64 flat =
                (u64)((K.o0 + c[0]) * K.gs0 + (K.o1 + c[1]) * K.gs1 + (K.o2 + c[2]));
            v = outlier_value(K.idx, K.val, K.n, flat);
          } else {
            const int q = (int)code - Q.R;
            const double qd =
                dsub(__hiloint2double(0x43300000, (int)((uint32_t)q ^ 0x80000000u)),
                     4503601774854144.0);  // exact int -> double
            v = __double2float_rn(dadd(pred, dmul(Q.e2, qd)));
          }
          *pp = v;
        }
      }
      vm3 = vm1;
      vm1 = vp1;
      vp1 = vp3;
      if (j + 1 < SEG) vp3 = (k + 3 <= NP) ? (double)base[(k + 3) * ES] : 0.0;
    }
  }
  __syncthreads();
}

template <class LY> DEV constexpr bool real_axis(int a) { return LY::C(a) > 1; }

// All passes of level S in the order (D0, D1, D2) (padded axes skipped).
template <class LY, int MODE, bool EXACT, bool BND, int NT, int S, int D0, int D1, int D2>
DEV void level(float *buf, uint16_t *codes, const uint16_t *csym, const double wo[3],
               const double wi[3], const Quant &Q, const Blk &K, const int ext[3]) {
  if constexpr (real_axis<LY>(D0))
    if (S < ext[D0]) pass<LY, MODE, EXACT, BND, NT, S, D0, 0>(buf, codes, csym, wo[D0], wi[D0], Q, K);
  if constexpr (real_axis<LY>(D1))
    if (S < ext[D1])
      pass<LY, MODE, EXACT, BND, NT, S, D1, (1 << D0)>(buf, codes, csym, wo[D1], wi[D1], Q, K);
  if constexpr (real_axis<LY>(D2))
    if (S < ext[D2])
      pass<LY, MODE, EXACT, BND, NT, S, D2, (1 << D0) | (1 << D1)>(buf, codes, csym, wo[D2],
                                                                   wi[D2], Q, K);
}

template <class LY, int MODE, bool EXACT, bool BND, int NT, int S, int D0, int D1, int D2>
DEV void levels_from(float *buf, uint16_t *codes, const uint16_t *csym, const LevelCfg &cfg,
                     const double wo[3], const double wi[3], Quant &Q, const Blk &K,
                     const int ext[3], int lv) {
  Q.leb = cfg.leb[lv];
  Q.e2 = dmul(2.0, Q.leb);
  Q.inv = cfg.inv[lv];
  level<LY, MODE, EXACT, BND, NT, S, D0, D1, D2>(buf, codes, csym, wo, wi, Q, K, ext);
  if constexpr (S > 1)
    levels_from<LY, MODE, EXACT, BND, NT, S / 2, D0, D1, D2>(buf, codes, csym, cfg, wo, wi, Q,
                                                             K, ext, lv + 1);
}

template <class LY, int MODE, bool EXACT, bool BND, int NT, int D0, int D1, int D2>
DEV void levels(float *buf, uint16_t *codes, const uint16_t *csym, const LevelCfg &cfg, int R,
                const Blk &K, const int ext[3]) {
  double wo[3], wi[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    wo[a] = cfg.variant[a] ? NAT_O : NAK_O;
    wi[a] = cfg.variant[a] ? NAT_I : NAK_I;
  }
  Quant Q;
  Q.R = R;
  Q.Rd = (double)R;
  levels_from<LY, MODE, EXACT, BND, NT, LY::S / 2, D0, D1, D2>(buf, codes, csym, cfg, wo, wi, Q,
                                                               K, ext, 0);
}

// dispatch on the (runtime) dimension order of the padded axes
template <class LY, int MODE, bool EXACT, bool BND, int NT>
DEV void run(float *buf, uint16_t *codes, const uint16_t *csym, const LevelCfg &cfg, int R,
             const Blk &K, const int ext[3], int rank) {
  if constexpr (LY::CZ == 1 && LY::CY == 1) {  // rank 1: order (2)
    levels<LY, MODE, EXACT, BND, NT, 2, 0, 1>(buf, codes, csym, cfg, R, K, ext);
  } else if constexpr (LY::CZ == 1) {  // rank 2: order (1,2) or (2,1)
    if (cfg.order[0] == 1)
      levels<LY, MODE, EXACT, BND, NT, 1, 2, 0>(buf, codes, csym, cfg, R, K, ext);
    else
      levels<LY, MODE, EXACT, BND, NT, 2, 1, 0>(buf, codes, csym, cfg, R, K, ext);
  } else {
    const int code = cfg.order[0] * 9 + cfg.order[1] * 3 + cfg.order[2];
    switch (code) {
      case 0 * 9 + 1 * 3 + 2: levels<LY, MODE, EXACT, BND, NT, 0, 1, 2>(buf, codes, csym, cfg, R, K, ext); break;
      case 0 * 9 + 2 * 3 + 1: levels<LY, MODE, EXACT, BND, NT, 0, 2, 1>(buf, codes, csym, cfg, R, K, ext); break;
      case 1 * 9 + 0 * 3 + 2: levels<LY, MODE, EXACT, BND, NT, 1, 0, 2>(buf, codes, csym, cfg, R, K, ext); break;
      case 1 * 9 + 2 * 3 + 0: levels<LY, MODE, EXACT, BND, NT, 1, 2, 0>(buf, codes, csym, cfg, R, K, ext); break;
      case 2 * 9 + 0 * 3 + 1: levels<LY, MODE, EXACT, BND, NT, 2, 0, 1>(buf, codes, csym, cfg, R, K, ext); break;
      default: levels<LY, MODE, EXACT, BND, NT, 2, 1, 0>(buf, codes, csym, cfg, R, K, ext); break;
    }
  }
}

DEV void cp_async4(void *sdst, const void *gsrc, bool valid) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(sdst);
  const int n = valid ? 4 : 0;  // src-size 0 zero-fills
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(gsrc), "r"(n)
               : "memory");
}
DEV void cp_async_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Stage the closed block into smem: one warp per row (z, y), lanes over x.
// 4-byte elements go through cp.async (all rows in flight at once, no
// registers); 2-byte symbols are loaded in batches of 8 rows per warp
// before being stored.  Points outside the grid read as zero.
template <class LY, bool BND, int NT, typename T>
DEV void stage(T *dst, const T *__restrict__ src, int64_t base, int pz, int py, const int e[3]) {
  const T *sb = src + base;  // block origin; in-block offsets fit 32 bits
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NROWS = LY::CZ * LY::CY;
  constexpr int NW = NT / 32;
  if constexpr (sizeof(T) == 4) {
    for (int row = warp; row < NROWS; row += NW) {
      const int z = row / LY::CY, y = row - z * LY::CY;
      const bool rv = !BND || (z < e[0] && y < e[1]);
      const T *g = sb + (z * pz + y * py);
      T *d = dst + row * LY::CX;
#pragma unroll
      for (int x0 = 0; x0 < LY::CX; x0 += 32) {
        const int x = x0 + lane;
        if (x < LY::CX) {
          const bool v = rv && (!BND || x < e[2]);
          cp_async4(d + x, v ? (const void *)(g + x) : (const void *)sb, v);
        }
      }
    }
    cp_async_wait();
  } else {
    constexpr int XW = (LY::CX + 31) / 32;  // elements per lane per row
    constexpr int RB = 8;                   // rows per batch
    for (int r0 = warp; r0 < NROWS; r0 += NW * RB) {
      T v[RB][XW];
#pragma unroll
      for (int b = 0; b < RB; ++b) {
        const int row = r0 + b * NW;
        const int z = row / LY::CY, y = row - z * LY::CY;
        const bool rv = row < NROWS && (!BND || (z < e[0] && y < e[1]));
        const T *g = sb + (z * pz + y * py);
#pragma unroll
        for (int c = 0; c < XW; ++c) {
          const int x = c * 32 + lane;
          v[b][c] = (rv && x < LY::CX && (!BND || x < e[2])) ? __ldg(g + x) : T(0);
        }
      }
#pragma unroll
      for (int b = 0; b < RB; ++b) {
        const int row = r0 + b * NW;
#pragma unroll
        for (int c = 0; c < XW; ++c) {
          const int x = c * 32 + lane;
          if (row < NROWS && x < LY::CX) dst[row * LY::CX + x] = v[b][c];
        }
      }
    }
  }
}

// Owned codes (smem, row-major BZ x BY x BX) -> global + block histogram
// (outlier sentinel 0 and symbol R are counted as R).
template <class LY, bool BND, int NT>
DEV uint32_t store_codes_hist(const uint16_t *codes, uint16_t *__restrict__ sym, int64_t base,
                              int64_t pz, int py, const int e[3], int R, uint32_t *hs,
                              bool hist_in_smem, u64 *hist) {
  constexpr int EPT = LY::NOWNED / NT;
  static_assert(LY::NOWNED % NT == 0 && LY::BX % EPT == 0, "owned block / threads");
  constexpr int TPR = LY::BX / EPT;  // threads per row
  const int t = threadIdx.x;
  const int row = t / TPR, part = t - row * TPR;
  const int z = row / LY::BY, y = row - z * LY::BY;
  if (BND && (z >= e[0] || y >= e[1])) return 0;
  const uint16_t *src = codes + row * LY::BX + part * EPT;
  uint16_t *dst = sym + base + ((int64_t)z * pz + (int64_t)y * py) + part * EPT;
  const int x0 = part * EPT;
  uint32_t v[EPT / 2];
#pragma unroll
  for (int k = 0; k < EPT / 2; ++k) v[k] = reinterpret_cast<const uint32_t *>(src)[k];
  const bool full = !BND || x0 + EPT <= e[2];
  if (full && (reinterpret_cast<uintptr_t>(dst) & 15) == 0 && EPT % 8 == 0) {
#pragma unroll
    for (int k = 0; k < EPT / 8; ++k)
      reinterpret_cast<uint4 *>(dst)[k] =
          make_uint4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
  } else {
#pragma unroll
    for (int k = 0; k < EPT; ++k)
      if (!BND || x0 + k < e[2])
        dst[k] = (uint16_t)((k & 1) ? (v[k >> 1] >> 16) : (v[k >> 1] & 0xffffu));
  }
  uint32_t zeros = 0;
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    if (BND && x0 + k >= e[2]) continue;
    const uint32_t sy = (k & 1) ? (v[k >> 1] >> 16) : (v[k >> 1] & 0xffffu);
    if (sy == (uint32_t)R || sy == 0) {
      zeros++;
    } else if (hist_in_smem) {
      atomicAdd(&hs[sy], 1u);
    } else {
      atomicAdd(&hist[sy], 1ull);
    }
  }
  return zeros;
}

}  // namespace fast
}  // namespace cszi
