// Warp-per-tile G-Interp predictor (compress) and inverse interpolation
// (decompress) for the 3-D default layout: anchor stride 8, super-chunk
// tiles (8, 8, 32) in (z, y, x) (predictor.py:71-72, 99-105).
//
// Reference semantics: predictor.py:283-344 (_run_pass), :367-392
// (interpolate_level), :395-465 (compress_predict / decompress_predict).
//
// Work unit: ONE WARP owns ONE tile.  Neighbour reads are confined to the
// tile plus its closing plane on each axis, so a warp stages
// the closed 9 x 9 x 33 box (one TMA load, box 36 x 9 x 9, out-of-grid
// elements zero-filled), runs all nine (level, dimension) passes with only
// __syncwarp() between them, and stores the owned 8 x 8 x 32 results.  No
// block barrier sits on the hot path: the warps of an SM drift through
// different passes, so the latency-bound coarse passes of one tile overlap
// the throughput-bound fine passes of another.
//
// Shared-memory layout per warp: buf[z][y][x] floats with row pitch 36
// (= the TMA box), codes[z][y][x] u16 with row pitch 36 (compress), syms
// [z][y][x] u16 with row pitch 40 (decompress, a second TMA box).  The fine
// passes (s = 2, 1) of interior tiles run as vectorised walks:
//   * D = x: a lane walks a whole row with 16-byte loads / stores (rows of
//     one quarter-warp hit 8 distinct 16-byte bank groups: conflict-free);
//   * D = y, z: a lane owns a quad of 4 adjacent x-lines and walks along D
//     (adjacent lanes on adjacent quads: conflict-free).
// Every point of a walk is independent (a pass never reads what it writes),
// so the unrolled walk exposes 8-16 independent fp64 chains per lane.  The
// coarse level (s = 4, 2% of the points) and tiles touching the grid edge
// run a generic per-point pass with runtime extents and closing anchors.
//
// Quantisation (predictor.py:327-339) in float64 with the reference's
// operation order: t = r * RN(1/e2) replaces the division away from
// half-integers (exact fallback otherwise), and the float32-rounding guard
// |f64(rec) - o| > eb is decided without the rec -> f64 round trip when
// |y - o| <= eb (1 - 2^-40) - 2^-23 |y| - 2^-148 proves it false (see
// quant_fast); every other point takes the exact scalar path.
#pragma once

#include <cuda.h>

#include "interp_common.cuh"

#include <atomic>
#include <cstdlib>
#include <cstring>

namespace cszi {
namespace t3 {

constexpr int TZ = 8, TY = 8, TX = 32;          // tile
constexpr int CZ = 9, CY = 9, CX = 33;          // closed tile
constexpr int PX = 36;                          // float row pitch (TMA box x)
constexpr int PZ = CY * PX;                     // 324
constexpr int NBUF = CZ * CY * PX;              // 2916 floats
constexpr int CP = 36;                          // code row pitch (u16)
constexpr int NCODE = TZ * TY * CP;             // 2304 u16
constexpr int SP = 40;                          // symbol row pitch (u16, TMA box x)
constexpr int NSYM = CZ * CY * SP;              // 3240 u16
#ifndef T3R_NW
#define T3R_NW 4
#endif
constexpr int NW = T3R_NW;                      // warps (tiles) per CTA (reconstruct)
constexpr int NT = NW * 32;
constexpr int MINB_R = (NW <= 4) ? 12 / NW : 1;
#ifndef T3P_NW
#define T3P_NW 12
#endif
constexpr int NWP = T3P_NW;                     // warps per CTA of the predictor
constexpr int NTP = NWP * 32;
#ifdef T3P_REGS
#define T3P_BOUNDS __maxnreg__(T3P_REGS)
#else
#define T3P_BOUNDS __launch_bounds__(NTP, MINB_P)
#endif
constexpr int MINB_P = (NWP <= 4) ? 12 / NWP : 1;  // resident CTAs per SM (launch bounds)
// per-warp shared regions (128-byte aligned for the TMA destinations)
constexpr int BUF_BYTES = NBUF * 4;                              // 11664
constexpr int NZ_BYTES = TZ * TY * 4;  // non-R bitmap words of a tile's rows
constexpr int P_WARP = ((BUF_BYTES + NCODE * 2 + NZ_BYTES) + 127) & ~127;   // 16640
constexpr int SYM_BYTES = ((NSYM * 2) + 127) & ~127;             // 6528
constexpr int R_WARP = ((SYM_BYTES + BUF_BYTES) + 127) & ~127;   // 18304

struct Lv {
  double leb, e2, inv, lebs;
  float a32;  // interior fast path: accept |RN32(rec - o)| <= a32 (see quant_i)
};

// Division by a launch-constant divisor d (n < 2^31): q = (umulhi(n, m) + n)
// >> s with s = ceil(log2 d), m = floor(2^32 (2^s - d) / d) + 1 (Granlund-
// Montgomery round-up method; t + n cannot wrap because t <= n < 2^31).
struct FDiv {
  uint32_t m, s, d;
};
DEV uint32_t fdiv(uint32_t n, const FDiv &f) { return (__umulhi(n, f.m) + n) >> f.s; }
static inline FDiv make_fdiv(uint32_t d) {
  FDiv f;
  f.d = d ? d : 1;
  uint32_t s = 0;
  while ((1ull << s) < f.d) ++s;
  f.s = s;
  f.m = (uint32_t)((((1ull << s) - f.d) << 32) / f.d + 1);
  return f;
}

struct Geo {
  int ext[3];        // global extents
  int nzl;           // planes held by the input buffer (slab incl. halo)
  int z0;            // global z of local plane 0
  int nt[3];         // tiles per axis (axis 0 over the owned planes)
  int ni[3];         // interior tiles per axis (closing plane inside the grid)
  int R;
  int hist_smem;
  int tma;           // 1: 3-D tensor map valid, 0: row-wise cp.async / load staging
  int exact;         // 1: force the true-division quantiser (tests)
  int64_t na1, na2;  // anchor lattice counts on axes 1, 2 (decompress)
  // tile-index divisors: ni[2], ni[1], nt[2], nt[1], nt[1] - ni[1], nt[2] - ni[2]
  FDiv d_ni2, d_ni1, d_nt2, d_nt1, d_wy, d_wx;
  int shell_a, shell_b;  // edge tiles beyond ni[0] on z / beyond ni[1] on y
};

// ---------------------------------------------------------------------------
// TMA + mbarrier helpers
// ---------------------------------------------------------------------------
DEV uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// The dynamic shared window is only guaranteed 16-byte aligned after the
// static variables; TMA destinations need 128.  The address is laundered
// through asm so the compiler cannot fold the test from the declaration.
DEV unsigned char *align128(unsigned char *p) {
  uint32_t a = smem_u32(p);
  asm volatile("" : "+r"(a));
  return p + ((128u - (a & 127u)) & 127u);
}

DEV void mbar_init(uint64_t *mb) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mb)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
DEV void mbar_expect(uint64_t *mb, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)),
               "r"(bytes)
               : "memory");
}
DEV void mbar_wait(uint64_t *mb, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "W_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n"
      "}\n" ::"r"(smem_u32(mb)),
      "r"(parity)
      : "memory");
}

// Stage the closed box of the tile at origin o into dst (one 3-D TMA box of
// 9 x 9 rows of BX elements) and arm mbar for it.  Called by all lanes.
template <int BX, int ESZ>
DEV void tile_load(uint32_t dst, const CUtensorMap *tm, const Geo &G, const int o[3],
                   uint64_t *mb) {
  if ((threadIdx.x & 31) == 0) {
    mbar_expect(mb, (uint32_t)(CZ * CY * BX * ESZ));
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], "
        "[%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(o[2]), "r"(o[1]), "r"(o[0] - G.z0),
        "r"(smem_u32(mb))
        : "memory");
  }
}

// ---------------------------------------------------------------------------
// per-point arithmetic
// ---------------------------------------------------------------------------
// spline predictions with dyadic weights: every w * v of a float v is exact
// in float64, so fma(w, v, acc) == RN(RN(w v) + acc) bit for bit.
DEV double p_cubic(bool nak, double a, double b, double c, double d) {
  if (nak) return __fma_rn(NAK_O, d, __fma_rn(NAK_I, c, __fma_rn(NAK_I, b, dmul(NAK_O, a))));
  return dadd(dadd(dadd(dmul(NAT_O, a), dmul(NAT_I, b)), dmul(NAT_I, c)), dmul(NAT_O, d));
}
DEV double p_m3(double a, double b, double c) {  // no +3 neighbour: (-1/8, 6/8, 3/8, 0)
  return __fma_rn(QF, c, __fma_rn(QN, b, dmul(QO, a)));
}
DEV double p_p3(double b, double c, double d) {  // no -3 neighbour: (0, 3/8, 6/8, -1/8)
  return __fma_rn(QO, d, __fma_rn(QN, c, dmul(QF, b)));
}
DEV double p_lin(double b, double c) { return __fma_rn(0.5, c, dmul(0.5, b)); }

// ---------------------------------------------------------------------------
// shared-memory access by 32-bit shared-window address (keeps every access
// an LDS/STS: the tile pointers live in a struct, where generic-pointer
// provenance would otherwise be lost)
// ---------------------------------------------------------------------------
DEV float lds_f(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
DEV void sts_f(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
DEV float4 lds_f4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a));
  return v;
}
DEV void sts_f4(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
// bit 0: low code of a packed pair differs from R; bit 1: high code does
DEV uint32_t ne_r2(uint32_t w, uint32_t rr) {
  const uint32_t d = w ^ rr;
  return (uint32_t)((d & 0xffffu) != 0u) | ((uint32_t)(d > 0xffffu) << 1);
}
DEV uint32_t lds_u16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
DEV void sts_u16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v) : "memory");
}
DEV uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
DEV uint2 lds_u2(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
DEV void sts_u2(uint32_t a, uint2 v) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(v.x), "r"(v.y) : "memory");
}
DEV uint4 lds_u4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a));
  return v;
}
DEV void sts_u4(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ---------------------------------------------------------------------------
// quantiser
// ---------------------------------------------------------------------------
struct QS {
  uint32_t sym;
  float rec;
};

// Exact scalar quantiser (predictor.py:327-339): the rare points the fast
// path cannot decide, and every point under G.exact.
static __device__ __noinline__ QS quant_slow(double pred, float o32, double leb, double e2, double inv,
                                      int R) {
  QS q;
  q.sym = quantize<true>(pred, o32, leb, e2, inv, R, q.rec);
  return q;
}

// The same for a walk point: the neighbours are reloaded from shared memory
// (a pass never writes them), so the walk keeps no predictions live.
// cs: spline case (0 cubic, 1 no +3, 2 no -3, 3 linear), st: neighbour
// distance in bytes.
static __device__ __noinline__ QS fix_point(uint32_t a, uint32_t st, int cs, double wo, double wi,
                                     float o32, double leb, double e2, double inv, int R) {
  float v[4];
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[1]) : "r"(a - st));
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[2]) : "r"(a + st));
  v[0] = 0.f;
  v[3] = 0.f;
  if (cs <= 1) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[0]) : "r"(a - 3 * st));
  if (cs == 0 || cs == 2) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[3]) : "r"(a + 3 * st));
  const double pred = spline4(cs, wo, wi, (double)v[0], (double)v[1], (double)v[2], (double)v[3]);
  return quant_slow(pred, o32, leb, e2, inv, R);
}

// Fast quantiser; returns false when undecided (then call quant_slow).
//  * t' = r * RN(1/e2) lies within 3 ulp of RN(r / e2); unless t' is within
//    2^-20 of a half-integer, rint(t') == trunc(t + copysign(.5, t)); the
//    magic-number round leaves rint(t') in the low word of m.
//  * y = RN(pred + RN(e2 q)); rec = RN32(y).  |rec - y| <= 2^-24 |y| +
//    2^-150, so |dy| <= leb (1 - 2^-40) - 2^-23 |y| - 2^-148 with
//    dy = RN(y - o) implies RN(f64(rec) - o) <= leb: the guard is false.
//    (lebs is capped at 2^100 so that such a y never overflows float32.)
// big (|q| >= R) points are outliers whatever the guard says.
DEV bool quant_fast(double pred, float o32, const Lv &L, double Rd, int R, float &recon,
                    uint32_t &sym) {
  const double o = (double)o32;
  const double r = dsub(o, pred);
  const double t = dmul(r, L.inv);
  const double m = dadd(t, MAGIC);
  const double rq = dsub(m, MAGIC);
  const bool near_ok = fabs(dsub(t, rq)) <= 0.49999904632568359375;
  const bool big = fabs(rq) >= Rd;
  const double y = dadd(pred, dmul(L.e2, rq));
  const double dy = dsub(y, o);
  const bool safe = fabs(dy) <= __fma_rn(fabs(y), -0x1p-23, L.lebs);
  recon = big ? o32 : __double2float_rn(y);
  sym = big ? 0u : (uint32_t)(__double2loint(m) + R);
  return near_ok && (big || safe);
}

struct Out {  // decompress outlier list
  const u64 *idx;
  const float *val;
  u64 n;
};

static __device__ __noinline__ float outlier_at(const u64 *idx, const float *val, u64 n, u64 flat) {
  return outlier_value(idx, val, n, flat);
}

// decompress: predictor.py:340-344
DEV float dequant(double pred, uint32_t code, const Lv &L, int R) {
  const int q = (int)code - R;
  const double qd = dsub(__hiloint2double(0x43300000, (int)((uint32_t)q ^ 0x80000000u)),
                         4503601774854144.0);  // exact int -> double
  return __double2float_rn(dadd(pred, dmul(L.e2, qd)));
}

// ---------------------------------------------------------------------------
// tile context
// ---------------------------------------------------------------------------
struct Tile {
  uint32_t buf;    // shared address of buf[0][0][0] (float, pitch PX)
  uint32_t codes;  // compress: codes[0][0][0] (u16, pitch CP)
  uint32_t syms;   // decompress: syms[0][0][0] (u16, pitch SP)
  int o[3];        // global origin
  int e[3];        // ext - origin
  bool bnd;
  int64_t gs0, gs1;  // flat-index strides (outlier lookup)
};

DEV uint32_t bufa(const Tile &T, int z, int y, int x) {
  return T.buf + 4u * (uint32_t)(z * PZ + y * PX + x);
}
DEV uint32_t codea(const Tile &T, int z, int y, int x) {
  return T.codes + 2u * (uint32_t)((z * TY + y) * CP + x);
}
DEV uint32_t syma(const Tile &T, int z, int y, int x) {
  return T.syms + 2u * (uint32_t)((z * CY + y) * SP + x);
}
DEV u64 flat_of(const Tile &T, int z, int y, int x) {
  return (u64)((T.o[0] + z) * T.gs0 + (T.o[1] + y) * T.gs1 + (T.o[2] + x));
}

// ---------------------------------------------------------------------------
// walks: every level, interior and edge tiles
// ---------------------------------------------------------------------------
// Spline case of the k-th point of a line (predictor.py:293-306).  Interior
// lines (closed plane present) have the compile-time pattern p3-only,
// cubic..., m3-only (a single point: linear); on edge tiles the case comes
// from the true extent and is warp-uniform (all lanes sit at the same
// position along D of the same tile).
template <int NP>
DEV int case_interior(int k) {
  return (NP == 1) ? 3 : (k == 0) ? 2 : (k == NP - 1) ? 1 : 0;
}

// Spline weights (vm3, vm1, vp1, vp3) per case for edge tiles; the cubic row
// is replaced by the tuned variant's (wo, wi).  The chain
// ((w0 a + w1 b) + w2 c) + w3 d is the reference expression (predictor.py
// :325, missing neighbours enter with weight 0); finite staged data stands
// in for missing neighbours, which only changes the sign of a zero term.
static __constant__ double c_w[5][4] = {{0.0, 0.0, 0.0, 0.0},
                                 {QO, QN, QF, 0.0},
                                 {0.0, QF, QN, QO},
                                 {0.0, 0.5, 0.5, 0.0},
                                 {0.0, 1.0, 0.0, 0.0}};

DEV double chain4(double w0, double w1, double w2, double w3, double a, double b, double c,
                  double d) {
  return dadd(dadd(dadd(dmul(w0, a), dmul(w1, b)), dmul(w2, c)), dmul(w3, d));
}

// interior lines: compile-time case pattern; edge tiles: case from the true
// extent (warp-uniform), weights from c_w.  cs < 0: interior.
template <int NP, bool BND, bool SW = false>
DEV double pred_k(int k, int cs, double wo, double wi, double a, double b, double c, double d) {
  if (!BND) {
    if (NP == 1) return p_lin(b, c);
    if (k == 0) return p_p3(b, c, d);
    if (k == NP - 1) return p_m3(a, b, c);
    return chain4(wo, wi, wi, wo, a, b, c, d);
  }
  if (cs == 0) return chain4(wo, wi, wi, wo, a, b, c, d);
  if (SW) {
    // compress edge tiles: the case is warp-uniform; its weights are
    // compile-time per branch (the c_w rows, with the zero-weight terms
    // dropped: they only change the sign of an exact zero, as in the
    // interior walks).  (Measured: predict -8 us on 512^3; the reconstructor
    // is faster with the table.)
    switch (cs) {
      case 1: return p_m3(a, b, c);
      case 2: return p_p3(b, c, d);
      case 3: return p_lin(b, c);
      default: return b;
    }
  }
  return chain4(c_w[cs][0], c_w[cs][1], c_w[cs][2], c_w[cs][3], a, b, c, d);
}

DEV bool anchor_coord(int c, int e) { return (c & 7) == 0 || c == e - 1; }

// D = x: lane walks rows (z, y) of the pass lattice.  S = 1, 2: 8 quads +
// x = 32 in 16-byte accesses; S = 4: 9 scalars.
template <int S, int MODE, bool BND>
DEV void walk_x(const Tile &T, int stz, int sty, double wo, double wi, const Lv &L, int R,
                bool exact, const Out &O) {
  const int lane = threadIdx.x & 31;
  const int ez = BND ? min(CZ, T.e[0]) : CZ, ey = BND ? min(CY, T.e[1]) : CY;
  const int ex = BND ? min(CX, T.e[2]) : CX;
  const int cz = (ez - 1) / stz + 1, cy = (ey - 1) / sty + 1;
  const int nl = cz * cy;
  const uint32_t mcy = (65536u + cy - 1) / cy;
  const double Rd = (double)R;
  constexpr int NP = 16 / S;  // points per row
  for (int l = lane; l < nl; l += 32) {
    const int iz = (int)(((uint32_t)l * mcy) >> 16);
    const int iy = l - iz * cy;
    const int z = iz * stz, y = iy * sty;
    const uint32_t row = bufa(T, z, y, 0);
    const bool row_anchor = BND && anchor_coord(z, T.e[0]) && anchor_coord(y, T.e[1]);
    double ev[NP + 1];  // even lattice values (neighbours)
    float pt[NP];       // pass points
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
            // word 4j + h holds x = 8j + 2h (low half) and 8j + 2h + 1 (high)
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
    uint32_t fail = 0, keep = 0;  // keep: point not updated (beyond / anchor)
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const int pd = (2 * k + 1) * S;
      int cs = -1;
      if (BND) {
        if (pd >= ex) {  // uniform: beyond the grid
          rec[k] = pt[k];
          code[k] = (uint32_t)R;
          keep |= 1u << k;
          continue;
        }
        cs = case_of(pd, S, TX, T.e[2]);
        if (row_anchor && pd == T.e[2] - 1) keep |= 1u << k;
      }
      const double pr = pred_k<NP, BND, MODE == 0>(k, cs, wo, wi, k > 0 ? ev[k - 1] : 0.0, ev[k],
                                                   ev[k + 1], k + 2 <= NP ? ev[k + 2] : 0.0);
      if (MODE == 0) {
        if (!quant_fast(pr, pt[k], L, Rd, R, rec[k], code[k])) fail |= 1u << k;
      } else {
        rec[k] = dequant(pr, sy[k], L, R);
        if (sy[k] == 0xFFFFu) fail |= 1u << k;
      }
    }
    if (MODE == 0 && exact) fail = (1u << NP) - 1;
    fail &= ~keep;
    if (fail) {  // rare: exact quantiser / outlier values
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        if (fail & (1u << k)) {
          const int pd = (2 * k + 1) * S;
          if (MODE == 0) {
            const int cs = BND ? case_of(pd, S, TX, T.e[2]) : case_interior<NP>(k);
            const QS q = fix_point(row + 4 * pd, 4 * S, cs, wo, wi, pt[k], L.leb, L.e2, L.inv, R);
            rec[k] = q.rec;
            code[k] = q.sym;
          } else {
            rec[k] = outlier_at(O.idx, O.val, O.n, flat_of(T, z, y, pd));
          }
        }
      }
    }
    if (BND && keep) {
#pragma unroll
      for (int k = 0; k < NP; ++k)
        if (keep & (1u << k)) {
          rec[k] = pt[k];
          code[k] = (uint32_t)R;  // anchors: code 0 (predictor.py:414)
        }
    }
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
    if (MODE == 0 && z < TZ && y < TY) {
      const uint32_t cr = codea(T, z, y, 0);
#pragma unroll
      for (int k = 0; k < NP; ++k) sts_u16(cr + 2 * (2 * k + 1) * S, code[k]);
    }
  }
}

// D in {0 (z), 1 (y)}: lane owns the quad x in [4j, 4j + 4) at one coordinate
// a of the other non-x axis and walks along D (closed length 9).  STX is the
// x-lattice step: 1 -> all four x-lines, 2 -> x = 4j, 4j + 2, 4 -> x = 4j,
// 8 -> x = 4j on even quads only.  Quad 8 (x = 32..35) carries one real
// line (x = 32); its other elements compute on staged data and are never
// stored as codes (nor are elements beyond the grid on edge tiles).
template <int S, int D, int STX, int MODE, bool BND>
DEV void walk_col(const Tile &T, int sta, double wo, double wi, const Lv &L, int R, bool exact,
                  const Out &O) {
  const int lane = threadIdx.x & 31;
  constexpr uint32_t PD4 = 4u * ((D == 0) ? PZ : PX);
  constexpr int NE = (STX == 1) ? 4 : (STX == 2) ? 2 : 1;  // x-lines per quad
  constexpr int QS_ = (STX == 8) ? 2 : 1;                   // quad step
  constexpr int NP = 4 / S;                                 // points per line
  constexpr int NV = NP + 1;                                // neighbours per line
  constexpr int A = (D == 0) ? 1 : 0;
  const int ed = BND ? min(9, T.e[D]) : 9;
  const int ea = BND ? min(9, T.e[A]) : 9;
  const int e2 = T.e[2];
  const int nq = BND ? ((min(CX, e2) - 1) / (4 * QS_) + 1) : (QS_ == 2 ? 5 : 9);
  const int ca = (ea - 1) / sta + 1;
  const int items = ca * nq;
  const double Rd = (double)R;
  for (int it = lane; it < items; it += 32) {
    const int ia = it / nq, jj = it - ia * nq;
    const int j = jj * QS_;
    const int a = ia * sta;
    const bool a_anchor = BND && anchor_coord(a, T.e[A]);
    const uint32_t col = (D == 0) ? bufa(T, 0, a, 4 * j) : bufa(T, a, 0, 4 * j);
    double ev[NE][NV];
    float pt[NE][NP];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if (BND && 2 * v * S >= ed) {  // uniform: beyond the grid (never used)
#pragma unroll
        for (int e = 0; e < NE; ++e) ev[e][v] = 0.0;
        continue;
      }
      const float4 q = lds_f4(col + (uint32_t)(2 * v * S) * PD4);
      const float qq[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int e = 0; e < NE; ++e) ev[e][v] = (double)qq[e * STX];
    }
    float4 P4[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      P4[k] = lds_f4(col + (uint32_t)((2 * k + 1) * S) * PD4);
      const float qq[4] = {P4[k].x, P4[k].y, P4[k].z, P4[k].w};
#pragma unroll
      for (int e = 0; e < NE; ++e) pt[e][k] = qq[e * STX];
    }
    uint32_t sy[NE][NP];
    if (MODE == 1) {
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const int p = (2 * k + 1) * S;
        const uint2 w = (D == 0) ? lds_u2(syma(T, p, a, 4 * j)) : lds_u2(syma(T, a, p, 4 * j));
        const uint32_t h[4] = {w.x & 0xffffu, w.x >> 16, w.y & 0xffffu, w.y >> 16};
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          const int x = 4 * j + e * STX;
          sy[e][k] = ((x < CX) && (!BND || x < e2)) ? h[e * STX] : 0u;
        }
      }
    }
    float rec[NE][NP];
    uint32_t code[NE][NP];
    uint32_t fail = 0, keep = 0;
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const int pd = (2 * k + 1) * S;
      int cs = -1;
      if (BND) {
        if (pd >= ed) {  // uniform: beyond the grid
#pragma unroll
          for (int e = 0; e < NE; ++e) {
            rec[e][k] = pt[e][k];
            code[e][k] = (uint32_t)R;
            keep |= 1u << (e * NP + k);
          }
          continue;
        }
        cs = case_of(pd, S, 8, T.e[D]);
        if (a_anchor && pd == T.e[D] - 1) {
#pragma unroll
          for (int e = 0; e < NE; ++e)
            if (anchor_coord(4 * j + e * STX, e2)) keep |= 1u << (e * NP + k);
        }
      }
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const double pr = pred_k<NP, BND, MODE == 0>(k, cs, wo, wi, k > 0 ? ev[e][k - 1] : 0.0,
                                                     ev[e][k], ev[e][k + 1],
                                                     k + 2 <= NP ? ev[e][k + 2] : 0.0);
        if (MODE == 0) {
          if (!quant_fast(pr, pt[e][k], L, Rd, R, rec[e][k], code[e][k]))
            fail |= 1u << (e * NP + k);
        } else {
          rec[e][k] = dequant(pr, sy[e][k], L, R);
          if (sy[e][k] == 0xFFFFu) fail |= 1u << (e * NP + k);
        }
      }
    }
    if (MODE == 0 && exact) fail = (1u << (NE * NP)) - 1;
    fail &= ~keep;
    if (fail) {  // rare: exact quantiser / outlier values
#pragma unroll
      for (int e = 0; e < NE; ++e) {
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          if (fail & (1u << (e * NP + k))) {
            const int p = (2 * k + 1) * S;
            if (MODE == 0) {
              const int cs = BND ? case_of(p, S, 8, T.e[D]) : case_interior<NP>(k);
              const QS q = fix_point(col + (uint32_t)p * PD4 + 4 * e * STX, S * PD4, cs, wo, wi,
                                     pt[e][k], L.leb, L.e2, L.inv, R);
              rec[e][k] = q.rec;
              code[e][k] = q.sym;
            } else {
              rec[e][k] = outlier_at(O.idx, O.val, O.n,
                                     (D == 0) ? flat_of(T, p, a, 4 * j + e * STX)
                                              : flat_of(T, a, p, 4 * j + e * STX));
            }
          }
        }
      }
    }
    if (BND && keep) {
#pragma unroll
      for (int e = 0; e < NE; ++e)
#pragma unroll
        for (int k = 0; k < NP; ++k)
          if (keep & (1u << (e * NP + k))) {
            rec[e][k] = pt[e][k];
            code[e][k] = (uint32_t)R;
          }
    }
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      if (BND && (2 * k + 1) * S >= ed) continue;
      float qq[4] = {P4[k].x, P4[k].y, P4[k].z, P4[k].w};
#pragma unroll
      for (int e = 0; e < NE; ++e) qq[e * STX] = rec[e][k];
      sts_f4(col + (uint32_t)((2 * k + 1) * S) * PD4, make_float4(qq[0], qq[1], qq[2], qq[3]));
    }
    if (MODE == 0 && a < 8 && j < 8) {
      const bool full = !BND || 4 * j + 3 < min(TX, e2);
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const int p = (2 * k + 1) * S;
        if (BND && p >= ed) continue;
        const uint32_t cr = (D == 0) ? codea(T, p, a, 4 * j) : codea(T, a, p, 4 * j);
        if (STX == 1 && full) {
          sts_u2(cr, make_uint2(code[0][k] | (code[1][k] << 16), code[2][k] | (code[3][k] << 16)));
        } else {
#pragma unroll
          for (int e = 0; e < NE; ++e)
            if (!BND || 4 * j + e * STX < e2) sts_u16(cr + 2 * e * STX, code[e][k]);
        }
      }
    }
  }
}

template <int MODE, bool BND>
DEV void run_pass(const Tile &T, int s, int D, int passed, bool nak, const Lv &L, int R,
                  bool exact, const Out &O) {
  const double wo = nak ? NAK_O : NAT_O, wi = nak ? NAK_I : NAT_I;
  const int stz = (passed & 1) ? s : 2 * s, sty = (passed & 2) ? s : 2 * s;
  const int stx = (passed & 4) ? s : 2 * s;
  if (s == 1) {
    if (D == 2) walk_x<1, MODE, BND>(T, stz, sty, wo, wi, L, R, exact, O);
    else if (D == 0) {
      if (stx == 1) walk_col<1, 0, 1, MODE, BND>(T, sty, wo, wi, L, R, exact, O);
      else walk_col<1, 0, 2, MODE, BND>(T, sty, wo, wi, L, R, exact, O);
    } else {
      if (stx == 1) walk_col<1, 1, 1, MODE, BND>(T, stz, wo, wi, L, R, exact, O);
      else walk_col<1, 1, 2, MODE, BND>(T, stz, wo, wi, L, R, exact, O);
    }
  } else if (s == 2) {
    if (D == 2) walk_x<2, MODE, BND>(T, stz, sty, wo, wi, L, R, exact, O);
    else if (D == 0) {
      if (stx == 2) walk_col<2, 0, 2, MODE, BND>(T, sty, wo, wi, L, R, exact, O);
      else walk_col<2, 0, 4, MODE, BND>(T, sty, wo, wi, L, R, exact, O);
    } else {
      if (stx == 2) walk_col<2, 1, 2, MODE, BND>(T, stz, wo, wi, L, R, exact, O);
      else walk_col<2, 1, 4, MODE, BND>(T, stz, wo, wi, L, R, exact, O);
    }
  } else {
    if (D == 2) walk_x<4, MODE, BND>(T, stz, sty, wo, wi, L, R, exact, O);
    else if (D == 0) {
      if (stx == 4) walk_col<4, 0, 4, MODE, BND>(T, sty, wo, wi, L, R, exact, O);
      else walk_col<4, 0, 8, MODE, BND>(T, sty, wo, wi, L, R, exact, O);
    } else {
      if (stx == 4) walk_col<4, 1, 4, MODE, BND>(T, stz, wo, wi, L, R, exact, O);
      else walk_col<4, 1, 8, MODE, BND>(T, stz, wo, wi, L, R, exact, O);
    }
  }
}

#ifdef T3_PROF
// per-phase cycle counters (tools/microbench/t3_phases.py; build with
// make EXTRA=-DT3_PROF OUT=...): [0] setup [1] TMA wait [2] passes
// [3] epilogue [4] tiles [6 + 3 lv + i] interior pass (lv, i)
static __device__ unsigned long long g_t3_prof[16];
#define T3P_CLOCK(v) const long long v = clock64()
#else
#define T3P_CLOCK(v)
#endif
struct Cfg {  // tuned configuration (per-CTA / per-warp copy)
  Lv lv[3];
  int order[3];
  int nak[3];
  int pc[3];  // interior pass codes (tile3i.cuh pass_codes)
};

template <int MODE, bool BND>
DEV void run_levels(const Tile &T, const Cfg &C, int R, bool exact, const Out &O) {
#pragma unroll 1
  for (int lv = 0; lv < 3; ++lv) {
    const int s = 4 >> lv;
    const Lv L = C.lv[lv];
    int passed = 0;
#pragma unroll 1
    for (int i = 0; i < 3; ++i) {
      const int D = C.order[i];
      run_pass<MODE, BND>(T, s, D, passed, C.nak[D] != 0, L, R, exact, O);
      passed |= 1 << D;
      __syncwarp();

    }
  }
}

#include "tile3i.cuh"

// Interior tiles (closing plane inside the grid on every axis) form the box
// ni[0] x ni[1] x ni[2]; edge tiles are the shell around it (z beyond, then
// y beyond, then x beyond).  t indexes one set, x fastest.
template <bool BND>
DEV int tile_count(const Geo &G) {
  const int ni = G.ni[0] * G.ni[1] * G.ni[2];
  return BND ? G.nt[0] * G.nt[1] * G.nt[2] - ni : ni;
}
template <bool BND>
DEV void tile_origin(const Geo &G, int t, int o[3]) {
  uint32_t tz, ty, tx;
  const uint32_t u = (uint32_t)t;
  if (!BND) {
    const uint32_t r = fdiv(u, G.d_ni2);
    tx = u - r * G.d_ni2.d;
    tz = fdiv(r, G.d_ni1);
    ty = r - tz * G.d_ni1.d;
  } else if (t < G.shell_a) {  // z beyond the interior box
    const uint32_t r = fdiv(u, G.d_nt2);
    tx = u - r * G.d_nt2.d;
    const uint32_t q = fdiv(r, G.d_nt1);
    ty = r - q * G.d_nt1.d;
    tz = (uint32_t)G.ni[0] + q;
  } else if (t < G.shell_a + G.shell_b) {  // y beyond
    const uint32_t v = u - (uint32_t)G.shell_a;
    const uint32_t r = fdiv(v, G.d_nt2);
    tx = v - r * G.d_nt2.d;
    tz = fdiv(r, G.d_wy);
    ty = (uint32_t)G.ni[1] + (r - tz * G.d_wy.d);
  } else {  // x beyond
    const uint32_t v = u - (uint32_t)(G.shell_a + G.shell_b);
    const uint32_t r = fdiv(v, G.d_wx);
    tx = (uint32_t)G.ni[2] + (v - r * G.d_wx.d);
    tz = fdiv(r, G.d_ni1);
    ty = r - tz * G.d_ni1.d;
  }
  o[0] = G.z0 + (int)tz * TZ;
  o[1] = (int)ty * TY;
  o[2] = (int)tx * TX;
}

DEV void tile_of(const Geo &G, int nint, int u, int o[3]) {
  if (u < nint) tile_origin<false>(G, u, o);
  else tile_origin<true>(G, u - nint, o);
}

DEV void tile_init(Tile &T, const Geo &G, const int o[3], bool bnd) {
  for (int a = 0; a < 3; ++a) {
    T.o[a] = o[a];
    T.e[a] = G.ext[a] - o[a];
  }
  T.bnd = bnd;
  T.gs0 = (int64_t)G.ext[1] * G.ext[2];
  T.gs1 = G.ext[2];
}

DEV void cp_async4_zfill(uint32_t sdst, const void *gsrc, bool valid) {
  const int n = valid ? 4 : 0;  // src-size 0 zero-fills
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(sdst), "l"(gsrc), "r"(n)
               : "memory");
}

// Manual staging (no tensor map: the row pitch is not a multiple of 16
// bytes, so neither a 3-D box nor a 16-byte copy can describe a tile row;
// TMA also needs 128-byte aligned destinations, which per-row boxes of the
// pitch-36 layout are not).  Row by row, lane l copies x = l (and 32 + l for
// the closing columns), zero-filling outside the grid / the held planes;
// same smem layout as the TMA box.  The float copy is asynchronous
// (cp.async groups): it is issued for the next tile right after the passes
// and waited for at the next tile's start, like the TMA prefetch.
DEV void stage_rows_f32_issue(uint32_t buf, const float *x, const Geo &G, const int o[3]) {
  const int lane = threadIdx.x & 31;
  const int zl0 = o[0] - G.z0;
  const int64_t nx = G.ext[2], pzs = (int64_t)G.ext[1] * nx;
  const int nzv = min(CZ, G.nzl - zl0), nyv = min(CY, G.ext[1] - o[1]);
  const int nxv = G.ext[2] - o[2];  // columns held from o[2] on
  const float *p = x + (int64_t)zl0 * pzs + (int64_t)o[1] * nx + o[2];
  // columns 0..31 (lane = x).  Rows beyond the grid read a held row with
  // size 0 (zero fill), so every source address stays inside the field.
  {
    const bool vx = lane < nxv;
    const float *pl = p + (vx ? lane : 0);
    uint32_t d = buf + 4u * (uint32_t)lane;
    for (int z = 0; z < CZ; ++z) {
      const bool vz = vx && z < nzv;
      const float *pr = pl + (int64_t)min(z, nzv - 1) * pzs;
#pragma unroll
      for (int y = 0; y < CY; ++y) {
        const bool v = vz && y < nyv;
        cp_async4_zfill(d + 4u * (uint32_t)(y * PX), pr + (int64_t)min(y, nyv - 1) * nx, v);
      }
      d += 4u * PZ;
    }
  }
  // closing column x = 32, lane = row (z, y) of the 81.  Columns 33..35 of
  // the pitch-36 rows are only read by the pad lines of quad 8, whose
  // results are never stored: they are not staged.
  for (int r = lane; r < CZ * CY; r += 32) {
    const int z = r / CY, y = r - z * CY;
    const bool v = nxv > 32 && z < nzv && y < nyv;
    const float *src = p + (int64_t)min(z, nzv - 1) * pzs + (int64_t)min(y, nyv - 1) * nx +
                       (nxv > 32 ? 32 : 0);
    cp_async4_zfill(buf + 4u * (uint32_t)(r * PX + 32), src, v);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}
DEV void stage_rows_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// symbols (2-byte elements: no 2-byte cp.async): plain loads, one z-plane
// (9 rows) in flight per batch, then the stores; the closing column x = 32
// with lane = row.  Columns 33..39 feed only pad lines: not staged.
DEV void stage_rows_u16(uint32_t dst, const uint16_t *sym, const Geo &G, const int o[3]) {
  const int lane = threadIdx.x & 31;
  const int zl0 = o[0] - G.z0;
  const int64_t nx = G.ext[2], pzs = (int64_t)G.ext[1] * nx;
  const int nzv = min(CZ, G.nzl - zl0), nyv = min(CY, G.ext[1] - o[1]);
  const int nxv = G.ext[2] - o[2];
  const uint16_t *p = sym + (int64_t)zl0 * pzs + (int64_t)o[1] * nx + o[2];
  const bool vx = lane < nxv;
  const uint16_t *pl = p + (vx ? lane : 0);
  uint32_t d = dst + 2u * (uint32_t)lane;
  for (int z = 0; z < CZ; ++z) {
    const bool vz = vx && z < nzv;
    const uint16_t *pr = pl + (int64_t)min(z, nzv - 1) * pzs;
    uint32_t a[CY];
#pragma unroll
    for (int y = 0; y < CY; ++y)
      a[y] = (vz && y < nyv) ? __ldg(pr + (int64_t)y * nx) : 0u;
#pragma unroll
    for (int y = 0; y < CY; ++y) sts_u16(d + 2u * (uint32_t)(y * SP), a[y]);
    d += 2u * (uint32_t)(CY * SP);
  }
  for (int r = lane; r < CZ * CY; r += 32) {
    const int z = r / CY, y = r - z * CY;
    const bool v = nxv > 32 && z < nzv && y < nyv;
    const uint32_t w = v ? __ldg(p + (int64_t)z * pzs + (int64_t)y * nx + 32) : 0u;
    sts_u16(dst + 2u * (uint32_t)(r * SP + 32), w);
  }
}

// ---------------------------------------------------------------------------
// tile schedule: when interior tiles (uniform cost) make up most of the
// grid (>= 80%: 512^3 91%, RTM 84%) they are dealt out statically, warp gw
// taking gw, gw + nw, gw + 2 nw, ... (nw warps in the grid); the rest (the
// edge shell: tiles cost 2-3x an interior one, and vary; or every tile of
// an edge-heavy grid such as 33120 x 69 x 69, where the static split
// measured 7% slower) comes from a dynamic queue, one atomic per tile,
// requested when a tile starts and read after its passes so the round trip
// hides under the work.  Each launch uses one slot of a ring; the last warp
// out resets its slot for reuse.
// ---------------------------------------------------------------------------
constexpr int SCHED_SLOTS = 64;
static __device__ unsigned int g_t3_sched[SCHED_SLOTS * 2];

struct Sched {
  unsigned int *q;
  int gw, nw, nint;  // nint: tiles dealt statically (the interior, or none)
};
DEV Sched sched_init(unsigned int *q, int nint, int ntiles) {
  Sched S;
  S.q = q;
  S.gw = (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
  S.nw = (int)(gridDim.x * (blockDim.x >> 5));
  S.nint = ((int64_t)nint * 5 >= (int64_t)ntiles * 4) ? nint : 0;
  return S;
}
DEV int next_tile(const Sched &S) {
  if (S.gw < S.nint) return S.gw;
  int t = 0;
  if ((threadIdx.x & 31) == 0) t = (int)atomicAdd(S.q, 1u);
  return S.nint + __shfl_sync(CSZI_FULL, t, 0);
}
// the tile after t: static while the interior lasts, else a queue ticket
// (bit 31 marks a static successor)
DEV unsigned int ticket_issue(const Sched &S, int t) {
  if (t < S.nint && t + S.nw < S.nint) return 0x80000000u | (unsigned)(t + S.nw);
  return ((threadIdx.x & 31) == 0) ? atomicAdd(S.q, 1u) : 0u;
}
DEV int ticket_read(const Sched &S, unsigned int raw) {
  const unsigned int v = __shfl_sync(CSZI_FULL, raw, 0);
  return (v & 0x80000000u) ? (int)(v & 0x7fffffffu) : S.nint + (int)v;
}
DEV void sched_done(unsigned int *q) {
  if ((threadIdx.x & 31) == 0) {
    __threadfence();
    if (atomicAdd(q + 1, 1u) == gridDim.x * (blockDim.x >> 5) - 1) {
      q[0] = 0;
      q[1] = 0;
      __threadfence();
    }
  }
}

// ---------------------------------------------------------------------------
// Exact-fit edge tiles (tile3i.cuh fit_mask), per kernel: 0 generic walks,
// 1 interior walks + FK walks, 3 one FK walk set for interior and exact-fit
// tiles (fit = 0 on interior tiles).  Measured (r02g, 512^3 / 256x384x384):
// predict 1: +10% / -4%, 3: -2% / -18%; reconstruct 1: -6% / -8%, 3: -2% /
// -7% against 0.  The kernels sit at their register caps, so the choice
// moves the register allocation of the whole kernel, not just edge tiles.
#ifndef T3_FIT_P
#define T3_FIT_P 3
#endif
#ifndef T3_FIT_R
#define T3_FIT_R 1
#endif
template <int MODE, int FM>
DEV void run_tile(const Tile &T, const Cfg &C, int R, bool exact, const Out &O) {
  const int fit = (FM == 0 || !T.bnd) ? 0 : fit_mask(T);
  if ((MODE == 0 && exact) || (T.bnd && (FM == 0 || fit < 0))) {
    run_levels<MODE, true>(T, C, R, exact, O);
  } else if (FM == 3) {
    run_levels_i<MODE, 1>(T, C, R, O, fit);
  } else if (!T.bnd) {
    run_levels_i<MODE, FM == 0 ? 0 : 2>(T, C, R, O);
  } else {
    run_levels_i<MODE, 1>(T, C, R, O, fit);
  }
}

// kernels: persistent warps take tiles from one queue, interior tiles first
// (their code has no edge logic), then the edge shell; one tile at a time; the next tile's TMA load is
// issued as soon as the passes release the staging buffer, so it overlaps
// the epilogue (code store / histogram, or the float store).
// ---------------------------------------------------------------------------
template <int FM>
__global__ void T3P_BOUNDS
    k_t3_predict(const __grid_constant__ CUtensorMap tm, const float *__restrict__ x, Geo G,
                 const cszi_ctl *__restrict__ ctl, uint16_t *__restrict__ sym,
                 u64 *__restrict__ hist, uint32_t *__restrict__ nzmap, int slot) {
  extern __shared__ __align__(128) unsigned char t3_smem[];
  __shared__ Cfg C;
  __shared__ uint64_t mbar[NWP];
  __shared__ uint32_t zero_ws[NWP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int R = G.R;
  unsigned char *sm = align128(t3_smem);
  uint32_t *hs = reinterpret_cast<uint32_t *>(sm + NWP * P_WARP);
  const uint32_t buf = smem_u32(sm + warp * P_WARP);
  const uint32_t codes = buf + BUF_BYTES;
  uint32_t *nzs = reinterpret_cast<uint32_t *>(sm + warp * P_WARP + BUF_BYTES + NCODE * 2);
  const int nint = tile_count<false>(G);
  const int ntiles = nint + tile_count<true>(G);
  unsigned int *q = g_t3_sched + 2 * slot;
  const Sched S = sched_init(q, nint, ntiles);
  int t = next_tile(S);
  if (lane == 0) mbar_init(&mbar[warp]);
  __syncwarp();
  int o[3] = {0, 0, 0};  // origin of tile t (carried from the prefetch)
  if (t < ntiles) {
    tile_of(G, nint, t, o);
    if (G.tma) tile_load<PX, 4>(buf, &tm, G, o, &mbar[warp]);
    else stage_rows_f32_issue(buf, x, G, o);
  }
  if (threadIdx.x < 3) {
    const int i = threadIdx.x;
    const double leb = ctl->level_eb[i];
    C.lv[i].leb = leb;
    C.lv[i].e2 = dmul(2.0, leb);
    C.lv[i].inv = ctl->inv_e2[i];
    C.lv[i].lebs = dsub(fmin(dmul(leb, 1.0 - 0x1p-40), 0x1p100), 0x1p-148);
    C.lv[i].a32 = __fmul_rd(__double2float_rd(leb), 1.0f - 0x1p-23f);
    C.order[i] = ctl->order[i];
    C.nak[i] = ctl->variant[i] == 0;
  }
  if (G.hist_smem)
    for (int i = threadIdx.x; i < 2 * R; i += NTP) hs[i] = 0;
  __syncthreads();  // cfg, hist, mbarrier init visible
  if (threadIdx.x == 0) pass_codes(C.order, C.nak, C.pc);
  __syncthreads();
  const Out O{nullptr, nullptr, 0};
  const bool exact = G.exact != 0;
  const uint32_t rr = (uint32_t)R | ((uint32_t)R << 16);
  const int64_t pz = (int64_t)G.ext[1] * G.ext[2];
  const int py = G.ext[2];
  uint32_t zeros = 0, phase = 0;
#ifdef T3_PROF
  unsigned long long pc[5] = {0, 0, 0, 0, 0};
#endif
  while (t < ntiles) {
    T3P_CLOCK(c0);
    Tile T;
    T.buf = buf;
    T.codes = codes;
    T.syms = 0;
    tile_init(T, G, o, t >= nint);
    // codes default to R (anchors: code 0, predictor.py:414).  Interior
    // tiles write every owned non-anchor code in their passes, so only the
    // four anchors of the tile's (0, 0) row are set; edge tiles reset all.
    if (t >= nint) {
      for (int i = lane; i < NCODE / 8; i += 32) sts_u4(codes + 16u * i, make_uint4(rr, rr, rr, rr));
    } else if (lane < 4) {
      sts_u16(codes + 2u * 8 * lane, (uint32_t)R);
    }
    if (nzmap) {  // non-R words of the tile's rows (epilogue)
      nzs[lane] = 0u;
      nzs[lane + 32] = 0u;
    }
    T3P_CLOCK(c1);
    if (G.tma) {
      mbar_wait(&mbar[warp], phase);
      phase ^= 1;
    } else {
      stage_rows_wait();
    }
    __syncwarp();
    T3P_CLOCK(c2);
    const unsigned int raw = ticket_issue(S, t);
    // edge tiles whose axes all end on the tile boundary or beyond run the
    // interior walks with their end cases (FK); the rest the generic walks
    run_tile<0, FM>(T, C, R, exact, O);
    T3P_CLOCK(c3);
#ifdef T3_PROF
    if (T.bnd && lane == 0) {  // [5] edge tiles, [15] their pass cycles
      atomicAdd(&g_t3_prof[5], 1ull);
      atomicAdd(&g_t3_prof[15], (unsigned long long)(c3 - c2));
    }
#endif
    // staging buffer free: prefetch the next tile
    const int tn = ticket_read(S, raw);
    int on[3] = {0, 0, 0};
    if (tn < ntiles) {
      tile_of(G, nint, tn, on);
      if (G.tma) {
        fence_proxy_async();
        tile_load<PX, 4>(buf, &tm, G, on, &mbar[warp]);
      } else {
        __syncwarp();  // every lane's pass reads of buf precede the copies
        stage_rows_f32_issue(buf, x, G, on);
      }
    }
    // owned codes -> global, histogram (anchors and outliers count as R)
    const int O0 = min(TZ, T.e[0]), O1 = min(TY, T.e[1]), O2 = min(TX, T.e[2]);
    const int64_t gbase = ((int64_t)(o[0] - G.z0) * G.ext[1] + o[1]) * G.ext[2] + o[2];
    if (O0 == TZ && O1 == TY && O2 == TX && (G.ext[2] & 7) == 0) {
#pragma unroll 2
      for (int i = lane; i < TZ * TY * 4; i += 32) {
        const int row = i >> 2, c = i & 3;
        const int z = row >> 3, y = row & 7;
        const uint32_t src = codea(T, z, y, 8 * c);
        const uint2 a = lds_u2(src);
        const uint2 b = lds_u2(src + 8);
        const int64_t g0 = gbase + z * pz + (int64_t)y * py;
        __stcs(reinterpret_cast<uint4 *>(sym + g0 + 8 * c), make_uint4(a.x, a.y, b.x, b.y));
        if (((a.x ^ rr) | (a.y ^ rr) | (b.x ^ rr) | (b.y ^ rr)) == 0) {
          zeros += 8;
          continue;
        }
        // non-R bit per code (outliers included) for the sparse encoder: the
        // map is zeroed beforehand and only groups holding a non-R code (~5%
        // on smooth fields) OR their byte into the row's word
        // the four lanes of a row own one byte each of its word: plain
        // byte stores (shared atomics here cost ~15 us over the launch)
        if (nzmap)
          reinterpret_cast<uint8_t *>(nzs)[4 * row + c] =
              (uint8_t)(ne_r2(a.x, rr) | (ne_r2(a.y, rr) << 2) | (ne_r2(b.x, rr) << 4) |
                        (ne_r2(b.y, rr) << 6));
        const uint32_t w[4] = {a.x, a.y, b.x, b.y};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          if (w[h] == rr) {
            zeros += 2;
          } else {
#pragma unroll
            for (int half = 0; half < 2; ++half) {
              const uint32_t sy = half ? (w[h] >> 16) : (w[h] & 0xffffu);
              if (sy == (uint32_t)R || sy == 0) zeros++;
              else if (G.hist_smem) atomicAdd(&hs[sy], 1u);
              else atomicAdd(&hist[sy], 1ull);
            }
          }
        }
      }
      if (nzmap) {  // rows with a non-R code -> the zeroed global map
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = lane + 32 * h;
          const uint32_t wd = nzs[row];
          if (wd) nzmap[(gbase + (row >> 3) * pz + (int64_t)(row & 7) * py) >> 5] = wd;
        }
      }
    } else if (!nzmap) {
      // (rows not 16-byte aligned, e.g. nx = 235 / 69) two rows per step:
      // half-warp h takes row (z, y0 + h), lane pair x = 2 (lane % 16) + {0, 1};
      // one 4-byte store when the pair is 4-byte aligned in global memory
      // (the row base parity), two 2-byte stores otherwise
      const int h = lane >> 4, xl = 2 * (lane & 15);
      const bool a0 = xl < O2, a1 = xl + 1 < O2;
      for (int z = 0; z < O0; ++z) {
        const int64_t gz = gbase + (int64_t)z * pz + xl;
        for (int y0 = 0; y0 < O1; y0 += 2) {
          const int y = y0 + h;
          const bool v0 = a0 && y < O1, v1 = a1 && y < O1;
          const uint32_t w = v0 ? lds_u32(codea(T, z, y, xl)) : rr;
          const uint32_t s0 = w & 0xffffu, s1 = w >> 16;
          uint16_t *g = sym + gz + (int64_t)y * py;
          if (v1 && !(reinterpret_cast<uintptr_t>(g) & 3)) {
            *reinterpret_cast<uint32_t *>(g) = w;
          } else {
            if (v0) g[0] = (uint16_t)s0;
            if (v1) g[1] = (uint16_t)s1;
          }
          const bool o0 = v0 && s0 != (uint32_t)R && s0 != 0;
          const bool o1 = v1 && s1 != (uint32_t)R && s1 != 0;
          zeros += (uint32_t)(v0 && !o0) + (uint32_t)(v1 && !o1);
          if (__any_sync(CSZI_FULL, o0 || o1)) {
            if (o0) {
              if (G.hist_smem) atomicAdd(&hs[s0], 1u);
              else atomicAdd(&hist[s0], 1ull);
            }
            if (o1) {
              if (G.hist_smem) atomicAdd(&hs[s1], 1u);
              else atomicAdd(&hist[s1], 1ull);
            }
          }
        }
      }
    } else {
      // row by row, lane = x: coalesced 2-byte stores, pointers stepped per
      // row; R / outlier codes counted per lane, the histogram atomics only
      // run for rows that hold another code
      const bool act = lane < O2;
      uint16_t *gz = sym + gbase + lane;
      uint32_t cz = codea(T, 0, 0, lane);
      for (int z = 0; z < O0; ++z) {
        uint16_t *gy = gz;
        uint32_t cy = cz;
        for (int y = 0; y < O1; ++y) {
          const uint32_t sy = act ? lds_u16(cy) : (uint32_t)R;
          if (act) *gy = (uint16_t)sy;
          if (nzmap) {  // O2 == 32 whenever nzmap is set
            const uint32_t wd = __ballot_sync(CSZI_FULL, sy != (uint32_t)R);
            if (lane == 0 && wd) nzmap[(gy - sym) >> 5] = wd;
          }
          const bool other = act && sy != (uint32_t)R && sy != 0;
          zeros += (uint32_t)(act && !other);
          if (__any_sync(CSZI_FULL, other) && other) {
            if (G.hist_smem) atomicAdd(&hs[sy], 1u);
            else atomicAdd(&hist[sy], 1ull);
          }
          gy += py;
          cy += 2u * CP;
        }
        gz += pz;
        cz += 2u * TY * CP;
      }
    }
    __syncwarp();  // codes read before the next tile resets them
    o[0] = on[0];
    o[1] = on[1];
    o[2] = on[2];
#ifdef T3_PROF
    pc[0] += c1 - c0;
    pc[1] += c2 - c1;
    pc[2] += c3 - c2;
    pc[3] += clock64() - c3;
    pc[4] += 1;
#endif
    t = tn;
  }
#ifdef T3_PROF
  if (lane == 0)
    for (int i = 0; i < 5; ++i) atomicAdd(&g_t3_prof[i], pc[i]);
#endif
  sched_done(q);
  zeros = warp_sum(zeros);
  if (lane == 0) zero_ws[warp] = zeros;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t z = 0;
    for (int w = 0; w < NWP; ++w) z += zero_ws[w];
    if (z) atomicAdd(&hist[R], (u64)z);
  }
  if (G.hist_smem)
    for (int i = threadIdx.x; i < 2 * R; i += NTP)
      if (hs[i]) atomicAdd(&hist[i], (u64)hs[i]);
}

// anchor value lane (< 20) seeds on an interior tile at origin o: z, y in
// {0, 8}, x in {0, 8, 16, 24, 32} of the closed tile (lattice row-major)
DEV float anchor_i(const float *anchors, const Geo &G, const int o[3], int lane) {
  if (lane >= 20) return 0.f;
  const int iz = lane / 10, iy = (lane / 5) & 1, ix = lane % 5;
  const int64_t kz = o[0] / 8 + iz, ky = o[1] / 8 + iy, kx = o[2] / 8 + ix;
  return __ldg(anchors + (kz * G.na1 + ky) * G.na2 + kx);
}

template <int FM>
__global__ void __launch_bounds__(NT, MINB_R)
    k_t3_reconstruct(const __grid_constant__ CUtensorMap tm, const uint16_t *__restrict__ sym,
                     const float *__restrict__ anchors, const u64 *out_idx,
                     const float *out_val, u64 n_out, const u64 *nout_dev, Geo G, LevelCfg lc,
                     float *__restrict__ yout, int slot) {
  extern __shared__ __align__(128) unsigned char t3_smem[];
  __shared__ Cfg C;
  __shared__ uint64_t mbar[NW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int R = G.R;
  unsigned char *sm = align128(t3_smem);
  const uint32_t syms = smem_u32(sm + warp * R_WARP);
  const uint32_t buf = syms + SYM_BYTES;
  const int nint = tile_count<false>(G);
  const int ntiles = nint + tile_count<true>(G);
  unsigned int *q = g_t3_sched + 2 * slot;
  const Sched S = sched_init(q, nint, ntiles);
  int t = next_tile(S);
  if (lane == 0) mbar_init(&mbar[warp]);
  __syncwarp();
  int o[3] = {0, 0, 0};  // origin of tile t (carried from the prefetch)
  float apre = 0.f;      // lane < 20: interior anchor value of tile t
  if (t < ntiles) {
    tile_of(G, nint, t, o);
    if (G.tma) tile_load<SP, 2>(syms, &tm, G, o, &mbar[warp]);
    if (t < nint) apre = anchor_i(anchors, G, o, lane);
  }
  if (threadIdx.x < 3) {
    const int i = threadIdx.x;
    const double leb = lc.leb[i];
    C.lv[i].leb = leb;
    C.lv[i].e2 = dmul(2.0, leb);
    C.lv[i].inv = 0.0;
    C.lv[i].lebs = 0.0;
    C.lv[i].a32 = 0.f;
    C.order[i] = lc.order[i];
    C.nak[i] = lc.variant[i] == 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) pass_codes(C.order, C.nak, C.pc);
  __syncthreads();
  const Out O{out_idx, out_val, nout_dev ? *nout_dev : n_out};
  const int64_t pz = (int64_t)G.ext[1] * G.ext[2];
  const int py = G.ext[2];
  uint32_t phase = 0;
  while (t < ntiles) {
    Tile T;
    T.buf = buf;
    T.codes = 0;
    T.syms = syms;
    tile_init(T, G, o, t >= nint);
    // edge tiles: zero the buffer so that weight-0 terms of missing
    // neighbours read finite values (interior tiles read only computed ones)
    if (T.bnd)
      for (int i = lane; i < NBUF / 4; i += 32) sts_f4(buf + 16u * i, make_float4(0.f, 0.f, 0.f, 0.f));
    __syncwarp();
    // seed the anchors of the closed tile (multiples of 8, plus ext - 1)
    if (!T.bnd) {
      // interior: z, y in {0, 8}, x in {0, 8, 16, 24, 32}; no closing anchors.
      // The values were loaded when this tile was prefetched (apre).
      if (lane < 20) sts_f(bufa(T, 8 * (lane / 10), 8 * ((lane / 5) & 1), 8 * (lane % 5)), apre);
    } else {
      int az[3], ay[3], ax[6];
      const int nz = anchor_axis_local<CZ, 8>(T.e[0], az);
      const int ny = anchor_axis_local<CY, 8>(T.e[1], ay);
      const int nx = anchor_axis_local<CX, 8>(T.e[2], ax);
      for (int i = lane; i < nz * ny * nx; i += 32) {
        const int iz = i / (ny * nx), r = i - iz * ny * nx, iy = r / nx, ix = r - iy * nx;
        const int lz = az[iz], ly = ay[iy], lx = ax[ix];
        const int gz = o[0] + lz, gy = o[1] + ly, gx = o[2] + lx;
        const int64_t kz = (gz % 8 == 0) ? gz / 8 : (G.ext[0] - 1) / 8 + 1;
        const int64_t ky = (gy % 8 == 0) ? gy / 8 : (G.ext[1] - 1) / 8 + 1;
        const int64_t kx = (gx % 8 == 0) ? gx / 8 : (G.ext[2] - 1) / 8 + 1;
        sts_f(bufa(T, lz, ly, lx), __ldg(anchors + (kz * G.na1 + ky) * G.na2 + kx));
      }
    }
    if (G.tma) {
      mbar_wait(&mbar[warp], phase);
      phase ^= 1;
    } else {
      stage_rows_u16(syms, sym, G, o);
    }
    __syncwarp();
    const unsigned int raw = ticket_issue(S, t);
    run_tile<1, FM>(T, C, R, false, O);
    const int tn = ticket_read(S, raw);
    int on[3] = {0, 0, 0};
    if (tn < ntiles) {
      tile_of(G, nint, tn, on);
      if (G.tma) {
        fence_proxy_async();
        tile_load<SP, 2>(syms, &tm, G, on, &mbar[warp]);
      }
      if (tn < nint) apre = anchor_i(anchors, G, on, lane);
    }
    const int O0 = min(TZ, T.e[0]), O1 = min(TY, T.e[1]), O2 = min(TX, T.e[2]);
    const int64_t gbase = ((int64_t)(o[0] - G.z0) * G.ext[1] + o[1]) * G.ext[2] + o[2];
    if (O0 == TZ && O1 == TY && O2 == TX && (G.ext[2] & 3) == 0) {
      // lane = (quad q = lane % 8, row y0 = lane / 8 and y0 + 4), z = 0..7
      const int q4 = 4 * (lane & 7), y0 = lane >> 3;
      const uint32_t s0 = bufa(T, 0, y0, q4);
      float *d0 = yout + gbase + (int64_t)y0 * py + q4;
#pragma unroll
      for (int z = 0; z < TZ; ++z) {
#pragma unroll
        for (int h = 0; h < 2; ++h)
          __stcs(reinterpret_cast<float4 *>(d0 + 4 * h * py),
                 lds_f4(s0 + 4u * (uint32_t)(z * PZ + 4 * h * PX)));
        d0 += pz;
      }
    } else if (lane < O2) {  // row by row, lane = x, pointers stepped per row
      float *dz = yout + gbase + lane;
      uint32_t sz = bufa(T, 0, 0, lane);
      for (int z = 0; z < O0; ++z) {
        float *dy = dz;
        uint32_t sy = sz;
        for (int y = 0; y < O1; ++y) {
          __stcs(dy, lds_f(sy));
          dy += py;
          sy += 4u * PX;
        }
        dz += pz;
        sz += 4u * PZ;
      }
    }
    __syncwarp();  // buf read before the next tile's anchors land
    o[0] = on[0];
    o[1] = on[1];
    o[2] = on[2];
    t = tn;
  }
  sched_done(q);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (EncodeTiledFn) nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// 3-D tensor map over a [nz][ny][nx] array; box (bx, 9, 9).  False when the
// layout violates TMA's 16-byte stride / address rules (manual staging).
static bool make_tmap(CUtensorMap *tm, const void *base, CUtensorMapDataType dt, int esz,
                      int64_t nx, int64_t ny, int64_t nz, int bx) {
  memset(tm, 0, sizeof(*tm));
  if (getenv("CSZI_NO_TMA")) return false;
  EncodeTiledFn fn = encode_fn();
  if (!fn || (reinterpret_cast<uintptr_t>(base) & 15) || ((nx * esz) & 15) || nx < 1 || ny < 1 ||
      nz < 1 || nx >= (1ll << 32) || ny >= (1ll << 32) || nz >= (1ll << 32))
    return false;
  const cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
  const cuuint64_t strides[2] = {(cuuint64_t)(nx * esz), (cuuint64_t)(nx * ny * esz)};
  const cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)CY, (cuuint32_t)CZ};
  const cuuint32_t es[3] = {1, 1, 1};
  return fn(tm, dt, 3, const_cast<void *>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// resident CTAs x SMs, capped by the tile count
static unsigned persistent_grid(const void *k, size_t smem, int64_t ntiles, int nw = NW) {
  const int sms = sm_count(), per = occupancy(k, nw * 32, smem);
  const int64_t need = (ntiles + nw - 1) / nw;
  const int64_t cap = (int64_t)per * sms;
  return (unsigned)(need < cap ? need : cap);
}

static int sched_slot() {
  static std::atomic<unsigned> seq{0};
  return (int)(seq.fetch_add(1) % SCHED_SLOTS);
}

static bool t3_geo(const cszi_geom *g, int32_t radius, Geo &G) {
  if (g->rank != 3 || g->stride != 8 || g->tile[0] != TZ || g->tile[1] != TY ||
      g->tile[2] != TX)
    return false;
  for (int a = 0; a < 3; ++a) {
    if (g->ext[a] < 1 || g->ext[a] > (1 << 30)) return false;
    G.ext[a] = (int)g->ext[a];
  }
  G.z0 = 0;
  G.nzl = G.ext[0];
  int64_t zown = g->ext[0];
  if (g->slab[1] > g->slab[0]) {
    if (g->slab[0] % TZ) return false;
    G.z0 = (int)g->slab[0];
    const int64_t zend = (g->slab[1] + 1 < g->ext[0]) ? g->slab[1] + 1 : g->ext[0];
    G.nzl = (int)(zend - g->slab[0]);
    zown = g->slab[1] - g->slab[0];
  }
  G.nt[0] = (int)((zown + TZ - 1) / TZ);
  G.nt[1] = (G.ext[1] + TY - 1) / TY;
  G.nt[2] = (G.ext[2] + TX - 1) / TX;
  {
    const int T3[3] = {TZ, TY, TX};
    const int64_t first[3] = {G.z0, 0, 0};
    for (int a = 0; a < 3; ++a) {
      // tiles whose closing plane o + T <= ext - 1
      const int64_t lim = (int64_t)G.ext[a] - 1 - first[a];
      int64_t n = lim >= T3[a] ? lim / T3[a] : 0;
      G.ni[a] = (int)(n < G.nt[a] ? n : G.nt[a]);
    }
  }
  if ((int64_t)G.nt[0] * G.nt[1] * G.nt[2] >= 0x7fffffffll) return false;  // int tile ids
  // flat indices of the outlier lookup and of planes are int64; the
  // in-kernel (z * gs0 + ...) products need ext[1] * ext[2] < 2^62: fine.
  G.d_ni2 = make_fdiv((uint32_t)G.ni[2]);
  G.d_ni1 = make_fdiv((uint32_t)G.ni[1]);
  G.d_nt2 = make_fdiv((uint32_t)G.nt[2]);
  G.d_nt1 = make_fdiv((uint32_t)G.nt[1]);
  G.d_wy = make_fdiv((uint32_t)(G.nt[1] - G.ni[1]));
  G.d_wx = make_fdiv((uint32_t)(G.nt[2] - G.ni[2]));
  G.shell_a = (G.nt[0] - G.ni[0]) * G.nt[1] * G.nt[2];
  G.shell_b = G.ni[0] * (G.nt[1] - G.ni[1]) * G.nt[2];
  G.R = radius;
  G.hist_smem = (2 * radius <= 2048) ? 1 : 0;
  G.tma = 0;
  G.exact = 0;
  auto na = [](int64_t e) { return (e - 1) / 8 + 1 + (((e - 1) % 8) ? 1 : 0); };
  G.na1 = na(g->ext[1]);
  G.na2 = na(g->ext[2]);
  return true;
}

template <int FM>
static int predict_t3_impl(const float *x, const cszi_geom *g, int32_t radius,
                           const cszi_ctl *ctl, uint16_t *sym, u64 *hist, bool exact,
                           cudaStream_t st, uint32_t *nzmap, bool *nz_done) {
  Geo G;
  if (!t3_geo(g, radius, G)) return CSZI_E_UNSUPPORTED;
  // the non-R bitmap needs every tile row to be one aligned 32-code word
  if (G.ext[2] % 32 != 0 || getenv("CSZI_NO_NZ")) nzmap = nullptr;
  if (nz_done) *nz_done = nzmap != nullptr;
  if (nzmap) cudaMemsetAsync(nzmap, 0, (size_t)G.nzl * G.ext[1] * G.ext[2] / 8, st);
  G.exact = exact ? 1 : 0;
  CUtensorMap tm;
  G.tma = make_tmap(&tm, x, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, G.ext[2], G.ext[1], G.nzl, PX)
              ? 1
              : 0;
  const int64_t nall = (int64_t)G.nt[0] * G.nt[1] * G.nt[2];
  const size_t smem =
      128 + (size_t)NWP * P_WARP + (G.hist_smem ? sizeof(uint32_t) * 2 * radius : 0);
  ensure_smem((const void *)k_t3_predict<FM>, smem);
  const unsigned grid = persistent_grid((const void *)k_t3_predict<FM>, smem, nall, NWP);
  k_t3_predict<FM><<<grid, NTP, smem, st>>>(tm, x, G, ctl, sym, hist, nzmap, sched_slot());
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

template <int FM>
static int recon_t3_impl(const uint16_t *sym, const float *anchors, const u64 *oidx,
                         const float *oval, u64 nout, const u64 *nout_dev, const cszi_geom *g,
                         int32_t radius, const LevelCfg &lc, float *y, cudaStream_t st) {
  Geo G;
  if (!t3_geo(g, radius, G) || lc.nlev != 3) return CSZI_E_UNSUPPORTED;
  CUtensorMap tm;
  G.tma = make_tmap(&tm, sym, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, G.ext[2], G.ext[1], G.nzl, SP)
              ? 1
              : 0;
  const int64_t nall = (int64_t)G.nt[0] * G.nt[1] * G.nt[2];
  const size_t smem = 128 + (size_t)NW * R_WARP;
  ensure_smem((const void *)k_t3_reconstruct<FM>, smem);
  const unsigned grid = persistent_grid((const void *)k_t3_reconstruct<FM>, smem, nall);
  k_t3_reconstruct<FM><<<grid, NT, smem, st>>>(tm, sym, anchors, oidx, oval, nout, nout_dev, G, lc,
                                           y, sched_slot());
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

#ifdef T3_PROF
// read and reset this translation unit's profile counters
static void t3_prof_take(unsigned long long *out) {
  unsigned long long v[16];
  cudaMemcpyFromSymbol(v, g_t3_prof, sizeof(v));
  for (int i = 0; i < 16; ++i) out[i] += v[i];
  const unsigned long long z[16] = {0};
  cudaMemcpyToSymbol(g_t3_prof, z, sizeof(z));
}
void t3_prof_fit(unsigned long long *out);
#endif

// The kernels come in two builds (run_tile's FM): FM = 0 runs every edge
// tile through the generic walks, the fit build (T3_FIT_P / T3_FIT_R, in
// t3f.cu) runs exact-fit edge tiles through the interior walks.  Each build
// is its own register allocation: the fit build is faster where exact-fit
// tiles are common (512^3: predict -2%, reconstruct -6%) and slower where
// there are none (449 x 449 x 235: +3%, +8%), so the launch picks per grid.
int launch_predict_t3_fit(const float *x, const cszi_geom *g, int32_t radius,
                          const cszi_ctl *ctl, uint16_t *sym, u64 *hist, bool exact,
                          cudaStream_t st, uint32_t *nzmap, bool *nz_done);
int launch_recon_t3_fit(const uint16_t *sym, const float *anchors, const u64 *oidx,
                        const float *oval, u64 nout, const u64 *nout_dev, const cszi_geom *g,
                        int32_t radius, const LevelCfg &lc, float *y, cudaStream_t st);

#ifdef T3_FIT_TU
int launch_predict_t3_fit(const float *x, const cszi_geom *g, int32_t radius,
                          const cszi_ctl *ctl, uint16_t *sym, u64 *hist, bool exact,
                          cudaStream_t st, uint32_t *nzmap, bool *nz_done) {
  return predict_t3_impl<T3_FIT_P>(x, g, radius, ctl, sym, hist, exact, st, nzmap, nz_done);
}
int launch_recon_t3_fit(const uint16_t *sym, const float *anchors, const u64 *oidx,
                        const float *oval, u64 nout, const u64 *nout_dev, const cszi_geom *g,
                        int32_t radius, const LevelCfg &lc, float *y, cudaStream_t st) {
  return recon_t3_impl<T3_FIT_R>(sym, anchors, oidx, oval, nout, nout_dev, g, radius, lc, y, st);
}
#ifdef T3_PROF
void t3_prof_fit(unsigned long long *out) { t3_prof_take(out); }
#endif
#else
// exact-fit edge tiles (every axis closed or ending on the tile boundary, at
// least one of the latter) against the other edge tiles (some axis ends
// inside the tile)
static bool t3_fit_pays(const cszi_geom *g, int32_t radius) {
  Geo G;
  if (!t3_geo(g, radius, G)) return false;
  const int T3[3] = {TZ, TY, TX};
  int64_t all = 1, inner = 1, closed = 1;
  for (int a = 0; a < 3; ++a) {
    const int64_t o_last = (a == 0 ? G.z0 : 0) + (int64_t)(G.nt[a] - 1) * T3[a];
    const bool fit = G.nt[a] > G.ni[a] && G.ext[a] - o_last == T3[a];
    all *= G.nt[a];
    inner *= G.ni[a] + (fit ? 1 : 0);
    closed *= G.ni[a];
  }
  const int64_t nfit = inner - closed, npart = all - inner;
  return nfit > 0 && nfit >= npart;
}

int launch_predict_t3(const float *x, const cszi_geom *g, int32_t radius, const cszi_ctl *ctl,
                      uint16_t *sym, u64 *hist, bool exact, cudaStream_t st, uint32_t *nzmap,
                      bool *nz_done) {
  if (!exact && t3_fit_pays(g, radius))
    return launch_predict_t3_fit(x, g, radius, ctl, sym, hist, exact, st, nzmap, nz_done);
  return predict_t3_impl<0>(x, g, radius, ctl, sym, hist, exact, st, nzmap, nz_done);
}

int launch_recon_t3(const uint16_t *sym, const float *anchors, const u64 *oidx,
                    const float *oval, u64 nout, const u64 *nout_dev, const cszi_geom *g,
                    int32_t radius, const LevelCfg &lc, float *y, cudaStream_t st) {
  if (t3_fit_pays(g, radius))
    return launch_recon_t3_fit(sym, anchors, oidx, oval, nout, nout_dev, g, radius, lc, y, st);
  return recon_t3_impl<0>(sym, anchors, oidx, oval, nout, nout_dev, g, radius, lc, y, st);
}
#endif

}  // namespace t3
}  // namespace cszi

#if defined(T3_PROF) && !defined(T3_FIT_TU)
extern "C" int cszi_t3_prof(unsigned long long *out) {  // read and reset (both builds)
  for (int i = 0; i < 16; ++i) out[i] = 0;
  cszi::t3::t3_prof_take(out);
  cszi::t3::t3_prof_fit(out);
  return 0;
}
#endif
