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
#include <algorithm>

#include "common.cuh"
#include "interp_common.cuh"

namespace cszi {

struct InterpParams {
  int64_t ext[3];
  int64_t tile[3];
  int64_t stride;
  int32_t rank;
  int32_t radius;
  int32_t nb[3];  // blocks per axis (axis 0: over the owned planes of a slab)
  int32_t z0;     // global z of local plane 0 (slab shards), else 0
};


// Uniform description of one (level, dimension) pass inside a CTA block.
// Work item = one segment of up to SEG consecutive pass points on one line
// along d; items are numbered segment-major so the 32 lanes of a warp sit
// on 32 different lines at the same position along d, which makes the
// spline case (a function of the position along d only) warp-uniform.
struct Pass {
  int d, s;
  int a1, a2;        // the two other axes (a1 slower)
  int st1, st2;      // lattice steps on a1, a2
  int cnt2;          // lattice count on a2
  int nlines;
  int npts;          // pass points per line
  int seg, nseg;     // points per segment, segments per line
  int pd_pitch;      // smem element distance between consecutive positions on d
  int p1_, p2_;      // smem pitch of a1, a2
  int tile;          // super-chunk tile on d
  int od, ext_d;     // block origin / grid extent on d
  int bd;            // owned extent on d
  int o1, o2, e1, e2, b1, b2;
  int maxeven;       // largest even-position index 2j*s inside the closed block
  int c_d, c_1, c_2;         // strides of the owned-code array per axis
  int64_t g_d, g_1, g_2;     // strides of the flat grid index per axis
  float r_nl, r_c2;
};

template <int PX, int PY, int BY, int BX>
DEV Pass make_pass(int d, int s, int passed, const int L[3], const int B[3],
                   const int o[3], const int ext[3], const int tile[3]) {
  Pass p;
  const int cstr[3] = {BY * BX, BX, 1};
  const int64_t gstr[3] = {(int64_t)ext[1] * ext[2], (int64_t)ext[2], 1};
  p.d = d;
  p.s = s;
  p.a1 = (d == 0) ? 1 : 0;
  p.a2 = (d == 2) ? 1 : 2;
  const int pitch[3] = {PY * PX, PX, 1};
  int st[3], cnt[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    st[a] = (a == d || !((passed >> a) & 1)) ? 2 * s : s;
    cnt[a] = (L[a] - 1) / st[a] + 1;
  }
  p.st1 = st[p.a1];
  p.st2 = st[p.a2];
  p.cnt2 = cnt[p.a2];
  p.nlines = cnt[p.a1] * cnt[p.a2];
  p.npts = (L[d] - 1 >= s) ? (L[d] - 1 - s) / (2 * s) + 1 : 0;
  const int pt = max(tile[d] / (2 * s), 1);
  p.seg = min(pt, 4);
  p.nseg = (p.npts + p.seg - 1) / p.seg;
  p.pd_pitch = pitch[d];
  p.p1_ = pitch[p.a1];
  p.p2_ = pitch[p.a2];
  p.tile = tile[d];
  p.od = o[d];
  p.bd = B[d];
  p.ext_d = ext[d];
  p.o1 = o[p.a1];
  p.o2 = o[p.a2];
  p.e1 = ext[p.a1];
  p.e2 = ext[p.a2];
  p.b1 = B[p.a1];
  p.b2 = B[p.a2];
  p.maxeven = (L[d] - 1) / (2 * s);
  p.c_d = cstr[d];
  p.c_1 = cstr[p.a1];
  p.c_2 = cstr[p.a2];
  p.g_d = gstr[d];
  p.g_1 = gstr[p.a1];
  p.g_2 = gstr[p.a2];
  p.r_nl = 1.0f / (float)max(p.nlines, 1);
  p.r_c2 = 1.0f / (float)max(p.cnt2, 1);
  return p;
}


// Run every pass of every level on the CTA's closed block held in `buf`.
// MODE 0 (compress): buf holds originals; writes recon + symbols (owned).
// MODE 1 (decompress): buf holds anchors; symbols come from `csym`.
template <int MODE, int BZ, int BY, int BX, int NT, bool EXACT>
DEV void run_levels(float *buf, uint16_t *codes, const uint16_t *csym, const LevelCfg &cfg,
                    const int L[3], const int o[3], const int ext[3], const int tile[3], int S,
                    int rank, int R, const u64 *out_idx, const float *out_val, u64 n_out,
                    const int64_t gext1, const int64_t gext2) {
  constexpr int CZ = BZ == 1 ? 1 : BZ + 1, CY = BY == 1 ? 1 : BY + 1, CX = BX + 1;
  constexpr int PX = CX, PY = CY;
  const int B[3] = {BZ, BY, BX};
  const int tid = threadIdx.x;
  for (int lv = 0; lv < cfg.nlev; ++lv) {
    const int s = S >> (lv + 1);
    const double leb = cfg.leb[lv];
    const double e2 = dmul(2.0, leb);
    const double inv = cfg.inv[lv];
    int passed = 0;
    for (int oi = 0; oi < rank; ++oi) {
      const int d = cfg.order[oi];
      if (s < ext[d]) {
        const Pass ps = make_pass<PX, PY, BY, BX>(d, s, passed, L, B, o, ext, tile);
        const double wo = cfg.variant[d] ? NAT_O : NAK_O;
        const double wi = cfg.variant[d] ? NAT_I : NAK_I;
        const int items = ps.nlines * ps.nseg;
        const int es = 2 * s * ps.pd_pitch;  // smem distance between even positions
        for (int it = tid; it < items; it += NT) {
          const int sg = fdiv(it, ps.nlines, ps.r_nl);
          const int line = it - sg * ps.nlines;
          const int i1 = fdiv(line, ps.cnt2, ps.r_c2);
          const int i2 = line - i1 * ps.cnt2;
          const int l1 = i1 * ps.st1, l2 = i2 * ps.st2;
          const int g1 = ps.o1 + l1, g2 = ps.o2 + l2;
          const bool line_anchor = (((g1 & (S - 1)) == 0) || g1 == ps.e1 - 1) &&
                                   (((g2 & (S - 1)) == 0) || g2 == ps.e2 - 1);
          const bool line_owned = l1 < ps.b1 && l2 < ps.b2;
          float *base = buf + l1 * ps.p1_ + l2 * ps.p2_;
          const int k0 = sg * ps.seg;
          // window over even positions j = k-1 .. k+2 (value at 2*j*s)
          double vm3 = (k0 >= 1) ? f2d(base[(k0 - 1) * es]) : 0.0;
          double vm1 = f2d(base[k0 * es]);
          double vp1 = (k0 + 1 <= ps.maxeven) ? f2d(base[(k0 + 1) * es]) : 0.0;
          double vp3 = (k0 + 2 <= ps.maxeven) ? f2d(base[(k0 + 2) * es]) : 0.0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int k = k0 + j;
            if (j < ps.seg && k < ps.npts) {
              const int pdl = (2 * k + 1) * s;
              const int pd = ps.od + pdl;
              if (!(line_anchor && pd == ps.ext_d - 1)) {
                const int cs = case_of(pd, s, ps.tile, ps.ext_d);
                const double pred = spline4(cs, wo, wi, vm3, vm1, vp1, vp3);
                float *pp = base + pdl * ps.pd_pitch;
                if (MODE == 0) {
                  float rec;
                  const uint32_t sy = quantize<EXACT>(pred, *pp, leb, e2, inv, R, rec);
                  *pp = rec;
                  if (line_owned && pdl < ps.bd)
                    codes[pdl * ps.c_d + l1 * ps.c_1 + l2 * ps.c_2] = (uint16_t)sy;
                } else {
                  const uint32_t code = csym[pp - buf];
                  float v;
                  if (code == 0xFFFFu) {
                    v = outlier_value(out_idx, out_val, n_out,
                                      (u64)(pd * ps.g_d + g1 * ps.g_1 + g2 * ps.g_2));
                  } else {
                    const int q = (int)code - R;
                    const double qd =
                        dsub(__hiloint2double(0x43300000, (int)((uint32_t)q ^ 0x80000000u)),
                             4503601774854144.0);  // 2^52 + 2^31
                    v = __double2float_rn(dadd(pred, dmul(e2, qd)));
                  }
                  *pp = v;
                }
              }
              // slide the window by one even position
              vm3 = vm1;
              vm1 = vp1;
              vp1 = vp3;
              vp3 = (k + 3 <= ps.maxeven) ? f2d(base[(k + 3) * es]) : 0.0;
            }
          }
        }
      }
      passed |= 1 << d;
      __syncthreads();
    }
  }
}

}  // namespace cszi
#include "interp_fast.cuh"
namespace cszi {

// ---------------------------------------------------------------------------
// compress: predict + quantize + histogram
// ---------------------------------------------------------------------------
template <int BZ, int BY, int BX, int NT, bool EXACT>
__global__ void __launch_bounds__(NT, 3) k_predict(const float *__restrict__ x, InterpParams P,
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
  const int o[3] = {bz * BZ, by * BY, bx * BX};
  const int ext[3] = {(int)P.ext[0], (int)P.ext[1], (int)P.ext[2]};
  const int tile[3] = {(int)P.tile[0], (int)P.tile[1], (int)P.tile[2]};
  int L[3];
  L[0] = min(CZ, ext[0] - o[0]);
  L[1] = min(CY, ext[1] - o[1]);
  L[2] = min(CX, ext[2] - o[2]);
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
  const int warp = tid >> 5, lane = tid & 31;
  const bool fast_path = false;
  {
    for (int row = warp; row < L[0] * L[1]; row += NT / 32) {
      const int lz = row / L[1], ly = row - lz * L[1];
      const float *src =
          x + ((int64_t)(o[0] + lz) * ext[1] + (o[1] + ly)) * (int64_t)ext[2] + o[2];
      float *dst = buf + (lz * PY + ly) * PX;
      for (int lx = lane; lx < L[2]; lx += 32) dst[lx] = __ldg(src + lx);
    }
  }
  for (int i = tid; i < BZ * BY * BX; i += NT) codes[i] = (uint16_t)R;
  __syncthreads();

  if (!fast_path)
    run_levels<0, BZ, BY, BX, NT, EXACT>(buf, codes, nullptr, cfg, L, o, ext, tile,
                                         (int)P.stride, P.rank, R, nullptr, nullptr, 0,
                                         P.ext[1], P.ext[2]);

  // codes out (coalesced rows) + histogram; outliers (symbol 0) count as R
  uint32_t zeros = 0;
  for (int row = warp; !fast_path && row < O0 * O1; row += NT / 32) {
    const int lz = row / O1, ly = row - lz * O1;
    uint16_t *dst = sym + ((int64_t)(o[0] + lz) * ext[1] + (o[1] + ly)) * (int64_t)ext[2] + o[2];
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

DEV int64_t anchor_index_axis(int64_t c, int64_t S, int64_t ext) {
  // position of coordinate c in predictor.py:230-235's closed axis
  return ((c & (S - 1)) == 0) ? (c / S) : ((ext - 1) / S + 1);
}

// ---------------------------------------------------------------------------
// decompress: inverse interpolation from symbols
// ---------------------------------------------------------------------------
template <int BZ, int BY, int BX, int NT>
__global__ void __launch_bounds__(NT, 3) k_reconstruct(
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
  const int o[3] = {bz * BZ, by * BY, bx * BX};
  const int ext[3] = {(int)P.ext[0], (int)P.ext[1], (int)P.ext[2]};
  const int tile[3] = {(int)P.tile[0], (int)P.tile[1], (int)P.tile[2]};
  int L[3];
  L[0] = min(CZ, ext[0] - o[0]);
  L[1] = min(CY, ext[1] - o[1]);
  L[2] = min(CX, ext[2] - o[2]);
  const int O0 = min(BZ, L[0]), O1 = min(BY, L[1]), O2 = min(BX, L[2]);
  const int64_t S = P.stride;
  const int64_t na1 = (P.ext[1] - 1) / S + 1 + (((P.ext[1] - 1) & (S - 1)) ? 1 : 0);
  const int64_t na2 = (P.ext[2] - 1) / S + 1 + (((P.ext[2] - 1) & (S - 1)) ? 1 : 0);

  const int warp = tid >> 5, lane = tid & 31;
  const bool fast_path = false;
  for (int row = warp; !fast_path && row < L[0] * L[1]; row += NT / 32) {
    const int lz = row / L[1], ly = row - lz * L[1];
    const int64_t g0 = o[0] + lz, g1 = o[1] + ly;
    const uint16_t *src = sym + (g0 * P.ext[1] + g1) * P.ext[2] + o[2];
    uint16_t *dst = cs_ + (lz * PY + ly) * PX;
    float *bd = buf + (lz * PY + ly) * PX;
    const bool a01 = ((g0 & (S - 1)) == 0 || g0 == P.ext[0] - 1) &&
                     ((g1 & (S - 1)) == 0 || g1 == P.ext[1] - 1);
    for (int lx = lane; lx < L[2]; lx += 32) {
      dst[lx] = src[lx];
      const int64_t g2 = o[2] + lx;
      if (a01 && ((g2 & (S - 1)) == 0 || g2 == P.ext[2] - 1)) {
        const int64_t ai = (anchor_index_axis(g0, S, P.ext[0]) * na1 +
                            anchor_index_axis(g1, S, P.ext[1])) * na2 +
                           anchor_index_axis(g2, S, P.ext[2]);
        bd[lx] = anchors[ai];
      }
    }
  }
  __syncthreads();

  if (!fast_path)
    run_levels<1, BZ, BY, BX, NT, false>(buf, nullptr, cs_, lc, L, o, ext, tile, (int)S,
                                         P.rank, R, out_idx, out_val, n_out, P.ext[1], P.ext[2]);

  for (int row = warp; row < O0 * O1; row += NT / 32) {
    const int lz = row / O1, ly = row - lz * O1;
    float *dst = y + ((int64_t)(o[0] + lz) * ext[1] + (o[1] + ly)) * (int64_t)ext[2] + o[2];
    const float *srow = buf + (lz * PY + ly) * PX;
    for (int lx = lane; lx < O2; lx += 32) dst[lx] = srow[lx];
  }
}


// ---------------------------------------------------------------------------
// specialised kernels for the default layouts (interp_fast.cuh)
// ---------------------------------------------------------------------------
template <class LY>
DEV bool is_interior(const int o[3], const int ext[3]) {
  return (LY::CZ == 1 || o[0] + LY::BZ <= ext[0] - 1) &&
         (LY::CY == 1 || o[1] + LY::BY <= ext[1] - 1) && (o[2] + LY::BX <= ext[2] - 1);
}

template <class LY, int NT>
DEV void block_coords(const InterpParams &P, int o[3], int e[3], int ext[3]) {
  int b = blockIdx.x;
  const int bx = b % P.nb[2];
  b /= P.nb[2];
  const int by = b % P.nb[1];
  const int bz = b / P.nb[1];
  o[0] = P.z0 + bz * LY::BZ;
  o[1] = by * LY::BY;
  o[2] = bx * LY::BX;
  for (int a = 0; a < 3; ++a) {
    ext[a] = (int)P.ext[a];
    e[a] = ext[a] - o[a];
  }
}

template <class LY, int NT, bool EXACT>
__global__ void __launch_bounds__(NT) k_predict_fast(const float *__restrict__ x, InterpParams P,
                                                     const cszi_ctl *__restrict__ ctl,
                                                     uint16_t *__restrict__ sym,
                                                     u64 *__restrict__ hist, int hist_in_smem) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float *buf = reinterpret_cast<float *>(smem_raw);
  uint16_t *codes = reinterpret_cast<uint16_t *>(buf + ((LY::NCLOSED + 3) & ~3));
  uint32_t *hs = reinterpret_cast<uint32_t *>(codes + LY::NOWNED);
  __shared__ LevelCfg cfg;
  __shared__ uint32_t zero_ws[NT / 32];
  const int R = P.radius;
  const int tid = threadIdx.x;
  int o[3], e[3], ext[3];
  block_coords<LY, NT>(P, o, e, ext);
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
    for (int i = tid; i < 2 * R; i += NT) hs[i] = 0;
  const int64_t base = ((int64_t)(o[0] - P.z0) * ext[1] + o[1]) * (int64_t)ext[2] + o[2];
  const int pz = ext[1] * ext[2], py = ext[2];
  const bool interior = is_interior<LY>(o, ext);
  if (interior)
    fast::stage<LY, false, NT>(buf, x, base, pz, py, e);
  else
    fast::stage<LY, true, NT>(buf, x, base, pz, py, e);
  const uint32_t rr = (uint32_t)R | ((uint32_t)R << 16);
  for (int i = tid; i < LY::NOWNED / 8; i += NT)
    reinterpret_cast<uint4 *>(codes)[i] = make_uint4(rr, rr, rr, rr);
  __syncthreads();
  fast::Blk K{};
  for (int a = 0; a < 3; ++a) K.e[a] = e[a];
  uint32_t zeros;
  if (interior) {
    fast::run<LY, 0, EXACT, false, NT>(buf, codes, nullptr, cfg, R, K, ext, P.rank);
    zeros = fast::store_codes_hist<LY, false, NT>(codes, sym, base, pz, py, e, R, hs,
                                                  hist_in_smem != 0, hist);
  } else {
    fast::run<LY, 0, EXACT, true, NT>(buf, codes, nullptr, cfg, R, K, ext, P.rank);
    zeros = fast::store_codes_hist<LY, true, NT>(codes, sym, base, pz, py, e, R, hs,
                                                 hist_in_smem != 0, hist);
  }
  const int warp = tid >> 5, lane = tid & 31;
  zeros = warp_sum(zeros);
  if (lane == 0) zero_ws[warp] = zeros;
  __syncthreads();
  if (tid == 0) {
    uint32_t z = 0;
    for (int w = 0; w < NT / 32; ++w) z += zero_ws[w];
    if (z) atomicAdd(&hist[R], (u64)z);
  }
  if (hist_in_smem)
    for (int i = tid; i < 2 * R; i += NT)
      if (hs[i]) atomicAdd(&hist[i], (u64)hs[i]);
}


template <class LY, int NT>
__global__ void __launch_bounds__(NT) k_reconstruct_fast(
    const uint16_t *__restrict__ sym, const float *__restrict__ anchors, const u64 *out_idx,
    const float *out_val, u64 n_out, const u64 *nout_dev, InterpParams P, LevelCfg lc,
    float *__restrict__ y) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float *buf = reinterpret_cast<float *>(smem_raw);
  uint16_t *cs_ = reinterpret_cast<uint16_t *>(buf + ((LY::NCLOSED + 3) & ~3));
  const int R = P.radius;
  const int tid = threadIdx.x;
  if (nout_dev) n_out = *nout_dev;
  int o[3], e[3], ext[3];
  block_coords<LY, NT>(P, o, e, ext);
  const int64_t base = ((int64_t)(o[0] - P.z0) * ext[1] + o[1]) * (int64_t)ext[2] + o[2];
  const int pz = ext[1] * ext[2], py = ext[2];
  const bool interior = is_interior<LY>(o, ext);
  if (interior)
    fast::stage<LY, false, NT>(cs_, sym, base, pz, py, e);
  else
    fast::stage<LY, true, NT>(cs_, sym, base, pz, py, e);
  {
    // seed the anchors of the closed block from the anchor section
    constexpr int S = LY::S;
    int az[LY::CZ / S + 2], ay[LY::CY / S + 2], ax[LY::CX / S + 2];
    const int nz = anchor_axis_local<LY::CZ, S>(e[0], az);
    const int ny = anchor_axis_local<LY::CY, S>(e[1], ay);
    const int nx = anchor_axis_local<LY::CX, S>(e[2], ax);
    const int64_t na1 = (P.ext[1] - 1) / S + 1 + (((P.ext[1] - 1) % S) ? 1 : 0);
    const int64_t na2 = (P.ext[2] - 1) / S + 1 + (((P.ext[2] - 1) % S) ? 1 : 0);
    for (int i = tid; i < nz * ny * nx; i += NT) {
      const int iz = i / (ny * nx), r = i - iz * ny * nx, iy = r / nx, ix = r - iy * nx;
      const int lz = az[iz], ly = ay[iy], lx = ax[ix];
      const int gz = o[0] + lz, gy = o[1] + ly, gx = o[2] + lx;
      const int64_t kz = (gz % S == 0) ? gz / S : (ext[0] - 1) / S + 1;
      const int64_t ky = (gy % S == 0) ? gy / S : (ext[1] - 1) / S + 1;
      const int64_t kx = (gx % S == 0) ? gx / S : (ext[2] - 1) / S + 1;
      buf[(lz * LY::PY + ly) * LY::PX + lx] = anchors[(kz * na1 + ky) * na2 + kx];
    }
  }
  __syncthreads();
  fast::Blk K;
  for (int a = 0; a < 3; ++a) K.e[a] = e[a];
  K.idx = out_idx;
  K.val = out_val;
  K.n = n_out;
  K.gs0 = (int64_t)ext[1] * ext[2];
  K.gs1 = ext[2];
  K.o0 = o[0];
  K.o1 = o[1];
  K.o2 = o[2];
  if (interior)
    fast::run<LY, 1, false, false, NT>(buf, nullptr, cs_, lc, R, K, ext, P.rank);
  else
    fast::run<LY, 1, false, true, NT>(buf, nullptr, cs_, lc, R, K, ext, P.rank);
  // owned region -> y
  const int O0 = min(LY::BZ, e[0]), O1 = min(LY::BY, e[1]), O2 = min(LY::BX, e[2]);
  const int warp = tid >> 5, lane = tid & 31;
  for (int row = warp; row < O0 * O1; row += NT / 32) {
    const int lz = row / O1, ly = row - lz * O1;
    float *dst = y + base + (int64_t)lz * pz + (int64_t)ly * py;
    const float *srow = buf + (lz * LY::PY + ly) * LY::PX;
    for (int lx = lane; lx < O2; lx += 32) dst[lx] = srow[lx];
  }
}

// ---------------------------------------------------------------------------
// anchors: gather_anchors (predictor.py:250-256) / lattice row-major order
// ---------------------------------------------------------------------------
// anchor planes i0 in [ia0, ia0 + na0) of the lattice; x holds planes from z0
__global__ void k_gather_anchors(const float *__restrict__ x, InterpParams P, int64_t ia0,
                                 int64_t na0, int64_t na1, int64_t na2, int64_t z0,
                                 float *__restrict__ out) {
  const int64_t total = na0 * na1 * na2;
  const int64_t S = P.stride;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i2 = i % na2, t = i / na2, i1 = t % na1, i0 = ia0 + t / na1;
    const int64_t c0 = min(i0 * S, P.ext[0] - 1), c1 = min(i1 * S, P.ext[1] - 1),
                  c2 = min(i2 * S, P.ext[2] - 1);
    out[i] = x[((c0 - z0) * P.ext[1] + c1) * P.ext[2] + c2];
  }
}

// anchor-lattice planes [ia0, ia1) whose z coordinate lies in the slab
static void slab_anchor_planes(const cszi_geom *g, int64_t &ia0, int64_t &ia1) {
  const int64_t e = g->ext[0], S = g->stride;
  const int64_t na = (e - 1) / S + 1 + (((e - 1) % S) ? 1 : 0);
  if (g->slab[1] <= g->slab[0]) {
    ia0 = 0;
    ia1 = na;
    return;
  }
  const int64_t z0 = g->slab[0], z1 = g->slab[1];
  ia0 = (z0 + S - 1) / S;
  ia1 = ia0;
  while (ia1 < na && std::min(ia1 * S, e - 1) < z1) ++ia1;
}

uint64_t slab_anchor_count(const cszi_geom *g) {
  int64_t ia0, ia1;
  slab_anchor_planes(g, ia0, ia1);
  int64_t c = ia1 - ia0;
  for (int a = 1; a < 3; ++a) {
    const int64_t e = g->ext[a], S = g->stride;
    c *= (e - 1) / S + 1 + (((e - 1) % S) ? 1 : 0);
  }
  return (uint64_t)c;
}

namespace t3 {  // t3.cu: the 3-D default-layout tile kernels
int launch_predict_t3(const float *x, const cszi_geom *g, int32_t radius, const cszi_ctl *ctl,
                      uint16_t *sym, u64 *hist, bool exact, cudaStream_t st, uint32_t *nzmap,
                      bool *nz_done);
int launch_recon_t3(const uint16_t *sym, const float *anchors, const u64 *oidx, const float *oval,
                    u64 nout, const u64 *nout_dev, const cszi_geom *g, int32_t radius,
                    const LevelCfg &lc, float *y, cudaStream_t st);
}  // namespace t3

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
  P.z0 = 0;
  if (g->slab[1] > g->slab[0]) {  // z-slab shard: blocks over the owned planes
    if (g->slab[0] % bz != 0) return false;
    P.z0 = (int)g->slab[0];
    P.nb[0] = (int)((g->slab[1] - g->slab[0] + bz - 1) / bz);
  }
  return true;
}

#define CSZI_NT 256

template <int BZ, int BY, int BX>
static int launch_predict_t(const float *x, const cszi_geom *g, int32_t radius,
                            const cszi_ctl *ctl, uint16_t *sym, u64 *hist, bool exact,
                            cudaStream_t st) {
  InterpParams P;
  if (!fill_params(g, radius, BZ, BY, BX, P) || P.z0 != 0 || g->slab[1] > g->slab[0])
    return CSZI_E_UNSUPPORTED;
  const bool hsm = 2 * radius <= 8192;
  const size_t smem = predict_smem<BZ, BY, BX>(radius, hsm);
  const int64_t nblk = (int64_t)P.nb[0] * P.nb[1] * P.nb[2];
  if (nblk > 0x7fffffffLL) return CSZI_E_UNSUPPORTED;
  if (exact) {
    auto k = k_predict<BZ, BY, BX, CSZI_NT, true>;
    ensure_smem((const void *)k, smem);
    k<<<(unsigned)nblk, CSZI_NT, smem, st>>>(x, P, ctl, sym, hist, hsm ? 1 : 0);
    note_launch();
  } else {
    auto k = k_predict<BZ, BY, BX, CSZI_NT, false>;
    ensure_smem((const void *)k, smem);
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
  if (!fill_params(g, radius, BZ, BY, BX, P) || g->slab[1] > g->slab[0])
    return CSZI_E_UNSUPPORTED;
  const size_t smem = recon_smem<BZ, BY, BX>();
  const int64_t nblk = (int64_t)P.nb[0] * P.nb[1] * P.nb[2];
  if (nblk > 0x7fffffffLL) return CSZI_E_UNSUPPORTED;
  auto k = k_reconstruct<BZ, BY, BX, CSZI_NT>;
  ensure_smem((const void *)k, smem);
  k<<<(unsigned)nblk, CSZI_NT, smem, st>>>(sym, anchors, oidx, oval, nout, nout_dev, P, lc, y);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

// Block shapes per layout: 3-D default (8,8,32) tiles -> 8x16x32 blocks;
// 2-D (16,16) tiles -> 1x32x64; 1-D 512 tile -> 1x1x1024.  Non-default
// strides (decode of archives with anchor_stride != default) use the shape
// whose extents are multiples of (stride,)*rank when one exists.
template <class LY>
static bool layout_is(const cszi_geom *g) {
  return g->stride == LY::S && g->tile[0] == LY::TZ && g->tile[1] == LY::TY &&
         g->tile[2] == LY::TX && (LY::CZ > 1 || g->ext[0] == 1) && (LY::CY > 1 || g->ext[1] == 1);
}

template <class LY, int NT>
static int launch_predict_fast(const float *x, const cszi_geom *g, int32_t radius,
                               const cszi_ctl *ctl, uint16_t *sym, u64 *hist, bool exact,
                               cudaStream_t st) {
  InterpParams P;
  if (!fill_params(g, radius, LY::BZ, LY::BY, LY::BX, P)) return CSZI_E_UNSUPPORTED;
  const bool hsm = 2 * radius <= 8192;
  const size_t smem = sizeof(float) * ((LY::NCLOSED + 3) & ~3) + sizeof(uint16_t) * LY::NOWNED +
                      (hsm ? sizeof(uint32_t) * 2 * (size_t)radius : 0);
  const int64_t nblk = (int64_t)P.nb[0] * P.nb[1] * P.nb[2];
  if (nblk > 0x7fffffffLL) return CSZI_E_UNSUPPORTED;
  if (exact) {
    auto k = k_predict_fast<LY, NT, true>;
    ensure_smem((const void *)k, smem);
    k<<<(unsigned)nblk, NT, smem, st>>>(x, P, ctl, sym, hist, hsm ? 1 : 0);
  } else {
    auto k = k_predict_fast<LY, NT, false>;
    ensure_smem((const void *)k, smem);
    k<<<(unsigned)nblk, NT, smem, st>>>(x, P, ctl, sym, hist, hsm ? 1 : 0);
  }
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

template <class LY, int NT>
static int launch_recon_fast(const uint16_t *sym, const float *anchors, const u64 *oidx,
                             const float *oval, u64 nout, const u64 *nout_dev,
                             const cszi_geom *g, int32_t radius, const LevelCfg &lc, float *y,
                             cudaStream_t st) {
  InterpParams P;
  if (!fill_params(g, radius, LY::BZ, LY::BY, LY::BX, P)) return CSZI_E_UNSUPPORTED;
  const size_t smem = sizeof(float) * ((LY::NCLOSED + 3) & ~3) + sizeof(uint16_t) * LY::NCLOSED + 16;
  const int64_t nblk = (int64_t)P.nb[0] * P.nb[1] * P.nb[2];
  if (nblk > 0x7fffffffLL) return CSZI_E_UNSUPPORTED;
  auto k = k_reconstruct_fast<LY, NT>;
  ensure_smem((const void *)k, smem);
  k<<<(unsigned)nblk, NT, smem, st>>>(sym, anchors, oidx, oval, nout, nout_dev, P, lc, y);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

int launch_predict(const float *x, const cszi_geom *g, int32_t radius, const cszi_ctl *ctl,
                   uint16_t *sym, u64 *hist, bool exact, cudaStream_t st, uint32_t *nzmap,
                   bool *nz_done) {
  if (nz_done) *nz_done = false;
  if (g->rank == 3 && layout_is<fast::L3>(g))
    return t3::launch_predict_t3(x, g, radius, ctl, sym, hist, exact, st, nzmap, nz_done);
  if (g->rank == 2 && layout_is<fast::L2>(g))
    return launch_predict_fast<fast::L2, 128>(x, g, radius, ctl, sym, hist, exact, st);
  if (g->rank == 1 && layout_is<fast::L1>(g))
    return launch_predict_fast<fast::L1, 128>(x, g, radius, ctl, sym, hist, exact, st);
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
  if (g->rank == 3 && layout_is<fast::L3>(g) && nlev == 3)
    return t3::launch_recon_t3(sym, anchors, oidx, oval, nout, nout_dev, g, radius, lc, y, st);
  if (g->rank == 2 && layout_is<fast::L2>(g))
    return launch_recon_fast<fast::L2, 128>(sym, anchors, oidx, oval, nout, nout_dev, g, radius,
                                            lc, y, st);
  if (g->rank == 1 && layout_is<fast::L1>(g))
    return launch_recon_fast<fast::L1, 128>(sym, anchors, oidx, oval, nout, nout_dev, g, radius,
                                            lc, y, st);
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

// ---------------------------------------------------------------------------
// interpolate_level (predictor.py:367-392): one level's per-dimension passes
// over a global-memory reconstruction buffer, one thread per pass point, in
// the reference's exact point set and arithmetic, anchors restored after
// each pass.  This is the fine-grained API (the reference's tests drive the
// predictor level by level); the compress / decompress path runs all levels
// inside the tile kernels instead.
// ---------------------------------------------------------------------------
struct LevelPass {
  int64_t ext[3];
  int64_t cnt[3];   // lattice points per axis
  int64_t step[3];  // lattice step per axis (d: 2s starting at s)
  int64_t tile;     // super-chunk extent along d
  int d;
  int s;
  int R;
  double leb, e2, wo, wi;
};

// mode 0 (Compress): source -> recon / codes (q or 0) / is_outlier;
// mode 1 (Decompress): codes / is_outlier / outlier_values -> recon
__global__ void k_level_pass(LevelPass L, int mode, float *__restrict__ recon,
                             const float *__restrict__ source, int32_t *__restrict__ codes,
                             uint8_t *__restrict__ is_out, const float *__restrict__ oval) {
  const int64_t total = L.cnt[0] * L.cnt[1] * L.cnt[2];
  const int64_t st1 = L.ext[2], st0 = L.ext[1] * L.ext[2];
  const int64_t sd = (L.d == 0) ? st0 : (L.d == 1) ? st1 : 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i2 = i % L.cnt[2], r = i / L.cnt[2], i1 = r % L.cnt[1], i0 = r / L.cnt[1];
    int64_t c[3] = {i0 * L.step[0], i1 * L.step[1], i2 * L.step[2]};
    c[L.d] += L.s;  // odd multiples of s along d
    const int64_t pd = c[L.d], ed = L.ext[L.d], s = L.s;
    const int64_t off = pd % L.tile;
    const bool m3 = off >= 3 * s;
    const bool p1 = pd + s <= ed - 1;
    const bool p3 = (off <= L.tile - 3 * s) && (pd + 3 * s <= ed - 1);
    const int cs = !p1 ? 4 : m3 ? (p3 ? 0 : 1) : (p3 ? 2 : 3);
    const int64_t ix = c[0] * st0 + c[1] * st1 + c[2];
    const double vm1 = f2d(recon[ix - s * sd]);
    const double vp1 = p1 ? f2d(recon[ix + s * sd]) : 0.0;
    const double vm3 = m3 ? f2d(recon[ix - 3 * s * sd]) : 0.0;
    const double vp3 = p3 ? f2d(recon[ix + 3 * s * sd]) : 0.0;
    const double pred = spline4(cs, L.wo, L.wi, vm3, vm1, vp1, vp3);
    if (mode == 0) {
      float rec;
      const uint32_t sy = quantize<true>(pred, source[ix], L.leb, L.e2, 0.0, L.R, rec);
      recon[ix] = rec;
      codes[ix] = sy ? (int32_t)sy - L.R : 0;
      is_out[ix] = sy ? 0 : 1;
    } else {
      const double q = (double)codes[ix];
      const float rec = __double2float_rn(dadd(pred, dmul(L.e2, q)));
      recon[ix] = is_out[ix] ? oval[ix] : rec;
    }
  }
}

// recon[anchor lattice] = anchor_block (lattice row-major)
__global__ void k_anchor_restore(float *__restrict__ recon, const float *__restrict__ block,
                                 int64_t e0, int64_t e1, int64_t e2, int64_t S, int64_t na0,
                                 int64_t na1, int64_t na2) {
  const int64_t total = na0 * na1 * na2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i2 = i % na2, t = i / na2, i1 = t % na1, i0 = t / na1;
    const int64_t c0 = min(i0 * S, e0 - 1), c1 = min(i1 * S, e1 - 1), c2 = min(i2 * S, e2 - 1);
    recon[(c0 * e1 + c1) * e2 + c2] = block[i];
  }
}

int launch_interp_level(float *recon, const float *source, int32_t *codes, uint8_t *is_out,
                        const float *oval, const float *anchor_block, const cszi_geom *g,
                        int64_t s, double leb, const int32_t variant[3], const int32_t order[3],
                        int32_t R, int32_t mode, cudaStream_t st) {
  if (s < 1 || (s & (s - 1)) || !(leb > 0) || R < 2 || (mode != 0 && mode != 1))
    return CSZI_E_INVALID_ARG;
  const int64_t S = g->stride;
  int64_t na[3];
  for (int a = 0; a < 3; ++a) na[a] = (g->ext[a] - 1) / S + 1 + (((g->ext[a] - 1) % S) ? 1 : 0);
  const int pad = 3 - g->rank;
  int passed = 0;
  for (int i = 0; i < g->rank; ++i) {
    const int d = order[i];
    if (d < pad || d > 2) return CSZI_E_INVALID_ARG;
    LevelPass L;
    int64_t total = 1;
    for (int a = 0; a < 3; ++a) {
      L.ext[a] = g->ext[a];
      if (a == d) {
        L.step[a] = 2 * s;
        L.cnt[a] = g->ext[a] > s ? (g->ext[a] - s + 2 * s - 1) / (2 * s) : 0;
      } else {
        L.step[a] = ((passed >> a) & 1) ? s : 2 * s;
        L.cnt[a] = (g->ext[a] + L.step[a] - 1) / L.step[a];
      }
      total *= L.cnt[a];
    }
    L.tile = g->tile[d];
    L.d = d;
    L.s = (int)s;
    L.R = R;
    L.leb = leb;
    L.e2 = 2.0 * leb;
    L.wo = variant[d] == 0 ? NAK_O : NAT_O;
    L.wi = variant[d] == 0 ? NAK_I : NAT_I;
    if (total > 0) {
      int64_t blocks = (total + 255) / 256;
      if (blocks > (int64_t)sm_count() * 16) blocks = (int64_t)sm_count() * 16;
      k_level_pass<<<(unsigned)blocks, 256, 0, st>>>(L, mode, recon, source, codes, is_out, oval);
      note_launch();
      const int64_t ta = na[0] * na[1] * na[2];
      k_anchor_restore<<<(unsigned)std::min<int64_t>((ta + 255) / 256, 4096), 256, 0, st>>>(
          recon, anchor_block, g->ext[0], g->ext[1], g->ext[2], S, na[0], na[1], na[2]);
      note_launch();
    }
    passed |= 1 << d;
  }
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
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
  int64_t ia0, ia1;
  slab_anchor_planes(g, ia0, ia1);
  const int64_t z0 = (g->slab[1] > g->slab[0]) ? g->slab[0] : 0;
  const int64_t total = (ia1 - ia0) * na[1] * na[2];
  if (total <= 0) return CSZI_OK;
  const int threads = 256;
  int64_t blocks = (total + threads - 1) / threads;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  k_gather_anchors<<<(unsigned)blocks, threads, 0, st>>>(x, P, ia0, ia1 - ia0, na[1], na[2], z0,
                                                         out);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

}  // namespace cszi
