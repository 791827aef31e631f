// Value range + finite scan, and the sampling auto-tuner, for sm_100a.
//
// Reference semantics: grid.py:60-62 (NaN/Inf scan -> first flat index),
// grid.py:104-108 (value_range), tuning.py:32-129 (profile_samples,
// compute_alpha, select_config), predictor.py:122-136 (plan_levels).
#include "common.cuh"

namespace cszi {

// ctl reset: keys for the min/max atomics, flags, counters.
__global__ void k_ctl_init(cszi_ctl *ctl) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    ctl->vmin_key = 0xffffffffu;
    ctl->vmax_key = 0u;
    ctl->first_nonfinite = ~0ull;
    ctl->bits = 0;
    ctl->n_outliers = 0;
    ctl->raw_len = 0;
    ctl->payload_len = 0;
    ctl->decoded_symbols = 0;
    ctl->flags = 0;
    ctl->max_len = 0;
    for (int i = 0; i < 8; ++i) ctl->scratch[i] = 0;
  }
}

// One read of x: min/max over order-preserving keys and the first non-finite
// flat index (NaN/Inf have an all-ones exponent).
__global__ void __launch_bounds__(256, 4) k_range(const float *__restrict__ x, uint64_t n,
                                               cszi_ctl *ctl) {
  uint32_t kmin = 0xffffffffu, kmax = 0u;
  u64 bad = ~0ull;
  const u64 tid = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  const u64 nthr = (u64)gridDim.x * blockDim.x;
  const bool aligned = ((uintptr_t)x & 15) == 0;
  u64 done = 0;
  if (aligned) {
    // two float4 per iteration in flight; keys of non-finite values enter the
    // min/max too (the caller raises NonFiniteValue before using the range),
    // so the exact first index is only computed on the rare bad vector
    const u64 n4 = n / 4;
    const float4 *x4 = reinterpret_cast<const float4 *>(x);
    constexpr uint32_t EXP = 0x7f800000u;
    u64 i = tid;
    // four float4 per thread in flight (64 KB per SM at 4 blocks): enough
    // bytes outstanding to cover HBM latency (two left it at ~75% of peak)
    for (; i + 3 * nthr < n4; i += 4 * nthr) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcs(x4 + i + u * nthr);
      bool nf = false;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t b[4] = {__float_as_uint(v[u].x), __float_as_uint(v[u].y),
                               __float_as_uint(v[u].z), __float_as_uint(v[u].w)};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          nf |= (b[j] & EXP) == EXP;
          const uint32_t k = b[j] ^ ((uint32_t)((int32_t)b[j] >> 31) | 0x80000000u);
          kmin = min(kmin, k);
          kmax = max(kmax, k);
        }
      }
      if (nf) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t b[4] = {__float_as_uint(v[u].x), __float_as_uint(v[u].y),
                                 __float_as_uint(v[u].z), __float_as_uint(v[u].w)};
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if ((b[j] & EXP) == EXP) bad = min(bad, 4 * (i + u * nthr) + j);
        }
      }
    }
    for (; i < n4; i += nthr) {
      const float4 v = __ldcs(x4 + i);
      const float a[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t b = __float_as_uint(a[j]);
        if ((b & EXP) == EXP) bad = min(bad, 4 * i + j);
        const uint32_t k = float_key(a[j]);
        kmin = min(kmin, k);
        kmax = max(kmax, k);
      }
    }
    done = n4 * 4;
  }
  for (u64 i = done + tid; i < n; i += nthr) {
    const float f = x[i];
    const uint32_t b = __float_as_uint(f);
    if ((b & 0x7f800000u) == 0x7f800000u) {
      bad = min(bad, i);
    } else {
      const uint32_t k = float_key(f);
      kmin = min(kmin, k);
      kmax = max(kmax, k);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    kmin = min(kmin, __shfl_xor_sync(CSZI_FULL, kmin, o));
    kmax = max(kmax, __shfl_xor_sync(CSZI_FULL, kmax, o));
    bad = min(bad, __shfl_xor_sync(CSZI_FULL, bad, o));
  }
  __shared__ uint32_t smin[8], smax[8];
  __shared__ u64 sbad[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    smin[warp] = kmin;
    smax[warp] = kmax;
    sbad[warp] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      kmin = min(kmin, smin[w]);
      kmax = max(kmax, smax[w]);
      bad = min(bad, sbad[w]);
    }
    atomicMin(&ctl->vmin_key, kmin);
    atomicMax(&ctl->vmax_key, kmax);
    if (bad != ~0ull) atomicMin((u64 *)&ctl->first_nonfinite, bad);
  }
}

struct TuneArgs {
  int64_t ext[3];  // padded (global)
  int32_t rank;
  int32_t pad_axes;  // 3 - rank
  int32_t mode_rel;
  int32_t have_variants, have_order;
  int32_t nlev;
  double eb;
  double alpha;
  double alpha_pow[CSZI_MAX_LEVELS];
  int32_t variant[3];
  int32_t order[3];
  int64_t z0;        // global z of local plane 0
  int64_t zlo, zhi;  // owned global z range (values outside read as 0)
};

// tuning.py:32-39 on one axis.
DEV int sample_axis(int64_t extent, int64_t *out) {
  const int64_t k = min((int64_t)4, extent / 7);
  for (int64_t j = 0; j < k; ++j) {
    int64_t c = (j + 1) * extent / (k + 1);
    out[j] = min(max(c, (int64_t)3), extent - 4);
  }
  return (int)k;
}

struct SamplePlan {
  int64_t pts[3][4];
  int npts[3];
  int prof[3];
  int P;
};

DEV void sample_plan(const TuneArgs &A, SamplePlan &sp) {
  const int rank = A.rank, pad = A.pad_axes;
  for (int d = 0; d < rank; ++d) {
    const int64_t e = A.ext[pad + d];
    const int k = sample_axis(e, sp.pts[d]);
    sp.prof[d] = k > 0;
    if (k == 0) {
      sp.pts[d][0] = e / 2;
      sp.npts[d] = 1;
    } else {
      sp.npts[d] = k;
    }
  }
  for (int d = rank; d < 3; ++d) {
    sp.npts[d] = 1;
    sp.prof[d] = 0;
    sp.pts[d][0] = 0;
  }
  sp.P = sp.npts[0] * sp.npts[1] * sp.npts[2];  // <= 64 mesh points, ij order
}

// Gather the profiled values (tuning.py:55-62): for mesh point p and
// profiled dim d, vals[(p*3 + d)*5 + k] = bits of the values at offsets
// -3, -1, +1, +3 along d (k = 0..3) and of the point itself (k = 4); 0 when
// the value's plane is outside [zlo, zhi) (another shard owns it).
// One block of 1024 threads: the plan is built once in shared memory and
// every sample load is in flight at the same time (a thread per value).
__global__ void __launch_bounds__(1024) k_sample_gather(const float *__restrict__ x, TuneArgs A,
                                                        int32_t *vals, cszi_ctl *reset_ctl) {
  __shared__ SamplePlan sp;
  if (threadIdx.x == 0) {
    if (reset_ctl) ctl_reset_outputs(reset_ctl);  // (was its own 1-thread launch)
    sample_plan(A, sp);
  }
  const int rank = A.rank, pad = A.pad_axes;
  for (int w = threadIdx.x; w < CSZI_SAMPLE_WORDS; w += blockDim.x) vals[w] = 0;
  __syncthreads();
  for (int w = threadIdx.x; w < sp.P * rank * 5; w += blockDim.x) {
    const int k = w % 5, pd = w / 5, p = pd / rank, d = pd - p * rank;
    if (!sp.prof[d]) continue;
    int idx[3];
    int rem = p;
    for (int a = rank - 1; a >= 0; --a) {
      idx[a] = rem % sp.npts[a];
      rem /= sp.npts[a];
    }
    int64_t c[3] = {0, 0, 0};
    for (int a = 0; a < rank; ++a) c[pad + a] = sp.pts[a][idx[a]];
    const int offs[5] = {-3, -1, 1, 3, 0};
    c[pad + d] += offs[k];
    if (c[0] < A.zlo || c[0] >= A.zhi) continue;
    const int64_t li = ((c[0] - A.z0) * A.ext[1] + c[1]) * A.ext[2] + c[2];
    vals[(p * 3 + d) * 5 + k] = __float_as_int(x[li]);
  }
}

// select_config + plan_levels from the gathered samples; the error sums are
// accumulated in the reference's order (mesh order, per (d, v)).
__global__ void __launch_bounds__(256) k_tune_decide(const int32_t *__restrict__ vals,
                                                     TuneArgs A, cszi_ctl *ctl, u64 *zero_hist,
                                                     int nzero) {
  __shared__ SamplePlan sp;
  __shared__ double errs[64][3][2];
  __shared__ double err_sum[3][2];
  __shared__ int64_t cnt[3];
  const int tid = threadIdx.x;
  const int rank = A.rank, pad = A.pad_axes;
  // the predictor's histogram bins (a memset node in the graph would cost a
  // few us of gap on each side)
  for (int i = tid; i < nzero; i += blockDim.x) zero_hist[i] = 0;
  if (tid == 0) sample_plan(A, sp);
  __syncthreads();
  const int P = sp.P;
  for (int w = tid; w < P * rank; w += blockDim.x) {
    const int p = w / rank, d = w - p * rank;
    if (!sp.prof[d]) continue;
    const int32_t *v = vals + (p * 3 + d) * 5;
    const double v0 = (double)__int_as_float(v[0]), v1 = (double)__int_as_float(v[1]);
    const double v2 = (double)__int_as_float(v[2]), v3 = (double)__int_as_float(v[3]);
    const double actual = (double)__int_as_float(v[4]);
    // tuning.py:63-66, weights predictor.py:62-65
    const double wts[2][2] = {{-1.0 / 16.0, 9.0 / 16.0}, {-3.0 / 40.0, 23.0 / 40.0}};
    for (int vv = 0; vv < 2; ++vv) {
      const double pred =
          dadd(dadd(dadd(dmul(wts[vv][0], v0), dmul(wts[vv][1], v1)), dmul(wts[vv][1], v2)),
               dmul(wts[vv][0], v3));
      errs[p][d][vv] = fabs(dsub(pred, actual));
    }
  }
  __syncthreads();
  if (tid < 6) {
    const int d = tid >> 1, v = tid & 1;
    double acc = 0.0;
    if (d < rank && sp.prof[d])
      for (int p = 0; p < P; ++p) acc = dadd(acc, errs[p][d][v]);
    err_sum[d][v] = acc;
    if (v == 0) cnt[d] = (d < rank && sp.prof[d]) ? P : 0;
  }
  __syncthreads();
  if (tid != 0) return;

  // range (grid.py:104-108): Python floats from float32, rng in float64
  const double lo = (double)key_float(ctl->vmin_key);
  const double hi = (double)key_float(ctl->vmax_key);
  const double rng = dsub(hi, lo);
  ctl->vmin = lo;
  ctl->vmax = hi;
  ctl->rng = rng;
  if (ctl->first_nonfinite != ~0ull) ctl->flags |= CSZI_F_NONFINITE;
  // tuning.py:100-109
  double eb_abs;
  if (A.mode_rel) {
    eb_abs = (rng > 0.0) ? dmul(A.eb, rng) : A.eb;
  } else {
    eb_abs = A.eb;
  }
  ctl->eb_abs = eb_abs;
  ctl->alpha = A.alpha;
  for (int d = 0; d < 3; ++d) {
    ctl->err_sum[d][0] = err_sum[d][0];
    ctl->err_sum[d][1] = err_sum[d][1];
    ctl->sample_count[d] = cnt[d];
  }
  // variants: tuning.py:111-114 (padded axes get NOTAKNOT)
  for (int a = 0; a < 3; ++a) ctl->variant[a] = 0;
  for (int d = 0; d < rank; ++d)
    ctl->variant[pad + d] =
        A.have_variants ? A.variant[pad + d] : (err_sum[d][0] <= err_sum[d][1] ? 0 : 1);
  // order: tuning.py:115-122 key (count == 0, -mean, d), stable sort
  if (A.have_order) {
    for (int i = 0; i < 3; ++i) ctl->order[i] = A.order[i];
  } else {
    int ord[3] = {0, 1, 2};
    double negmean[3];
    for (int d = 0; d < rank; ++d) {
      const double mean = cnt[d] ? ddiv(dadd(err_sum[d][0], err_sum[d][1]), (double)cnt[d]) : 0.0;
      negmean[d] = -mean;
    }
    for (int i = 1; i < rank; ++i) {
      int j = i;
      while (j > 0) {
        const int a = ord[j - 1], b = ord[j];
        const bool za = cnt[a] == 0, zb = cnt[b] == 0;
        bool greater;  // key(a) > key(b)
        if (za != zb) greater = za && !zb;
        else if (negmean[a] != negmean[b]) greater = negmean[a] > negmean[b];
        else greater = a > b;
        if (!greater) break;
        ord[j - 1] = b;
        ord[j] = a;
        --j;
      }
    }
    for (int i = 0; i < 3; ++i) ctl->order[i] = (i < rank) ? pad + ord[i] : 0;
  }
  // plan_levels (predictor.py:122-136): eb / alpha ** (level - 1); the
  // powers come from the host (CPython float pow).
  ctl->nlev = A.nlev;
  for (int lv = 0; lv < CSZI_MAX_LEVELS; ++lv) {
    if (lv < A.nlev) {
      const int level = A.nlev - lv;  // coarse -> fine: level = log2(s) + 1
      const double leb = ddiv(eb_abs, A.alpha_pow[level - 1]);
      ctl->level_eb[lv] = leb;
      ctl->inv_e2[lv] = ddiv(1.0, dmul(2.0, leb));
    } else {
      ctl->level_eb[lv] = 0.0;
      ctl->inv_e2[lv] = 0.0;
    }
  }
  if (!(eb_abs > 0.0)) ctl->flags |= CSZI_F_EB_NONPOSITIVE;
}

int launch_ctl_init(cszi_ctl *ctl, cudaStream_t st) {
  k_ctl_init<<<1, 32, 0, st>>>(ctl);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

int launch_range(const float *x, uint64_t n, cszi_ctl *ctl, cudaStream_t st) {
  const int sms = sm_count();
  u64 blocks = (n / 4 + 255) / 256;
  const u64 cap = (u64)sms * occupancy((const void *)k_range, 256, 0);  // one resident wave
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  k_range<<<(unsigned)blocks, 256, 0, st>>>(x, n, ctl);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

static int tune_args(const cszi_geom *g, const cszi_params *p, TuneArgs &A) {
  for (int a = 0; a < 3; ++a) A.ext[a] = g->ext[a];
  A.rank = g->rank;
  A.pad_axes = 3 - g->rank;
  A.mode_rel = p->mode_rel;
  A.have_variants = p->have_variants;
  A.have_order = p->have_order;
  int nlev = 0;
  for (int64_t s = g->stride / 2; s >= 1; s /= 2) nlev++;
  if (nlev > CSZI_MAX_LEVELS) return CSZI_E_UNSUPPORTED;
  A.nlev = nlev;
  A.eb = p->eb;
  if (!p->have_alpha) return CSZI_E_INVALID_ARG;
  A.alpha = p->alpha;
  for (int i = 0; i < CSZI_MAX_LEVELS; ++i) A.alpha_pow[i] = p->alpha_pow[i];
  for (int a = 0; a < 3; ++a) {
    A.variant[a] = p->variant[a];
    A.order[a] = p->order[a];
  }
  const bool slab = g->slab[1] > g->slab[0];
  A.z0 = slab ? g->slab[0] : 0;
  A.zlo = slab ? g->slab[0] : 0;
  A.zhi = slab ? g->slab[1] : g->ext[0];
  return CSZI_OK;
}

int launch_sample_gather(const float *x, const cszi_geom *g, int32_t *vals, cudaStream_t st,
                         cszi_ctl *reset_ctl) {
  TuneArgs A;
  cszi_params p{};
  p.have_alpha = 1;
  const int rc = tune_args(g, &p, A);
  if (rc != CSZI_OK) return rc;
  k_sample_gather<<<1, 1024, 0, st>>>(x, A, vals, reset_ctl);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

int launch_tune_from_samples(const int32_t *vals, const cszi_geom *g, const cszi_params *p,
                             cszi_ctl *ctl, cudaStream_t st, u64 *zero_hist, int nzero) {
  TuneArgs A;
  const int rc = tune_args(g, p, A);
  if (rc != CSZI_OK) return rc;
  k_tune_decide<<<1, 256, 0, st>>>(vals, A, ctl, zero_hist, zero_hist ? nzero : 0);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? CSZI_OK : CSZI_E_CUDA;
}

// single device: gather (into ctl->scratch-sized device buffer) + decide
int launch_tune(const float *x, const cszi_geom *g, const cszi_params *p, cszi_ctl *ctl,
                int32_t *vals, cudaStream_t st, bool reset_outputs, u64 *zero_hist, int nzero) {
  int rc = launch_sample_gather(x, g, vals, st, reset_outputs ? ctl : nullptr);
  if (rc != CSZI_OK) return rc;
  return launch_tune_from_samples(vals, g, p, ctl, st, zero_hist, nzero);
}

}  // namespace cszi
