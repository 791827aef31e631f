// Shared device utilities for libcszi (sm_100a): warp/block scans, the
// decoupled look-back used by every stream-compaction stage (bit offsets,
// outlier positions, pass-2 segments), exact-rounding fp64 helpers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "cszi.h"

#define DEV __device__ __forceinline__
#define CSZI_FULL 0xffffffffu

namespace cszi {

typedef unsigned long long u64;

// Host-side count of kernels this library launched (cszi_launch_count()).
void note_launch(int n = 1);
// Reset the output fields of ctl, keeping the range (and tuned config) of a
// prior scan: one thread.
DEV void ctl_reset_outputs(cszi_ctl *ctl) {
  ctl->bits = 0;
  ctl->n_outliers = 0;
  ctl->raw_len = 0;
  ctl->payload_len = 0;
  ctl->decoded_symbols = 0;
  ctl->flags = 0;
  ctl->max_len = 0;
  for (int i = 0; i < 8; ++i) ctl->scratch[i] = 0;
}
// Host-side launch helpers with per-device caches (the runtime queries cost
// microseconds of CPU each, and the GPU idles while the host launches the
// first kernels of a call): SM count, the dynamic shared-memory opt-in
// (raised only when a larger size is requested) and occupancy.
int sm_count();
void ensure_smem(const void *fn, size_t smem);
int occupancy(const void *fn, int threads, size_t smem);

// ---------------------------------------------------------------------------
// memory-model helpers (release/acquire at gpu scope)
// ---------------------------------------------------------------------------
DEV void st_release(u64 *p, u64 v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
DEV u64 ld_acquire(const u64 *p) {
  u64 v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// relaxed (no fence) variants for look-back status words: the 64-bit word
// carries flag and value together, so no other data is ordered by it.
DEV void st_relaxed(u64 *p, u64 v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
DEV u64 ld_relaxed(const u64 *p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
DEV uint32_t ld_volatile_u32(const uint32_t *p) { return *(const volatile uint32_t *)p; }

DEV uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// Order-preserving key of a float (for atomicMin/atomicMax on raw bits).
__host__ __device__ __forceinline__ uint32_t float_key(float f) {
#ifdef __CUDA_ARCH__
  uint32_t b = __float_as_uint(f);
#else
  uint32_t b;
  __builtin_memcpy(&b, &f, 4);
#endif
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__host__ __device__ __forceinline__ float key_float(uint32_t k) {
  uint32_t b = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
#ifdef __CUDA_ARCH__
  return __uint_as_float(b);
#else
  float f;
  __builtin_memcpy(&f, &b, 4);
  return f;
#endif
}

// ---------------------------------------------------------------------------
// scans
// ---------------------------------------------------------------------------
template <typename T>
DEV T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T t = __shfl_up_sync(CSZI_FULL, v, o);
    if (lane >= o) v += t;
  }
  return v;
}
template <typename T>
DEV T warp_incl_max(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T t = __shfl_up_sync(CSZI_FULL, v, o);
    if (lane >= o && t > v) v = t;
  }
  return v;
}
template <typename T>
DEV T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(CSZI_FULL, v, o);
  return v;
}

// Block-wide exclusive scan; `ws` holds NT/32 elements; returns the
// exclusive prefix of the calling thread and the block total in `total`.
template <int NT, typename T>
DEV T block_excl_scan(T v, T *ws, T &total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T inc = warp_incl_scan(v);
  if (lane == 31) ws[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = (lane < NT / 32) ? ws[lane] : T(0);
    T wi = warp_incl_scan(w);
    if (lane < NT / 32) ws[lane] = wi - w;
    if (lane == NT / 32 - 1) ws[NT / 32] = wi;
  }
  __syncthreads();
  T excl = ws[warp] + inc - v;
  total = ws[NT / 32];
  __syncthreads();
  return excl;
}

// ---------------------------------------------------------------------------
// decoupled look-back (single-pass chained scan across tiles).  Status words
// are published / polled with relaxed 64-bit accesses (flag and value in one
// single-copy-atomic word; nothing else is ordered by them).
// status word: [63:62] flag (0 invalid, 1 aggregate, 2 inclusive), [61:0] value
// Must be called by all 32 lanes of ONE warp; tiles must be processed in
// ticket order (tile t only waits on tiles < t, which started earlier).
// ---------------------------------------------------------------------------
constexpr u64 LB_AGG = 1ull << 62;
constexpr u64 LB_INC = 2ull << 62;
constexpr u64 LB_VAL = (1ull << 62) - 1;

template <typename T>
DEV T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const T t = __shfl_xor_sync(CSZI_FULL, v, o);
    v = t > v ? t : v;
  }
  return v;
}

// MAX = false: prefix sums; MAX = true: prefix maxima (values < 2^62).
// Each lane polls LB_PER_LANE consecutive predecessors per round trip.
constexpr int LB_PER_LANE = 1;

template <bool MAX = false>
DEV u64 lookback_exclusive(u64 *status, u64 tile, u64 aggregate) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_relaxed(&status[0], LB_INC | aggregate);
    return 0;
  }
  if (lane == 0) st_relaxed(&status[tile], LB_AGG | aggregate);
  u64 excl = 0;
  long long top = (long long)tile - 1;
  for (;;) {
    u64 s[LB_PER_LANE];
#pragma unroll
    for (int k = 0; k < LB_PER_LANE; ++k) {
      const long long idx = top - (lane * LB_PER_LANE + k);
      s[k] = (idx >= 0) ? ld_relaxed(&status[idx]) : LB_INC;
    }
    // nearest inclusive prefix inside this lane's group, and whether an
    // unpublished tile sits before it
    int fk = LB_PER_LANE;
    bool inv = false;
    u64 v = 0;
#pragma unroll
    for (int k = LB_PER_LANE - 1; k >= 0; --k) {
      const uint32_t f = (uint32_t)(s[k] >> 62);
      if (f == 2) {
        fk = k;
        inv = false;
        v = s[k] & LB_VAL;
      } else {
        inv = inv || f == 0;
        const u64 x = s[k] & LB_VAL;
        v = MAX ? (x > v ? x : v) : v + x;
      }
    }
    // v now folds the group up to and including its first inclusive entry
    // (entries after it were discarded when it was found)
    const uint32_t inc_mask = __ballot_sync(CSZI_FULL, fk < LB_PER_LANE);
    const int first_lane = inc_mask ? (__ffs(inc_mask) - 1) : 32;
    const uint32_t inv_mask = __ballot_sync(CSZI_FULL, inv && lane <= first_lane);
    if (inv_mask) continue;  // a predecessor has not published yet: re-poll
    if (lane > first_lane) v = 0;
    if (MAX) {
      v = warp_max(v);
      excl = v > excl ? v : excl;
    } else {
      excl += warp_sum(v);
    }
    if (inc_mask) break;
    top -= 32 * LB_PER_LANE;
  }
  const u64 inc = MAX ? (aggregate > excl ? aggregate : excl) : excl + aggregate;
  if (lane == 0) st_relaxed(&status[tile], LB_INC | inc);
  return excl;
}

// ---------------------------------------------------------------------------
// exact fp64 helpers (numpy float64 semantics, never contracted)
// ---------------------------------------------------------------------------
DEV double dadd(double a, double b) { return __dadd_rn(a, b); }
DEV double dsub(double a, double b) { return __dsub_rn(a, b); }
DEV double dmul(double a, double b) { return __dmul_rn(a, b); }
DEV double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// float -> double, exact (F2F.F64.F32: 16/clk/SM on B200 — a separate pipe
// from the fp64 FMA unit; the predictor is issue-bound, so one conversion
// beats the six-instruction integer rebias).
DEV double f2d(float f) { return (double)f; }

}  // namespace cszi
