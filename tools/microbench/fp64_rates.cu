// Microbenchmark: FP64 pipe and conversion throughput on the B200 (sm_100a).
// Measures ops/clk/SM for DADD, DMUL, F2F.F64.F32, F2F.F32.F64, trunc, DDIV.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
#define CHAINS 8

__global__ void k_dadd(double* out, double a) {
  double x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = __dadd_rn(x[c], a);
  double s = 0; for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_dmul(double* out, double a) {
  double x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = __dmul_rn(x[c], a);
  double s = 0; for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_dfma(double* out, double a) {
  double x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = __fma_rn(x[c], a, a);
  double s = 0; for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 1.2345) out[0] = s;
}
// f32 -> f64 -> f32 round trip chain (two conversions per step)
__global__ void k_cvt(double* out, float a) {
  float x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      double d = (double)x[c];
      x[c] = __double2float_rn(d + 0.0) ;
    }
  float s = 0; for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 1.2345f) out[0] = s;
}
__global__ void k_f2d(double* out, float a) {
  double x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = 0;
  float v = threadIdx.x * 1e-3f;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      x[c] = (double)__int_as_float(__float_as_int(v) ^ __double2loint(x[c]));
    }
  }
  double s = 0; for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_trunc(double* out, double a) {
  double x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c + 0.5;
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = trunc(x[c]) + a;
  double s = 0; for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_ddiv(double* out, double a) {
  double x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c + 1.0;
  for (int i = 0; i < ITERS / 8; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = __ddiv_rn(x[c], a);
  double s = 0; for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_iadd(double* out, int a) {
  uint32_t x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x + c;
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = (x[c] ^ a) + 0x9e3779b9u;
  uint32_t s = 0; for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345) out[0] = s;
}

template <typename K, typename A>
void run(const char* name, K k, A a, double ops_per_thread_iter, double div) {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  double* out; cudaMalloc(&out, 8);
  int blocks = p.multiProcessorCount * 8, threads = 256;
  k<<<blocks, threads>>>(out, a);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<<<blocks, threads>>>(out, a);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
  double ops = (double)blocks * threads * (ITERS / div) * CHAINS * ops_per_thread_iter;
  double gops = ops / (ms * 1e-3) / 1e9;
  printf("%-10s %8.3f ms  %10.1f Gop/s  %6.2f op/clk/SM (at max clk %d MHz)\n", name, ms, gops,
         gops * 1e9 / (p.multiProcessorCount * (clk_khz * 1e3)), clk_khz / 1000);
  cudaFree(out);
}

int main() {
  run("dadd", k_dadd, 1.0000001, 1, 1);
  run("dmul", k_dmul, 1.0000001, 1, 1);
  run("dfma", k_dfma, 1.0000001, 1, 1);
  run("cvt_rt", k_cvt, 1.0f, 2, 1);
  run("f2d", k_f2d, 1.0f, 1, 1);
  run("trunc+add", k_trunc, 0.25, 1, 1);
  run("ddiv", k_ddiv, 1.0000001, 1, 8);
  run("iadd+xor", k_iadd, 7, 2, 1);
  return 0;
}
