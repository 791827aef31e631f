// Pure store-stream rates on this GPU (for the decode write kernels): a
// 268 MB fill with 16-byte streaming / plain stores and cudaMemsetAsync.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o store_rate store_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void fill_cs(uint4 *p, size_t n) {
  const uint4 z = make_uint4(0x02000200u, 0x02000200u, 0x02000200u, 0x02000200u);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(p + i, z);
}
__global__ void fill_st(uint4 *p, size_t n) {
  const uint4 z = make_uint4(0x02000200u, 0x02000200u, 0x02000200u, 0x02000200u);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = z;
}
// warp-contiguous ranges of 16 KB (as k_dec_write_zr: one warp fills its own range)
__global__ void fill_warp_ranges(uint4 *p, size_t n) {
  const size_t w = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const size_t per = 1024;  // uint4 = 16 KB per warp
  const uint4 z = make_uint4(0x02000200u, 0x02000200u, 0x02000200u, 0x02000200u);
  const size_t a = w * per;
  for (size_t i = a + lane; i < a + per && i < n; i += 32) __stcs(p + i, z);
}
int main() {
  const size_t bytes = 268435456, n = bytes / 16;
  uint4 *p;
  cudaMalloc(&p, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int k = 0; k < 4; ++k) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      for (int it = 0; it < 10; ++it) {
        if (k == 0) fill_cs<<<148 * 16, 256>>>(p, n);
        if (k == 1) fill_st<<<148 * 16, 256>>>(p, n);
        if (k == 2) cudaMemsetAsync(p, 0, bytes);
        if (k == 3) fill_warp_ranges<<<(unsigned)((n / 1024 * 32 + 127) / 128), 128>>>(p, n);
      }
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2)
        printf("%s: %.1f us, %.2f TB/s\n", k == 0 ? "stcs grid-stride" : k == 1 ? "st grid-stride" : k == 2 ? "memset" : "stcs 16KB warp ranges",
               ms * 100, bytes / (ms / 10 * 1e-3) / 1e12);
    }
  }
  return 0;
}
