// Probe: 3-D TMA load of a (36, 9, 9) float box into shared memory.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <vector>
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap tm, float *out, int c0, int c1, int c2, int align) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t mbar;
  unsigned char *sm = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u) + align;
  float *buf = (float *)sm;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(36 * 81 * 4) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(smem_u32(buf)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(&mbar)) : "memory");
  }
  __syncthreads();
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(smem_u32(&mbar)) : "memory");
  for (int i = threadIdx.x; i < 36 * 81; i += blockDim.x) out[i] = buf[i];
}
typedef CUresult (*Fn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                       const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                       CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  const int n = 64;
  std::vector<float> h(n * n * n);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  float *d, *o;
  cudaMalloc(&d, h.size() * 4);
  cudaMalloc(&o, 36 * 81 * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void *p; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  Fn fn = (Fn)p;
  CUtensorMap tm;
  cuuint64_t dims[3] = {64, 64, 64}, str[2] = {64 * 4, 64 * 64 * 4};
  cuuint32_t box[3] = {36, 9, 9}, es[3] = {1, 1, 1};
  CUresult r = fn(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  for (int align : {0, 16, 64}) {
    for (int c0 : {0, 32}) {
      k<<<1, 128, 36 * 81 * 4 + 256>>>(tm, o, c0, 8, 8, align);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<float> ho(36 * 81);
      cudaMemcpy(ho.data(), o, ho.size() * 4, cudaMemcpyDeviceToHost);
      printf("align %d c0 %d: %s  first %g (want %g) last-row x35 %g\n", align, c0, cudaGetErrorString(e), ho[0],
             (float)(8 * 4096 + 8 * 64 + c0), ho[35]);
      if (e) return 1;
    }
  }
  return 0;
}
