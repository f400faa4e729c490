// minimal 1-D tensor-map TMA load test
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
struct __align__(64) Maps { CUtensorMap m[2]; int off; };
__global__ void k(const __grid_constant__ Maps maps, int c, double* out, int which) {
  __shared__ __align__(1024) double buf[256];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar)), "r"(130 * 8) : "memory");
    asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
                 ::"r"(s32(buf)), "l"(reinterpret_cast<uint64_t>(&maps.m[which])), "r"(c + maps.off), "r"(s32(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::"r"(s32(&bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < 130; i += blockDim.x) out[i] = buf[i];
}
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  const int n = 100000;
  double* d; cudaMalloc(&d, (n + 16) * 8);
  double* h = new double[n]; for (int i = 0; i < n; i++) h[i] = i;
  cudaMemcpy(d, h, n * 8, cudaMemcpyHostToDevice);
  double* out; cudaMalloc(&out, 256 * 8);
  void* f = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  printf("entry %p q=%d\n", f, (int)q);
  Enc enc = (Enc)f;
  Maps maps; memset(&maps, 0, sizeof(maps));
  cuuint64_t dim[1] = {(cuuint64_t)n}, str[1] = {0}; cuuint32_t box[1] = {130}, es[1] = {1};
  CUresult r = enc(&maps.m[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, d, dim, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  maps.m[1] = maps.m[0]; maps.off = 0;
  for (int c : {0, 1, 12345}) {
    k<<<1, 128>>>(maps, c, out, 1);
    cudaError_t e = cudaDeviceSynchronize();
    double o[130]; cudaMemcpy(o, out, sizeof(o), cudaMemcpyDeviceToHost);
    printf("c=%d err=%s out[0]=%g out[129]=%g\n", c, cudaGetErrorString(e), o[0], o[129]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
