#include <cstdio>
#include <cstdlib>
#include <cudaTypedefs.h>
#include <cuda.h>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void tload2(uint32_t dst, const void* map, uint32_t bar, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
               ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1) : "memory");
}
template <int MODE>
__global__ void k(const __grid_constant__ CUtensorMap m, const CUtensorMap* gm, float* out) {
  __shared__ __align__(128) float buf[16 * 16];
  __shared__ __align__(8) uint64_t bar;
  uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar), d = (uint32_t)__cvta_generic_to_shared(buf);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(16 * 16 * 4) : "memory");
    tload2(d, MODE == 0 ? (const void*)&m : (const void*)gm, b, MODE == 2 ? -4 : (MODE == 3 ? 60 : 0), MODE == 1 ? -1 : (MODE == 3 ? -3 : 0));
  }
  __syncthreads();
  asm volatile("{\n .reg .pred P1;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra W_%=;\n}\n" ::"r"(b), "r"(0) : "memory");
  out[threadIdx.x] = buf[threadIdx.x];
}
int main() {
  float* g; CK(cudaMalloc(&g, 64 * 64 * 4));
  float h[64 * 64]; for (int i = 0; i < 64 * 64; i++) h[i] = i;
  CK(cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice));
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q));
  printf("query %d fn %p\n", (int)q, fn);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap m;
  cuuint64_t d[2] = {64, 64}; cuuint64_t s[1] = {64 * 4}; cuuint32_t bx[2] = {16, 16}, e[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, d, s, bx, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("enc %d\n", (int)r);
  CUtensorMap* gm; CK(cudaMalloc(&gm, sizeof(CUtensorMap))); CK(cudaMemcpy(gm, &m, sizeof(m), cudaMemcpyHostToDevice));
  float* out; CK(cudaMalloc(&out, 256 * 4));
  for (int mode = 0; mode < 4; mode++) {
    if (mode == 0) k<0><<<1, 256>>>(m, gm, out);
    if (mode == 1) k<1><<<1, 256>>>(m, gm, out);
    if (mode == 2) k<2><<<1, 256>>>(m, gm, out);
    if (mode == 3) k<3><<<1, 256>>>(m, gm, out);
    cudaError_t er = cudaDeviceSynchronize();
    float o[256]; cudaMemcpy(o, out, sizeof(o), cudaMemcpyDeviceToHost);
    printf("mode %d: %s  out[0]=%g out[17]=%g out[255]=%g\n", mode, cudaGetErrorString(er), o[0], o[17], o[255]);
    if (er != cudaSuccess) return 1;
  }
  return 0;
}
