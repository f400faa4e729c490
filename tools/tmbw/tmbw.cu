// TMA streaming microbenchmark: the apply's producer/consumer ring without the stencil arithmetic, to
// measure the bandwidth a box geometry reaches.  Usage: tmbw BOXW BOXH STAGES NTHR [nx ny nz]
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cudaTypedefs.h>
#include <cuda.h>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(c) : "memory"); }
__device__ __forceinline__ void mbar_tx(uint32_t bar, uint32_t b) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(b) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t ph) {
  asm volatile("{\n .reg .pred P1;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra W_%=;\n}\n" ::"r"(bar), "r"(ph) : "memory");
}
__device__ __forceinline__ void tload3(uint32_t dst, const void* m, uint32_t bar, int a, int b, int c) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst), "l"((uint64_t)m), "r"(bar), "r"(a), "r"(b), "r"(c) : "memory");
}

__global__ void k(const __grid_constant__ CUtensorMap m, int bw, int bh, int S, int ntx, int nty, int nz, float* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t ring = bar0 + 1024;
  const uint32_t stB = ((uint32_t)bw * bh * 8 + 127) & ~127u;
  const int ntiles = ntx * nty;
  // each CTA: tiles blockIdx.x, +gridDim.x ...; each tile all nz planes
  int p_t = blockIdx.x, p_z = 0, p_st = 0;
  auto issue = [&]() {
    if (p_t >= ntiles) return;
    const uint32_t b = bar0 + 8 * p_st;
    mbar_tx(b, bw * bh * 8);
    tload3(ring + p_st * stB, &m, b, (p_t % ntx) * (bw - 2) - 2, (p_t / ntx) * (bh - 2) - 1, p_z);
    if (++p_st == S) p_st = 0;
    if (++p_z == nz) { p_z = 0; p_t += gridDim.x; }
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; s++) mbar_init(bar0 + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < S; s++) issue();
  }
  __syncthreads();
  float acc = 0.f;
  int c_st = 0; uint32_t ph = 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x)
    for (int z = 0; z < nz; z++) {
      mbar_wait(bar0 + 8 * c_st, ph);
      const float* f = reinterpret_cast<const float*>(sm + 1024 + c_st * stB);
      acc += f[threadIdx.x % (bw * bh)];
      if (warp == 0) { asm volatile("bar.sync %0, %1;" ::"r"(1 + c_st), "r"(blockDim.x) : "memory"); if (lane == 0) issue(); }
      else asm volatile("bar.arrive %0, %1;" ::"r"(1 + c_st), "r"(blockDim.x) : "memory");
      if (++c_st == S) { c_st = 0; ph ^= 1; }
    }
  if (acc == 12345.f) out[0] = acc;
}

int main(int argc, char** argv) {
  const int bw = atoi(argv[1]), bh = atoi(argv[2]), S = atoi(argv[3]), nthr = atoi(argv[4]);
  const int nx = argc > 5 ? atoi(argv[5]) : 804, ny = argc > 6 ? atoi(argv[6]) : 801, nz = argc > 7 ? atoi(argv[7]) : 189;
  const size_t n = (size_t)nx * ny * nz;
  double* g; CK(cudaMalloc(&g, n * 8)); CK(cudaMemset(g, 0, n * 8));
  float* out; CK(cudaMalloc(&out, 4));
  void* fn; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q));
  CUtensorMap m;
  cuuint64_t d[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz}, s[2] = {(cuuint64_t)nx * 8, (cuuint64_t)nx * ny * 8};
  cuuint32_t b[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 1}, e[3] = {1, 1, 1};
  CUresult r = ((PFN_cuTensorMapEncodeTiled_v12000)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, g, d, s, b, e,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) { printf("enc %d\n", r); return 1; }
  const int ntx = (nx + bw - 3) / (bw - 2), nty = (ny + bh - 3) / (bh - 2);
  const size_t smem = 1024 + (size_t)S * (((size_t)bw * bh * 8 + 127) & ~127);
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int nb = 0; CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, nthr, smem));
  const int grid = 148 * nb;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 2; it++) k<<<grid, nthr, smem>>>(m, bw, bh, S, ntx, nty, nz, out);
  CK(cudaDeviceSynchronize());
  float best = 1e9;
  for (int it = 0; it < 5; it++) {
    cudaEventRecord(e0); k<<<grid, nthr, smem>>>(m, bw, bh, S, ntx, nty, nz, out); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  const double useful = (double)n * 8, moved = (double)ntx * nty * nz * bw * bh * 8;
  printf("box %dx%d S=%d thr=%d ctas/SM=%d: %.3f ms, useful %.0f GB/s, box bytes %.0f GB/s\n", bw, bh, S, nthr, nb, best,
         useful / best / 1e6, moved / best / 1e6);
  return 0;
}
