// 2-D tensor-map TMA load with an odd (not 16-byte aligned) innermost start coordinate: complex64 and
// float32 maps of a pitched [ny][ldx] array, box starting at x0 - 1 (and negative coordinates)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstring>
__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int ESZ>
__global__ void k(const __grid_constant__ CUtensorMap m, int c0, int c1, float* out, int nbytes) {
  __shared__ __align__(1024) float buf[4096];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar)), "r"(nbytes) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(s32(buf)), "l"(reinterpret_cast<uint64_t>(&m)), "r"(c0), "r"(c1), "r"(s32(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::"r"(s32(&bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < nbytes / 4; i += blockDim.x) out[i] = buf[i];
}
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  const int nx = 801, ldx = 804, ny = 50;
  float* d; cudaMalloc(&d, (size_t)ldx * ny * 8);
  float* h = new float[(size_t)ldx * ny * 2];
  for (int i = 0; i < ldx * ny * 2; i++) h[i] = (float)i;
  cudaMemcpy(d, h, (size_t)ldx * ny * 8, cudaMemcpyHostToDevice);
  float* out; cudaMalloc(&out, 4096 * 4);
  void* f = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  Enc enc = (Enc)f;
  int bad = 0;
  for (int esz : {8, 4}) {
    CUtensorMap m; memset(&m, 0, sizeof(m));
    const int bx = esz == 8 ? 66 : 68, by = 14;
    cuuint64_t dim[2] = {(cuuint64_t)nx, (cuuint64_t)ny}, str[1] = {(cuuint64_t)ldx * esz};
    cuuint32_t box[2] = {(cuuint32_t)bx, (cuuint32_t)by}, es[2] = {1, 1};
    CUresult r = enc(&m, esz == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dim, str, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("esz %d encode %d\n", esz, (int)r);
    for (int c0 : {-1, 63, 127, 767, 0, 1, 3}) for (int c1 : {-1, 5}) {
      const int nb = bx * by * esz;
      if (esz == 8) k<8><<<1, 128>>>(m, c0, c1, out, nb); else k<4><<<1, 128>>>(m, c0, c1, out, nb);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("esz %d c0 %d c1 %d: %s\n", esz, c0, c1, cudaGetErrorString(e)); return 1; }
      float o[4096]; cudaMemcpy(o, out, nb, cudaMemcpyDeviceToHost);
      int err = 0;
      for (int yy = 0; yy < by; yy++) for (int xx = 0; xx < bx; xx++) {
        const int gx = c0 + xx, gy = c1 + yy;
        const bool in = gx >= 0 && gx < nx && gy >= 0 && gy < ny;
        for (int p = 0; p < esz / 4; p++) {
          const float want = in ? h[((size_t)gy * ldx + gx) * (esz / 4) + p] : 0.f;
          if (o[(yy * bx + xx) * (esz / 4) + p] != want) err++;
        }
      }
      printf("esz %d c0 %d c1 %d: mismatches %d\n", esz, c0, c1, err);
      bad += err;
    }
  }
  printf(bad ? "FAIL\n" : "PASS\n");
  return bad != 0;
}
