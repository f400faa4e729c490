// Debug harness for apply27_tm: one tiny launch with hand-built tensor maps (no libhz).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cudaTypedefs.h>
#include "apply27_tm.cuh"
using namespace hz;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

int main(int argc, char** argv) {
  const int nx = argc > 1 ? atoi(argv[1]) : 5, ny = argc > 2 ? atoi(argv[2]) : 4, nz = argc > 3 ? atoi(argv[3]) : 3;
  const int ldx = (nx + 3) & ~3;
  const int ntx = (ldx + 1 + 63) / 64;
  int tx = argc > 6 ? atoi(argv[6]) : 64;
  const int mode = argc > 7 ? atoi(argv[7]) : 0;
  const int ty = tm_rows(tx);
  const int nblk = argc > 5 ? atoi(argv[5]) : 148;
  const long long plane = (long long)ldx * ny, fstride = plane * (nz + 2);
  printf("nx %d ldx %d tx %d ty %d\n", nx, ldx, tx, ty);
  const int nr = argc > 9 ? atoi(argv[9]) : 1;
  const int ng = argc > 10 ? atoi(argv[10]) : 1;   // RHS groups (grid.y)
  float* w; float2* u; float2* au; float* ctab;
  CK(cudaMalloc(&w, fstride * 4)); CK(cudaMalloc(&u, fstride * 8 * nr * ng)); CK(cudaMalloc(&au, fstride * 8 * nr * ng));
  CK(cudaMemset(w, 0, fstride * 4)); CK(cudaMemset(u, 0, fstride * 8 * nr * ng)); CK(cudaMemset(au, 0, fstride * 8 * nr * ng));
  const int rnd = argc > 8 ? atoi(argv[8]) : 0;
  std::vector<float> wh(fstride, 1.0f / (3000.f * 3000.f));
  if (rnd) { unsigned st = 1; for (auto& v : wh) { st = st * 1664525u + 1013904223u; float vv = 2100.f + 3900.f * (st >> 8) / 16777216.f; v = 1.f / (vv * vv); } }
  CK(cudaMemcpy(w, wh.data(), fstride * 4, cudaMemcpyHostToDevice));
  const int tab_n = rnd ? 200 : 4;
  std::vector<float> ct(tab_n * 12, 0.01f);
  CK(cudaMalloc(&ctab, ct.size() * 4)); CK(cudaMemcpy(ctab, ct.data(), ct.size() * 4, cudaMemcpyHostToDevice));
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q));
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap mw, mu;
  const int org = 1, nval = nz;
  {
    cuuint64_t d[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nval};
    cuuint64_t s[2] = {(cuuint64_t)ldx * 4, (cuuint64_t)plane * 4};
    cuuint32_t b[3] = {(cuuint32_t)tm_bxw(tx), (cuuint32_t)ty + 2, 1};
    cuuint32_t e[3] = {1, 1, 1};
    CUresult r = enc(&mw, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, w + org * plane, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("enc w %d\n", (int)r);
  }
  {
    cuuint64_t d[4] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nval, (cuuint64_t)(nr * ng)};
    cuuint64_t s[3] = {(cuuint64_t)ldx * 8, (cuuint64_t)plane * 8, (cuuint64_t)fstride * 8};
    cuuint32_t b[4] = {(cuuint32_t)tm_bxu(tx), (cuuint32_t)ty + 2, 1, 1};
    cuuint32_t e[4] = {1, 1, 1, 1};
    CUresult r = enc(&mu, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, u + org * plane, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("enc u %d\n", (int)r);
  }
  ApplyParams<float, float> p;
  memset(&p, 0, sizeof(p));
  p.nx = nx; p.ny = ny; p.ldx = ldx; p.nzl = nz; p.z0 = 0; p.nzg = nz; p.plane = plane; p.fstride = fstride;
  p.tm_tx = tx; p.tm_ty = ty; p.tm_org = org; p.nrhs = nr * ng;
  p.w = w; p.u = u; p.au = au; p.ctab = ctab; p.tab_lo = 0; p.tab_n = tab_n; p.n_g = tab_n;
  p.inv_fh = 1.f / (10.f * 25.f); p.inv_dg = 10.f; p.g_min = 4.f; p.ih2 = 1.f / 400.f; p.w2 = 1000.f;
  p.invih2 = 400.f; p.inv2ih2 = 200.f; p.inv3ih2 = 133.f;
  p.lo[0] = p.lo[1] = p.lo[2] = 0; p.hi[0] = nx - 1; p.hi[1] = ny - 1; p.hi[2] = nz - 1;
  if (mode) { p.lo[0] = p.lo[1] = p.lo[2] = 2; p.hi[0] = nx - 3; p.hi[1] = ny - 3; p.hi[2] = nz - 3; }
  float2* dd; CK(cudaMalloc(&dd, 6 * 4096 * 8)); CK(cudaMemset(dd, 0, 6 * 4096 * 8));
  for (int a = 0; a < 3; a++) { p.dm[a] = dd + a * 4096; p.dp[a] = dd + (3 + a) * 4096; }
  std::vector<int4> items;
  for (int y0 = 0; y0 < ny; y0 += ty)
    for (int x0 = 0; x0 < ntx * tx; x0 += tx) items.push_back(tm_item(x0, y0, 0, nz, mode));
  int4* wk; CK(cudaMalloc(&wk, items.size() * sizeof(int4)));
  CK(cudaMemcpy(wk, items.data(), items.size() * sizeof(int4), cudaMemcpyHostToDevice));
  p.tm_work = wk; p.tm_nitems = (int)items.size(); p.tm_nblocks = std::min((int)items.size(), nblk / ng);
  const int gam = argc > 4 ? atoi(argv[4]) : 0;
  float* gm; CK(cudaMalloc(&gm, 5 * fstride * 4)); CK(cudaMemset(gm, 0, 5 * fstride * 4));
  if (gam) p.gam = gm;
  auto kern = nr == 2 ? apply27_tm<64, 2, false, EPI_PLAIN, false> : (gam ? apply27_tm<64, 1, false, EPI_PLAIN, true> : apply27_tm<64, 1, false, EPI_PLAIN, false>);
  const size_t smem = tm_smem_bytes(tab_n, tx, ty, nr);
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  printf("launch %zu items smem %zu\n", items.size(), smem);
  kern<<<dim3((unsigned)p.tm_nblocks, (unsigned)ng), TM_NTHR, smem>>>(mw, mu, p);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int it = 0; it < 5; it++) {
    cudaEventRecord(e0); kern<<<dim3((unsigned)p.tm_nblocks, (unsigned)ng), TM_NTHR, smem>>>(mw, mu, p); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  printf("OK %.3f ms  %.1f Gpts/s  %.0f GB/s\n", best, (double)nx * ny * nz / best / 1e6, (double)nx * ny * nz * 20 / best / 1e6);
  return 0;
}
