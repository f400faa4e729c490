// Launchers of the complex64 tensor-map apply for one tile width TX (instantiated by tm64.cu / tm32.cu,
// compiled in parallel): RHS groups, epilogue, mass form and weight rule select the kernel variant.
#pragma once
#include "kernels.h"

namespace hz {

template <int TX, int NR, bool COLLOC, int EPI, bool GAM>
static cudaError_t tm_launch_variant(const TmLaunch& L, const ApplyParams<float, float>& p, int nrhs, cudaStream_t s) {
  const int ngroups = (nrhs + NR - 1) / NR;
  auto kern = apply27_tm<TX, NR, COLLOC, EPI, GAM>;
  const size_t smem = tm_smem_bytes(p.tab_n, TX, tm_rows(TX), NR);
  static size_t attr = 0;
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  kern<<<dim3((unsigned)p.tm_nblocks, (unsigned)ngroups), TM_NTHR, smem, s>>>(*L.w, *L.u, p);
  return cudaGetLastError();
}

template <int TX, int NR, bool COLLOC, int EPI>
static cudaError_t tm_launch_rule(const TmLaunch& L, const ApplyParams<float, float>& p, int nrhs, cudaStream_t s) {
  return p.gam != nullptr ? tm_launch_variant<TX, NR, COLLOC, EPI, true>(L, p, nrhs, s)
                          : tm_launch_variant<TX, NR, COLLOC, EPI, false>(L, p, nrhs, s);
}

template <int TX, bool COLLOC, int EPI>
static cudaError_t tm_launch_epi(const TmLaunch& L, ApplyParams<float, float> p, int nrhs, cudaStream_t s) {
  p.nrhs = nrhs;
  if constexpr (EPI == EPI_PLAIN) {
    if (tm_group(nrhs, EPI) == 2) return tm_launch_rule<TX, 2, COLLOC, EPI>(L, p, nrhs, s);
  }
  return tm_launch_rule<TX, 1, COLLOC, EPI>(L, p, nrhs, s);
}

template <int TX>
cudaError_t launch_apply_tm_tx(const TmLaunch& L, const ApplyParams<float, float>& p, int nrhs, bool colloc, int epi,
                               cudaStream_t s) {
  switch (epi) {
    case EPI_PLAIN: return colloc ? tm_launch_epi<TX, true, EPI_PLAIN>(L, p, nrhs, s) : tm_launch_epi<TX, false, EPI_PLAIN>(L, p, nrhs, s);
    case EPI_DOT1: return colloc ? tm_launch_epi<TX, true, EPI_DOT1>(L, p, nrhs, s) : tm_launch_epi<TX, false, EPI_DOT1>(L, p, nrhs, s);
    case EPI_DOT4: return colloc ? tm_launch_epi<TX, true, EPI_DOT4>(L, p, nrhs, s) : tm_launch_epi<TX, false, EPI_DOT4>(L, p, nrhs, s);
  }
  return cudaErrorInvalidValue;
}

template <int TX>
int tm_occupancy_tx(int tab_n, int nr) {
  int nb = 0;
  if (nr == 1)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, apply27_tm<TX, 1, false, EPI_DOT4, false>, TM_NTHR,
                                                  tm_smem_bytes(tab_n, TX, tm_rows(TX), 1));
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, apply27_tm<TX, 2, false, EPI_PLAIN, false>, TM_NTHR,
                                                  tm_smem_bytes(tab_n, TX, tm_rows(TX), 2));
  return nb > 0 ? nb : 1;
}

}  // namespace hz
