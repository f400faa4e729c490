// Launchers of the complex64 tensor-map apply for one tile width TX (instantiated by tm64.cu / tm32.cu,
// compiled in parallel): epilogue, mass form and weight rule select the kernel variant.
#pragma once
#include "kernels.h"

namespace hz {

template <int TX, bool COLLOC, int EPI, bool GAM>
static cudaError_t tm_launch_variant(const TmLaunch& L, const ApplyParams<float, float>& p, cudaStream_t s) {
  auto kern = apply27_tm<TX, COLLOC, EPI, GAM>;
  const size_t smem = tm_smem_bytes(p.tab_n, TX, tm_rows(TX), epi_k(EPI) > 0);
  static size_t attr = 0;
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  kern<<<(unsigned)p.tm_nblocks, TM_NTHR, smem, s>>>(*L.w, *L.u, L.r ? *L.r : *L.u, p);
  return cudaGetLastError();
}

template <int TX, bool COLLOC, int EPI>
static cudaError_t tm_launch_rule(const TmLaunch& L, const ApplyParams<float, float>& p, cudaStream_t s) {
  return p.gam != nullptr ? tm_launch_variant<TX, COLLOC, EPI, true>(L, p, s)
                          : tm_launch_variant<TX, COLLOC, EPI, false>(L, p, s);
}

template <int TX>
cudaError_t launch_apply_tm_tx(const TmLaunch& L, const ApplyParams<float, float>& p0, int nrhs, bool colloc, int epi,
                               cudaStream_t s) {
  ApplyParams<float, float> p = p0;
  p.nrhs = nrhs;
  switch (epi) {
    case EPI_PLAIN: return colloc ? tm_launch_rule<TX, true, EPI_PLAIN>(L, p, s) : tm_launch_rule<TX, false, EPI_PLAIN>(L, p, s);
    case EPI_DOT1: return colloc ? tm_launch_rule<TX, true, EPI_DOT1>(L, p, s) : tm_launch_rule<TX, false, EPI_DOT1>(L, p, s);
    case EPI_DOT4: return colloc ? tm_launch_rule<TX, true, EPI_DOT4>(L, p, s) : tm_launch_rule<TX, false, EPI_DOT4>(L, p, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hz
