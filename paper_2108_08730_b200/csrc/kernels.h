// Launch interface between the ABI layer (api.cu) and the kernels (kernels.cu).
#pragma once
#include <cuda_runtime.h>

#include "apply.cuh"
#include "apply27.cuh"
#include "apply27_tm.cuh"

namespace hz {

// Per-RHS BiCGSTAB scalars on the device (see bicg_* kernels for who writes what).
struct SolverState {
  double rho_next[2];  // ρ for the next α (written by update / init / rho_reset)
  double rho_used[2];  // ρ used by the last α (written by s-kernel, read by update)
  double alpha[2];
  double omega[2];
  int flags;           // bit 0: breakdown detected
  int pad;
};

template <typename R>
struct VecParams {
  typedef typename Cx<R>::T C;
  long long n;        // owned storage elements per RHS (nzl*plane, pad columns included: they stay 0)
  long long plane;    // halo-plane offset
  long long fstride;  // per-RHS stride
  int nblocks;        // CTAs per RHS
  C *x, *r, *rhat, *p, *v, *t;
  C* xlo;              // compensation term of the iterate (complex64 solver) or null
  C *r1, *r2;          // BiCGStab(2) only: A-images of r0 (= r) within one outer step
  const C *ph, *sh;    // right-preconditioned BiCGSTAB: x += α M⁻¹p + ω M⁻¹s (null: x += α p + ω s)
  const double* dotA;  // [nrhs][2]
  const double* dotB;  // [nrhs][7]
  double* dotR;        // [nrhs][3]
  double* dotG;        // BiCGStab(2) only: [nrhs] ‖r1‖²
  double* partials;
  unsigned int* tickets;
  SolverState* state;
  const int* active;
};

enum { BICG_INIT = 0, BICG_S = 1, BICG_UPDATE = 2, BICG_RHO_RESET = 3 };
// BiCGStab(2) vector steps (bicgl_kernel): one outer step = BCL_A, apply, BCL_B, apply, BCL_C, apply,
// BCL_D, apply (DOT4), BCL_E
enum { BCL_INIT = 0, BCL_A = 1, BCL_B = 2, BCL_C = 3, BCL_D = 4, BCL_E = 5 };

int apply_last_launches();   // kernels launched by the last apply launch on this thread (1 or 2)
// register path (R = double): complex128 and the fp64 residual of the complex64 solver
template <typename R> int apply_occupancy(bool colloc);
template <typename R> long long apply_nblocks_x(int nx, int ny);   // CTAs along x of one z-chunk
template <typename R, typename S> long long apply_plan(ApplyParams<R, S>& p);   // CTAs per RHS, both launches
template <typename R, typename S>
cudaError_t launch_apply(const ApplyParams<R, S>& p, int nrhs, bool colloc, int epi, cudaStream_t s);
template <>
cudaError_t launch_apply<double, double>(const ApplyParams<double, double>& p, int nrhs, bool colloc, int epi,
                                         cudaStream_t s);
template <>
cudaError_t launch_apply<double, float>(const ApplyParams<double, float>& p, int nrhs, bool colloc, int epi,
                                        cudaStream_t s);
// complex64 tensor-map apply (apply27_tm): the tensor maps of the launch (w, u of this call, and r̂₀ of
// the dot epilogues — null for the plain apply)
struct TmLaunch {
  const CUtensorMap* w;
  const CUtensorMap* u;
  const CUtensorMap* r;
};
template <int TX>
cudaError_t launch_apply_tm_tx(const TmLaunch& L, const ApplyParams<float, float>& p, int nrhs, bool colloc, int epi,
                               cudaStream_t s);
cudaError_t launch_apply_tm(const TmLaunch& L, const ApplyParams<float, float>& p, int nrhs, bool colloc, int epi,
                            cudaStream_t s);
// visco-acoustic / variable-density apply (apply_medium.cu; NEXT-2, readings A24, A25): bmed = b,
// kinv = κ⁻¹ = b/(v²(1 − i/(2Q))²), both [nzl+2][ny][ldx] with halo planes.  err == nullptr: no
// launch, returns the CTAs per RHS (partial slots); else launches and returns the same count.
template <typename R, typename S>
long long launch_apply_medium(const ApplyParams<R, S>& p, const S* bmed, const typename Cx<S>::T* kinv, int nrhs,
                              bool colloc, int epi, cudaStream_t s, cudaError_t* err);
template <typename S>
cudaError_t launch_medium_kinv(const S* v, const S* b, const S* q, typename Cx<S>::T* out, long long n, cudaStream_t s);
template <typename S> cudaError_t launch_medium_fill(S* out, long long n, S val, cudaStream_t s);
template <typename S>
cudaError_t launch_medium_check(const S* b, const S* q, long long n, int nx, int ldx, unsigned long long* bad,
                                cudaStream_t s);
// loopback communicator: the ranks' buffers (same device), reduced in rank order; op 0 = sum, 1 = max
constexpr int LOOP_MAX_RANKS = 16;
struct LoopPtrs {
  const double* p[LOOP_MAX_RANKS];
};
cudaError_t launch_loop_reduce(const LoopPtrs& ptrs, int np, double* out, long long n, int op, cudaStream_t s);
template <typename R> cudaError_t launch_winv(const R* v, R* w, long long n, cudaStream_t s);
template <typename R> cudaError_t launch_record(const ApplyParams<R>& p, R* rec, cudaStream_t s);
template <typename R> cudaError_t launch_gam_field(const ApplyParams<R>& p, R* out, int radius, cudaStream_t s);
template <typename R>
cudaError_t launch_eqerror(const typename Cx<R>::T* uref, const typename Cx<R>::T* u, int nx, int ny, int ldx, int nzl,
                           int z0, int nzg, const long long* src, double h, int npml, double ball, double* partials,
                           int nblocks, cudaStream_t s);
template <typename R>
cudaError_t launch_matrix(const ApplyParams<R>& p, bool colloc, long long* cols, typename Cx<R>::T* vals, cudaStream_t s);
cudaError_t launch_dispersion(const double* w7, const double* G, int nG, const double* theta, const double* phi, int nang,
                              double* out, cudaStream_t s);
template <typename R>
cudaError_t launch_sources(const ApplyParams<R>& p, int nsrc, const long long* nodes, const double* amps,
                           int consistent, R ih3, typename Cx<R>::T* b, cudaStream_t s);
template <typename R>
cudaError_t launch_vstats(const R* v, long long n, int nx, int ldx, R inv_fh, R g_min, R g_max, unsigned long long* out,
                          cudaStream_t s);
template <typename R> cudaError_t launch_bicg(int which, const VecParams<R>& q, int nrhs, cudaStream_t s);
template <typename R> cudaError_t launch_bicgl(int which, const VecParams<R>& q, int nrhs, cudaStream_t s);
template <typename R>
cudaError_t launch_norm2(const typename Cx<R>::T* f, long long fstride, long long plane, long long n, int nx, int ldx,
                         int nrhs, int nblocks, double* partials, double* out, unsigned int* tickets, cudaStream_t s);

// complex shifted-Laplacian multigrid preconditioner (mg.cu; hz_solve_opts.precond = 1)
struct MgSpec {
  int nx, ny, nz;                 // the slab (single rank)
  long long ldx, plane, fstride;  // field layout ([nrhs][nz+2][ny][ldx])
  const float* w;                 // 1/v² in the field layout (first field)
  double h, omega, beta, vmin, vmax, v_pml, r_coeff;
  int npml, nrhs, max_levels;
};
struct MgHierarchy;
cudaError_t mg_create(const MgSpec& spec, MgHierarchy** out);
void mg_destroy(MgHierarchy* m);
int mg_levels(const MgHierarchy* m);
cudaError_t mg_vcycle(MgHierarchy* m, const float2* f, float2* e, int nrhs, const int* active, cudaStream_t s,
                      long long* launches);

}  // namespace hz
