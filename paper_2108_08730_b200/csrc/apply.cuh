// Shared definitions of the fused coefficient build + matrix-free 27-point impedance apply
// (north-star steps a2–a6): launch parameters, epilogue kinds, the z-chunk ranges, the free-weight
// interpolation used outside the apply, the GAm row coefficients, the dot-product reductions.
//
//   (Au)_n = ω² Σ_d μ_{|d|}(w_n) u_{n+d} / v²_{n+d}                 Eq. 8, A2, A4
//          + Σ_a Σ_e D_a(n_a,e) Σ_{p,q} T(p,q; w_n) u_{n+e ê_a+p ê_b+q ê_c}   A6 (App. A), A8
//   w_n = linear interpolation of the Tikhonov table at G = v_n/(f h), clamped   P:36, A13
//
// The kernels: apply27_tm.cuh (complex64: tensor-map TMA tiles, RHS-fused, every tile class in one
// launch), apply27.cuh (register path: complex128 and the fp64 residual of the complex64 solver).
// DESIGN.md §5.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "cplx.cuh"

namespace hz {

enum { EPI_PLAIN = 0, EPI_DOT1 = 1, EPI_DOT4 = 2, EPI_RESID = 3 };
// doubles produced per RHS by each epilogue
//  DOT1:  (r̂0, v)                       → 2 (re, im)
//  DOT4:  (t, s), (t, t), (r̂0, s), (r̂0, t) → 7
//  RESID: ‖r‖², (r̂0, r)                  → 3
__host__ __device__ constexpr int epi_k(int epi) { return epi == 1 ? 2 : (epi == 2 ? 7 : (epi == 3 ? 3 : 0)); }

constexpr int TAB_STRIDE = 12;   // table row: t1 t2 mu0 mu1 mu2 | dt1 dt2 dmu0 dmu1 dmu2 | pad pad
constexpr int TMTAB_STRIDE = 16;   // apply27_tm table row: c0..c3 m0..m3 | their differences

// R: arithmetic type; S: storage type of the fields and the velocity (S = R except the
// mixed-precision residual of the complex64 solver, which reads c64 storage and computes in fp64).
template <typename R, typename S = R>
struct ApplyParams {
  typedef typename Cx<R>::T C;
  typedef typename Cx<S>::T CS;
  int nx, ny, nzl;            // local slab dims
  int ldx;                    // row pitch of every field / model array (elements): nx rounded up to 4
  int z0, nzg;                // global index of local plane 0, global nz
  long long plane;            // ny*ldx
  long long fstride;          // (nzl+2)*plane: per-RHS field stride (elements)
  // z-chunks of the local planes: [0, zlo) (if nlow = 1), nint chunks of ≤ zc planes covering
  // [zlo, zhi) (the planes whose outputs are outside the z-PML and the grid's first/last plane), then
  // [zhi, nzl) (if non-empty); nchunks = nlow + nint + nhigh.  See chunk_range().
  int zc, nchunks, zlo, zhi, nlow, nint;
  int nbx, nrhs;              // CTAs over all (strip, x-tile) warps of one z-chunk; RHS in the launch
  // interior "box" (no PML, no boundary) covered by the lean launch: strips [box_s0, box_s1),
  // x-tiles [box_t0, box_t1), z-chunks [box_c0, box_c1); box_nbx CTAs per chunk
  int box_s0, box_s1, box_t0, box_t1, box_c0, box_c1, box_nbx;
  // general launch work list per RHS: the boundary z-chunks (low, high) × all warps (nbx CTAs each),
  // then the interior z-chunks × the "frame" of warps outside the box (nbx_frame CTAs each)
  int nbound, nbx_frame, frame_warps, gen_blocks;
  // complex64 tensor-map launch (apply27_tm): tm_nitems work items (tm_item: tile × z-chunk, x/y-PML
  // tiles first), each run once per RHS, handed out by the counter tm_ctr[0] to a persistent grid of
  // tm_nblocks CTAs (tm_ctr[1]: finished CTAs; both zero between launches); tiles of tm_tx × tm_ty
  // points; tm_org = first storage plane covered by the tensor maps (planes outside the global grid
  // are zero-filled).  A launch runs the items [tm_item0, tm_item0 + tm_nitems) of the list (dot
  // partial slot = list index · nrhs + RHS); its last CTA reduces the partials of list items
  // [0, tm_nred) into dots (tm_nred = 0: no reduction — the interior half of a halo-overlapped apply)
  const int4* tm_work;
  unsigned int* tm_ctr;
  int tm_nitems, tm_nblocks, tm_tx, tm_ty, tm_org;
  int tm_item0, tm_nred;
  const S* v;                 // [nzl+2][ny][ldx] velocity incl. halo planes
  const S* w;                 // [nzl+2][ny][ldx] 1/v² incl. halo planes (apply input)
  const S* gam;               // GAm rule (A19): [5][nzl+2][ny][ldx] row weights (t1, t2, μ0, μ1, μ2)
                              // averaged over the 27 stencil nodes (stride fstride), or null (GA)
  const R* ctab;              // [n_g][CTAB_STRIDE] pre-scaled class coefficients + differences
  const float* ctm;           // [n_g][TMTAB_STRIDE] complex64 tensor-map apply: c0..c3, m0..m3 + differences
  int tab_lo, tab_n;          // rows [tab_lo, tab_lo + tab_n) cover every G of the model (staged in smem)
  const CS* u;                // [nrhs][nzl+2][ny][ldx]
  const CS* ulo;              // optional low part of u (mixed-precision residual of the c64 solver:
                              // u = u + ulo in fp64; only read when R != S), else null
  CS* au;                     // output
  const R* tab;               // [n_g][TAB_STRIDE]
  int n_g;                    // >= 2
  R g_min, g_max, inv_dg, inv_fh, ih2, w2;
  R invih2, inv2ih2, inv3ih2;  // h², h²/2, h²/3 (class coefficients → transverse weights)
  const C* dm[3];             // PML δ⁻ per axis (x, y, z[global])
  const C* dp[3];             // PML δ⁺
  int lo[3], hi[3];           // per-axis index range where δ± == 0 (inclusive)
  // epilogue inputs / outputs
  const CS* rhat;             // r̂0 (DOT1, DOT4, RESID) — may be null for RESID
  const CS* bvec;             // b (RESID)
  double* partials;           // [nrhs][gridDim.x*gridDim.y][K]
  double* dots;               // [nrhs][K]
  unsigned int* tickets;      // [nrhs]
  const int* active;          // [nrhs] or null
};

template <typename R, typename S>
__host__ __device__ __forceinline__ void chunk_range(const ApplyParams<R, S>& p, int k, int& a, int& b) {
  if (k < p.nlow) {
    a = 0;
    b = p.zlo;
  } else if (k < p.nlow + p.nint) {
    a = p.zlo + (k - p.nlow) * p.zc;
    b = a + p.zc < p.zhi ? a + p.zc : p.zhi;
  } else {
    a = p.zhi;
    b = p.nzl;
  }
}

// ---------------------------------------------------------------------------------------------
// Free weights of one row from its velocity: G = v/(f h) clamped, linear interpolation (A13).
// (The apply kernels interpolate the pre-scaled class-coefficient table instead; this form serves
// the record export, the consistent sources and the GAm field.)
// ---------------------------------------------------------------------------------------------
template <typename R>
__device__ __forceinline__ void interp_weights(R v, const R* __restrict__ tab, int n_g, R g_min, R g_max,
                                               R inv_dg, R inv_fh, R& t1, R& t2, R& mu0, R& mu1, R& mu2) {
  R G = v * inv_fh;                        // a2: G = v/(f h)
  G = fmin(fmax(G, g_min), g_max);         // clamp (A13)
  R s = (G - g_min) * inv_dg;
  int i = min((int)s, n_g - 2);            // s >= 0 → trunc == floor
  R tau = s - (R)i;
  const R* row = tab + i * TAB_STRIDE;     // a3: lookup + linear interpolation
  t1 = fma(tau, row[5], row[0]);
  t2 = fma(tau, row[6], row[1]);
  mu0 = fma(tau, row[7], row[2]);
  mu1 = fma(tau, row[8], row[3]);
  mu2 = fma(tau, row[9], row[4]);
}

// GAm row weights (t1, t2, μ0, μ1, μ2 at element idx of the [5][...] field) → the six register
// coefficients of a row, as the host builds the table rows: c1..c3 = h⁻²(t0 − 4t1, 2t1 − 2t2, 3t2),
// m1..m3 = ω²(μ1, μ2, μ3), t0 = 1 − 4t1 − 4t2, μ3 = (1 − μ0 − 6μ1 − 12μ2)/8 (A6).
template <typename R, typename S>
__device__ __forceinline__ void gam_row(const S* __restrict__ g, long long stride, long long idx, R ih2, R w2, R& c1,
                                        R& c2, R& c3, R& m1, R& m2, R& m3) {
  const R t1 = (R)__ldg(g + idx), t2 = (R)__ldg(g + stride + idx);
  const R mu0 = (R)__ldg(g + 2 * stride + idx), mu1 = (R)__ldg(g + 3 * stride + idx);
  const R mu2 = (R)__ldg(g + 4 * stride + idx);
  const R t0 = R(1) - R(4) * (t1 + t2);
  c1 = ih2 * (t0 - R(4) * t1);
  c2 = ih2 * (R(2) * (t1 - t2));
  c3 = ih2 * (R(3) * t2);
  m1 = w2 * mu1;
  m2 = w2 * mu2;
  m3 = w2 * ((R(1) - mu0 - R(6) * mu1 - R(12) * mu2) * R(0.125));
}

// field value at element idx of this RHS: storage → arithmetic type, plus the compensation term
// of the double-float iterate in the mixed-precision residual (R = double, S = float)
template <typename R, typename S>
__device__ __forceinline__ typename Cx<R>::T load_u(const typename Cx<S>::T* __restrict__ ub,
                                                    const typename Cx<S>::T* __restrict__ ulb, long long idx) {
  typename Cx<R>::T u = to_cx(ldg_c(ub + idx), R(0));
  if constexpr (sizeof(R) != sizeof(S)) {
    if (ulb != nullptr) u = cadd(u, to_cx(ldg_c(ulb + idx), R(0)));
  }
  return u;
}

// conj(a) * b accumulated in double
template <typename C>
__device__ __forceinline__ void acc_cdot(double& re, double& im, C a, C b) {
  re += (double)a.x * (double)b.x + (double)a.y * (double)b.y;
  im += (double)a.x * (double)b.y - (double)a.y * (double)b.x;
}

// Deterministic block reduction of K doubles, then grid reduction by the last block (ticket).
template <int K, int NT>
__device__ __forceinline__ void block_grid_reduce(double (&part)[K > 0 ? K : 1], double* partials, double* dots,
                                                  unsigned int* ticket, int nblocks, int bid) {
  if (K == 0) return;
  __shared__ double red[NT / 32][K > 0 ? K : 1];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; k++) {
    double s = part[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[warp][k] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 0; k < K; k++) {
      double s = 0;
      for (int w = 0; w < NT / 32; w++) s += red[w][k];
      partials[(long long)bid * K + k] = s;
    }
    __threadfence();
    unsigned int t = atomicAdd(ticket, 1u);
    last = (t == (unsigned)nblocks - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // fixed-order grid reduction: thread j sums blocks j, j+NT, ... ; then a fixed tree in smem
  __shared__ double gred[NT];
  for (int k = 0; k < K; k++) {
    double s = 0;
    for (int b = threadIdx.x; b < nblocks; b += NT) s += ((volatile double*)partials)[(long long)b * K + k];
    gred[threadIdx.x] = s;
    __syncthreads();
    for (int w = NT / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w) gred[threadIdx.x] += gred[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) dots[k] = gred[0];
    __syncthreads();
  }
  if (threadIdx.x == 0) *ticket = 0u;
}

}  // namespace hz
