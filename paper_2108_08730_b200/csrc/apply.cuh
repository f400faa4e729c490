// Fused coefficient build + matrix-free 27-point impedance apply (north-star steps a2–a6).
//
//   (Au)_n = ω² Σ_d μ_{|d|}(w_n) u_{n+d} / v²_{n+d}                 Eq. 8, A2, A4
//          + Σ_a Σ_e D_a(n_a,e) Σ_{p,q} T(p,q; w_n) u_{n+e ê_a+p ê_b+q ê_c}   A6 (App. A), A8
//   w_n = linear interpolation of the Tikhonov table at G = v_n/(f h), clamped   P:36, A13
//
// Design (B200): HBM-bound stencil (20 B/point for complex64, nrhs = 1: read u, read v, write Au).
//  * The coefficients are recomputed from v in registers (no coefficient record in HBM: "fused
//    mode").  The table (≤ 1024 rows × 12 values) lives in shared memory; per row it stores
//    (t1, t2, μ0, μ1, μ2) and their forward differences, so the interpolation is 5 FMAs and the
//    class coefficients follow from t0 = 1 − 4t1 − 4t2 and μ3 = (1 − μ0 − 6μ1 − 12μ2)/8.
//  * Interior rows use the class-sum form: per plane and point the in-plane sums
//    P0 = u, P1 = 4 faces, P2 = 4 corners (and the same Q for q = u/v²); the 27-point row is then
//      c0 U0 + c1 U1 + c2 U2 + c3 U3 + m0 Q0 + … with U1 = P1(k) + P0(k±1), U2 = P2(k) + P1(k±1),
//      U3 = P2(k±1), c = h⁻²(−6t0, t0−4t1, 2t1−2t2, 3t2), m = ω²μ.
//  * Thread mapping: a lane owns one x position and a strip of NY consecutive y rows, and the
//    warp marches a chunk of z planes.  Lanes of a warp cover 32 consecutive (strip, x) positions
//    of the flattened strip-row space (no padding waste for nx not a multiple of 32); x-neighbours
//    come from warp shuffles (lanes 0/31 load the warp-edge halo), y-neighbours from the thread's
//    own strip (+1 halo row each side), z-neighbours by scatter-accumulation into the partial
//    outputs of planes k−1, k, k+1 (two complex accumulators + two planes of coefficients
//    persist per point).  No shared memory is used for the field.
//  * complex64 arithmetic runs on the packed FP32x2 pipe (FFMA2/FADD2).
//  * PML rows (a few % of the grid) add the stretched per-axis correction
//      Σ_a δ⁻_a (T_a u(n−ê_a) − T_a u(n)) + δ⁺_a (T_a u(n+ê_a) − T_a u(n)),  δ± = a± − h⁻²
//    in a divergent slow path that re-reads the 27-neighbourhood from L1/L2.
//  * Optional epilogues fuse the BiCGSTAB dot products (fp64 accumulation, deterministic
//    block-then-grid reduction with a last-block ticket).
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

// R: arithmetic type; S: storage type of the fields and the velocity (S = R except the
// mixed-precision residual of the complex64 solver, which reads c64 storage and computes in fp64).
template <typename R, typename S = R>
struct ApplyParams {
  typedef typename Cx<R>::T C;
  typedef typename Cx<S>::T CS;
  int nx, ny, nzl;            // local slab dims
  int z0, nzg;                // global index of local plane 0, global nz
  long long plane;            // nx*ny
  long long fstride;          // (nzl+2)*plane: per-RHS field stride (elements)
  long long nlanes;           // nstrips*nx (set by the launcher)
  // z-chunks of the local planes: [0, zlo) (if nlow = 1), nint chunks of ≤ zc planes covering
  // [zlo, zhi) (the planes whose outputs are outside the z-PML and the grid's first/last plane), then
  // [zhi, nzl) (if non-empty); nchunks = nlow + nint + nhigh.  See chunk_range().
  int zc, nchunks, zlo, zhi, nlow, nint;
  int nbx, nrhs;              // CTAs over all (strip, x-tile) warps of one z-chunk; RHS in the launch
  // interior "box" (no PML, no boundary) covered by the lean launch: strips [box_s0, box_s1),
  // x-tiles [box_t0, box_t1), z-chunks [box_c0, box_c1); box_nbx CTAs per chunk
  int box_s0, box_s1, box_t0, box_t1, box_c0, box_c1, box_nbx;
  // complex64 interior launch (apply27_tma): the box as points [tma_x0, tma_x1) × [tma_y0, tma_y1),
  // tiled by tma_ntx × tma_nty CTA tiles (then box_nbx = tma_ntx · tma_nty)
  int tma_x0, tma_x1, tma_y0, tma_y1, tma_ntx, tma_nty;
  // general launch work list per RHS: the boundary z-chunks (low, high) × all warps (nbx CTAs each),
  // then the interior z-chunks × the "frame" of warps outside the box (nbx_frame CTAs each)
  int nbound, nbx_frame, frame_warps, gen_blocks;
  // complex64 RHS-fused launch (apply27_cp): work items (cp_item) — first cp_n_pml x/y-PML tiles,
  // then cp_n_int tiles outside the x/y-PML; cp_nblocks = dot partial slots per RHS
  const int4* cp_work;
  int cp_n_pml, cp_n_int, cp_nblocks;
  const S* v;                 // [nzl+2][ny][nx] velocity incl. halo planes
  const S* w;                 // [nzl+2][ny][nx] 1/v² incl. halo planes (apply input)
  const S* gam;               // GAm rule (A19): [5][nzl+2][ny][nx] row weights (t1, t2, μ0, μ1, μ2)
                              // averaged over the 27 stencil nodes (stride fstride), or null (GA)
  const R* ctab;              // [n_g][CTAB_STRIDE] pre-scaled class coefficients + differences
  int tab_lo, tab_n;          // rows [tab_lo, tab_lo + tab_n) cover every G of the model (staged in smem)
  const CS* u;                // [nrhs][nzl+2][ny][nx]
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
// Coefficients of one row from its velocity: interpolated (t1, t2, μ0, μ1, μ2) → c0..c3, m0..m3.
// ---------------------------------------------------------------------------------------------
template <typename R>
struct RowCoef {
  R c0, c1, c2, c3, m0, m1, m2, m3;
};

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

template <typename R, typename S>
__device__ __forceinline__ RowCoef<R> row_coef(R v, const R* __restrict__ tab, const ApplyParams<R, S>& p) {
  R t1, t2, mu0, mu1, mu2;
  interp_weights<R>(v, tab, p.n_g, p.g_min, p.g_max, p.inv_dg, p.inv_fh, t1, t2, mu0, mu1, mu2);
  RowCoef<R> c;
  // t0 = ws1 + 2/3 ws2 + 1/2 ws3 = 1 − 4 t1 − 4 t2 (A6);  class coefficients × h⁻²
  const R t12 = t1 + t2;
  c.c0 = p.ih2 * fma((R)24, t12, (R)-6);                 // −6 t0
  c.c1 = p.ih2 * fma((R)-8, t1, fma((R)-4, t2, (R)1));   // t0 − 4 t1
  c.c2 = p.ih2 * ((R)2 * (t1 - t2));                     // 2 t1 − 2 t2
  c.c3 = p.ih2 * ((R)3 * t2);                            // 3 t2
  const R mu3 = ((R)1 - mu0 - (R)6 * mu1 - (R)12 * mu2) * (R)0.125;   // wm3/8
  c.m0 = p.w2 * mu0;
  c.m1 = p.w2 * mu1;
  c.m2 = p.w2 * mu2;
  c.m3 = p.w2 * mu3;
  return c;
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

// ---------------------------------------------------------------------------------------------
// PML correction for one row (slow path).  zl: local plane index of the output.
// ---------------------------------------------------------------------------------------------
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

template <typename R, typename S>
__device__ __noinline__ typename Cx<R>::T pml_correction(const ApplyParams<R, S>& p, const R* __restrict__ tab,
                                                         const typename Cx<S>::T* __restrict__ ub,
                                                         const typename Cx<S>::T* __restrict__ ulb,
                                                         int x, int y, int zl) {
  typedef typename Cx<R>::T C;
  const int zg = p.z0 + zl;
  C n[3][3][3];
#pragma unroll
  for (int dz = 0; dz < 3; dz++)
#pragma unroll
    for (int dy = 0; dy < 3; dy++)
#pragma unroll
      for (int dx = 0; dx < 3; dx++) {
        int xx = x + dx - 1, yy = y + dy - 1, zz = zg + dz - 1;
        bool in = xx >= 0 && xx < p.nx && yy >= 0 && yy < p.ny && zz >= 0 && zz < p.nzg;
        n[dz][dy][dx] = in ? load_u<R, S>(ub, ulb, (long long)(zl + dz) * p.plane + (long long)yy * p.nx + xx) : czero(R(0));
      }
  R t1, t2, mu0, mu1, mu2;
  const R vv = (R)p.v[(long long)(zl + 1) * p.plane + (long long)y * p.nx + x];
  interp_weights<R>(vv, tab, p.n_g, p.g_min, p.g_max, p.inv_dg, p.inv_fh, t1, t2, mu0, mu1, mu2);
  const R t0 = (R)1 - (R)4 * (t1 + t2);
  C corr = czero(R(0));
  const int idx[3] = {x, y, zg};
#pragma unroll
  for (int a = 0; a < 3; a++) {
    if (idx[a] >= p.lo[a] && idx[a] <= p.hi[a]) continue;
    C T[3];
#pragma unroll
    for (int e = 0; e < 3; e++) {
      C c, f, k;
      if (a == 0) {        // transverse plane (y, z) at x + e − 1
        c = n[1][1][e];
        f = cadd(cadd(n[1][0][e], n[1][2][e]), cadd(n[0][1][e], n[2][1][e]));
        k = cadd(cadd(n[0][0][e], n[0][2][e]), cadd(n[2][0][e], n[2][2][e]));
      } else if (a == 1) { // transverse plane (x, z) at y + e − 1
        c = n[1][e][1];
        f = cadd(cadd(n[1][e][0], n[1][e][2]), cadd(n[0][e][1], n[2][e][1]));
        k = cadd(cadd(n[0][e][0], n[0][e][2]), cadd(n[2][e][0], n[2][e][2]));
      } else {             // transverse plane (x, y) at z + e − 1
        c = n[e][1][1];
        f = cadd(cadd(n[e][1][0], n[e][1][2]), cadd(n[e][0][1], n[e][2][1]));
        k = cadd(cadd(n[e][0][0], n[e][0][2]), cadd(n[e][2][0], n[e][2][2]));
      }
      T[e] = cfma(t0, c, cfma(t1, f, cscale(t2, k)));
    }
    const C dmv = p.dm[a][idx[a]], dpv = p.dp[a][idx[a]];
    corr = cadd(corr, cadd(cmul(dmv, csub(T[0], T[1])), cmul(dpv, csub(T[2], T[1]))));
  }
  return corr;
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
