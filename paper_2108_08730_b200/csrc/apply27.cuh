// K2 — fused coefficient build + matrix-free 27-point impedance apply (north-star steps a2–a6).
//
//   (Au)_n = Σ_d ω² μ_{|d|}(w_n) u_{n+d} / v²_{n+d}                        Eq. 8, A2, A4
//          + Σ_a Σ_{e∈{-1,0,1}} D_a(n_a, e) Σ_{p,q} T(p,q; w_n) u_{n+e ê_a+p ê_b+q ê_c}   A6 (App. A), A8
//   w_n = clamped linear interpolation of the Tikhonov weight table at G_n = v_n/(f h)  P:36, A13
//
// B200 design (HBM-bound: 4 + 16·nrhs bytes/point for complex64):
//  * Data: u (complex, [nrhs][nzl+2][ny][ldx]) and w = 1/v² (real, [nzl+2][ny][ldx], library-owned) are
//    the only per-point inputs; the row coefficients are recomputed from w in registers (G = 1/(√w f h)).
//    The coefficient table is pre-scaled on the host to the class coefficients
//    (c1..c3 = h⁻²(t0−4t1, 2t1−2t2, 3t2), m1..m3 = ω²μ1..3) with forward differences, 12 values per
//    G row, staged in shared memory for the model's G range: interpolation = 6 FMAs; c0 and m0 follow
//    from the sum rules.
//  * Mapping: a lane owns one x position and a strip of NY consecutive y rows; a warp covers 32
//    consecutive (strip, x) positions of the flattened strip-row space (no idle lanes for ragged nx:
//    where x wraps inside a warp the missing neighbours are Dirichlet zeros anyway).  x-neighbours come
//    from warp shuffles of (u, w) (lanes 0/31 load the warp-edge column), y-neighbours from the strip's
//    own registers (+1 halo row each side), z by marching planes with scatter-accumulation into the
//    partial outputs of planes k−1, k, k+1.  The next plane's loads are issued before the current
//    plane is consumed (register double-buffering) to keep ~2 planes of loads in flight.
//  * Interior (warp-uniform test): class-sum form, SURVEY App. A.5 — per input plane P0 = u, P1 = 4 faces,
//    P2 = 4 corners (and Q0..Q2 of q = u·w), then 18 real×complex FMAs (packed FFMA2 for complex64).
//  * PML (warp-uniform branch, no divergence within a warp's strip): per-axis form with the stretched
//    1-D operators D_a = (a⁻, −a⁻−a⁺, a⁺) (A8).  Per input plane and point
//      L1 = D_x u + D_y u,  L2 = D_x Y + D_y X   (X, Y = in-plane x-/y-neighbour sums)
//    and the contribution to output plane k from plane k+e is
//      e = 0:  t0 L1 + t1 L2 + D_z(k,0)(t0 P0 + t1 P1 + t2 P2)
//      e = ±1: t1 L1 + t2 L2 + D_z(k,e)(t0 P0 + t1 P1 + t2 P2)
//    which reduces exactly to the class form when every a± = h⁻².
//  * Mixed precision (R = double, S = float): the complex64 solver's residual b − A(x + x_lo) in fp64
//    arithmetic on c64 storage; w is then recomputed in fp64 from the float velocity.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "apply.cuh"

namespace hz {

template <typename R> struct Vec4;
template <> struct Vec4<float> { typedef float4 T; };
template <> struct Vec4<double> { typedef double4 T; };

// Table row: the six register coefficients of an output row and their forward differences,
//   c1 c2 c3 m1 | m2 m3 dc1 dc2 | dc3 dm1 dm2 dm3   (c = h⁻²·class stiffness, m = ω²·per-point mass)
// c0 and m0 follow from the sum rules (Coef6).  48 bytes (fp32) = 3 × 16-byte shared loads per point.
constexpr int CTAB_STRIDE = 12;
// shared-memory row pitch (elements): 12 floats = 48 B puts 8 consecutive rows on distinct banks
template <typename R> struct SmemPitch { enum { V = 12 }; };
template <> struct SmemPitch<double> { enum { V = 12 }; };

template <typename R>
__device__ __forceinline__ typename Vec4<R>::T lds4(const R* p);
template <>
__device__ __forceinline__ float4 lds4<float>(const float* p) { return *reinterpret_cast<const float4*>(p); }
template <>
__device__ __forceinline__ double4 lds4<double>(const double* p) {
  const double2 a = reinterpret_cast<const double2*>(p)[0];
  const double2 b = reinterpret_cast<const double2*>(p)[1];
  return make_double4(a.x, a.y, b.x, b.y);
}

__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ double4 ldg4(const double* p) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(p));
  const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

template <typename R>
struct Coef8 {
  R c0, c1, c2, c3, m0, m1, m2, m3;
};
// Register state of one output row: c1..c3, m1..m3.  The centre coefficients follow from the stencil's
// exact sum rules: c0 = −(6c1 + 12c2 + 8c3) (the stiffness annihilates constants, App. A) and
// m0 = ω² − 6m1 − 12m2 − 8m3 (Σ class mass weights = 1); for Eq. "10" m0 = ω²w0 − … likewise.
template <typename R>
struct Coef6 {
  R c1, c2, c3, m1, m2, m3;
};

// complex × complex (PML path); the rounding is spelled out (no compiler contraction choice) so that
// every unrolled copy of the kernel body computes bitwise the same value.  complex64: two packed FMAs
//   (acc.x, acc.y) += (a.x, a.x)·(b.x, b.y);  += (−a.y, a.y)·(b.y, b.x)
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float2 zfma(float2 a, float2 b, float2 acc) {
  acc = pk_fma(make_float2(a.x, a.x), b, acc);
  return pk_fma(make_float2(-a.y, a.y), make_float2(b.y, b.x), acc);
}
__device__ __forceinline__ float2 zmulc(float2 a, float2 b) { return zfma(a, b, make_float2(0.f, 0.f)); }
__device__ __forceinline__ double2 zfma(double2 a, double2 b, double2 acc) {
  acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
  return acc;
}
__device__ __forceinline__ double2 zmulc(double2 a, double2 b) {
  double2 r;
  r.x = fma(a.x, b.x, -mul_rn(a.y, b.y));
  r.y = fma(a.x, b.y, mul_rn(a.y, b.x));
  return r;
}

// Per-lane view of one input plane: rows 0..NY+1 = y0-1 .. y0+NY
template <typename R, int NY>
struct PlaneRegs {
  typedef typename Cx<R>::T C;
  C u[NY + 2];
  R w[NY + 2];
};

// Warp tiling: a warp covers 32 consecutive x positions x0-1 .. x0+30 of one strip of NY rows; lanes
// 1..30 produce outputs, lanes 0 and 31 are halo lanes that only load (so x-neighbours come from plain
// shuffles, and out-of-grid columns/rows load zeros: Dirichlet without masks).  XT = 30 outputs/warp.
constexpr int XT = 30;

// resident CTAs per SM (4 warps each) the register budget is sized for
template <typename R> struct ApplyBounds { enum { MINB = 3 }; };

// The apply is two launches of this template (same arithmetic per point, so results do not depend on
// which launch computes a point):
//   INTERIOR = true : the "box" — warps whose footprint is inside the grid and outside the x/y PML,
//                     for z-chunks whose output planes are outside the z PML: no PML code, no load
//                     predicates, 32-bit element offsets from per-CTA uniform base pointers.
//   INTERIOR = false: every other (warp, z-chunk); class form + per-axis PML corrections.
template <typename R, typename S, int NY, int W, bool COLLOC, int EPI, bool INTERIOR>
__global__ void __launch_bounds__(32 * W, ApplyBounds<R>::MINB) apply27_v2(ApplyParams<R, S> p) {
  typedef typename Cx<R>::T C;
  typedef typename Cx<S>::T CS;
  constexpr bool MIXED = !std::is_same<R, S>::value;
  constexpr int K = epi_k(EPI);
  const unsigned FULL = 0xffffffffu;

  // ---- block → (rhs, warp group, z-chunk); rhs fastest so the RHS of one tile share w through L2
  const int nrhs = p.nrhs;
  const int bid = blockIdx.x;
  const int rhs = bid % nrhs;
  const int tile = bid / nrhs;
  // chunk and first warp of this CTA
  int chunk, gw0;
  bool frame = false;                    // general launch, interior chunk: warps of the frame only
  if (INTERIOR) {
    chunk = p.box_c0 + tile / p.box_nbx;
    gw0 = (tile % p.box_nbx) * W;
  } else if (p.nbound == p.nchunks) {    // no box: plain (chunk, warp group) enumeration
    chunk = tile / p.nbx;
    gw0 = (tile % p.nbx) * W;
  } else if (tile < p.nbound * p.nbx) {  // boundary chunks: low (if any), then high
    const int b = tile / p.nbx;
    chunk = (b == 0 && p.nlow) ? 0 : p.nchunks - 1;
    gw0 = (tile % p.nbx) * W;
  } else {
    const int t = tile - p.nbound * p.nbx;
    chunk = p.nlow + t / p.nbx_frame;
    gw0 = (t % p.nbx_frame) * W;
    frame = true;
  }
  if (p.active != nullptr && p.active[rhs] == 0) return;   // converged RHS (uniform per CTA)

  // stage the used rows of the coefficient table in shared memory
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* stab = reinterpret_cast<R*>(smem_raw);
  constexpr int SP = SmemPitch<R>::V;
  for (int e = threadIdx.x; e < p.tab_n * CTAB_STRIDE; e += 32 * W) {
    const int r = e / CTAB_STRIDE, k = e - r * CTAB_STRIDE;
    stab[r * SP + k] = p.ctab[(long long)(p.tab_lo + r) * CTAB_STRIDE + k];
  }
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nx = p.nx, ny = p.ny, lx = p.ldx;
  const int ntx = (nx + XT - 1) / XT;
  const int nstrips = (ny + NY - 1) / NY;
  const int gw = gw0 + warp;
  int strip, xt;
  bool warp_ok;
  if (INTERIOR) {
    const int bw = p.box_t1 - p.box_t0;
    strip = p.box_s0 + gw / bw;
    xt = p.box_t0 + gw % bw;
    warp_ok = strip < p.box_s1;
  } else if (!frame) {
    strip = gw / ntx;
    xt = gw - strip * ntx;
    warp_ok = strip < nstrips;
  } else {
    // frame = strips above the box (all tiles), the box's strips outside [box_t0, box_t1), strips below
    const int bw = p.box_t1 - p.box_t0, side = ntx - bw;
    const int n_top = p.box_s0 * ntx, n_mid = (p.box_s1 - p.box_s0) * side;
    warp_ok = gw < p.frame_warps;
    if (gw < n_top) {
      strip = gw / ntx;
      xt = gw - strip * ntx;
    } else if (gw < n_top + n_mid) {
      const int k = gw - n_top;
      strip = p.box_s0 + k / side;
      const int jx = k - (strip - p.box_s0) * side;
      xt = jx < p.box_t0 ? jx : jx + bw;
    } else {
      const int k = gw - n_top - n_mid;
      strip = p.box_s1 + k / ntx;
      xt = k - (strip - p.box_s1) * ntx;
    }
  }
  const int x = xt * XT - 1 + lane;
  const int y0 = strip * NY;
  const bool xin = warp_ok && x >= 0 && x < nx;
  const bool is_out = xin && lane >= 1 && lane <= XT;     // this lane produces outputs

  unsigned rmask = 0;                           // bit r: row y0-1+r inside the grid (and lane in x)
#pragma unroll
  for (int r = 0; r < NY + 2; r++) {
    const int y = y0 - 1 + r;
    if (xin && y >= 0 && y < ny) rmask |= 1u << r;
  }
  bool gen_x = false, gen_y = false;   // warp-uniform: x-PML among the lanes / y-PML among the strip rows
  if (!INTERIOR) {
    const bool xp = is_out && (x < p.lo[0] || x > p.hi[0]);
    bool yp = false;
#pragma unroll
    for (int i = 0; i < NY; i++) {
      const int y = y0 + i;
      yp = yp || (is_out && y < ny && (y < p.lo[1] || y > p.hi[1]));
    }
    gen_x = __any_sync(FULL, xp);
    gen_y = __any_sync(FULL, yp);
  }
  const bool gen_col = gen_x || gen_y;

  int zc0, zc1;
  chunk_range(p, chunk, zc0, zc1);
  if (!warp_ok) zc1 = zc0 - 2;                                   // idle warps skip the march
  const int plane = (int)p.plane;                                // host checks fstride < 2^31
  // uniform per-CTA bases + 32-bit per-lane element offsets
  const CS* __restrict__ ubase = p.u + (long long)rhs * p.fstride;
  const CS* __restrict__ ulbase = (MIXED && p.ulo != nullptr) ? p.ulo + (long long)rhs * p.fstride : nullptr;
  const S* __restrict__ wbase = MIXED ? p.v : p.w;
  const int loff = (y0 - 1) * lx + x;          // (storage plane 0, row y0-1, column x); < 0 only if masked
  const C czv = czero(R(0));
  const int zlo = p.lo[2], zhi = p.hi[2];
  const int zbase = p.z0;
  // warp-uniform: the whole footprint inside the grid (no load predicates)
  const bool full_tile = INTERIOR || (warp_ok && (xt * XT - 1 >= 0) && (xt * XT + XT <= nx - 1) &&
                                      (y0 - 1 >= 0) && (y0 + NY <= ny - 1));

  // fetch plane pl (local index; storage index pl+1)
  auto fetch = [&](PlaneRegs<R, NY>& P, int pl) {
    const int off = loff + (pl + 1) * plane;
    if (!MIXED && (INTERIOR || (full_tile && zbase + pl >= 0 && zbase + pl < p.nzg))) {
#pragma unroll
      for (int r = 0; r < NY + 2; r++) {
        P.u[r] = to_cx(ldg_c(ubase + (unsigned)(off + r * lx)), R(0));
        P.w[r] = (R)__ldg(wbase + (unsigned)(off + r * lx));
      }
      return;
    }
    const int zg = zbase + pl;
    const unsigned m = (zg >= 0 && zg < p.nzg) ? rmask : 0u;
#pragma unroll
    for (int r = 0; r < NY + 2; r++) {
      const bool ok = (m >> r) & 1u;
      const unsigned o = (unsigned)(off + r * lx);
      if (!MIXED) {
        P.u[r] = ok ? to_cx(ldg_c(ubase + o), R(0)) : czv;
        P.w[r] = ok ? (R)__ldg(wbase + o) : R(0);
      } else {
        P.u[r] = ok ? load_u<R, S>(ubase, ulbase, o) : czv;
        const R vv = ok ? (R)__ldg(wbase + o) : R(1);
        P.w[r] = ok ? R(1) / (vv * vv) : R(0);
      }
    }
  };
  // own-row w of plane pl, for the coefficients (prefetched one plane earlier than the field)
  auto fetch_w = [&](R (&wc)[NY], int pl) {
    const int zg = zbase + pl;
    const bool pin = INTERIOR || (zg >= 0 && zg < p.nzg);
    const int off = loff + (pl + 1) * plane + lx;
#pragma unroll
    for (int i = 0; i < NY; i++) {
      const bool ok = INTERIOR || (pin && ((rmask >> (i + 1)) & 1u));
      const unsigned o = (unsigned)(off + i * lx);
      if (!MIXED) {
        wc[i] = ok ? (R)__ldg(wbase + o) : R(0);
      } else {
        const R vv = ok ? (R)__ldg(wbase + o) : R(1);
        wc[i] = ok ? R(1) / (vv * vv) : R(0);
      }
    }
  };

  double part[K > 0 ? K : 1];
#pragma unroll
  for (int k = 0; k < (K > 0 ? K : 1); k++) part[k] = 0.0;

  // PML x coefficients of this lane (gen_col warps): δ± = a± − h⁻²
  C dxm = czv, dxp = czv;
  if (!INTERIOR && gen_x && xin) {
    dxm = p.dm[0][x];
    dxp = p.dp[0][x];
  }
  const R i3h = p.inv3ih2, i2h = p.inv2ih2, i1h = p.invih2;
  const R s_k1 = p.inv_fh * p.inv_dg, s_k0 = -p.g_min * p.inv_dg, s_max = (R)(p.n_g - 1);

  // coefficients of output rows of plane pl+1 from w of that plane (a2 + a3)
  auto coefs = [&](Coef6<R> (&cn)[NY], R (&m0n)[NY], const R (&wc)[NY], bool valid, int pl) {
#pragma unroll
    for (int i = 0; i < NY; i++) {
      const R wn = wc[i];
      if (valid) {
        if (p.gam != nullptr) {   // GAm: the row's 27-node mean weights (A19)
          gam_row<R, S>(p.gam, p.fstride, (long long)(pl + 2) * plane + loff + (i + 1) * lx, p.ih2, p.w2, cn[i].c1,
                        cn[i].c2, cn[i].c3, cn[i].m1, cn[i].m2, cn[i].m3);
        } else {
        const R vv = rsqrt_r(wn);                           // w > 0 on valid rows
        R sidx = fma(vv, s_k1, s_k0);                      // (G − g_min)/ΔG, G = v/(f h)
        sidx = fmin(fmax(sidx, R(0)), s_max);              // clamp (A13)
        const int ii = min((int)sidx, p.n_g - 2);
        const R tau = sidx - (R)ii;
        const int li = min(max(ii - p.tab_lo, 0), p.tab_n - 2);   // staged range covers the model's G
        const R* row = stab + li * SP;
        typedef typename Vec4<R>::T V4;
        const V4 a = lds4<R>(row), b = lds4<R>(row + 4), d = lds4<R>(row + 8);
        cn[i].c1 = fma(tau, b.z, a.x);
        cn[i].c2 = fma(tau, b.w, a.y);
        cn[i].c3 = fma(tau, d.x, a.z);
        cn[i].m1 = fma(tau, d.y, a.w);
        cn[i].m2 = fma(tau, d.z, b.x);
        cn[i].m3 = fma(tau, d.w, b.y);
        }
        if (COLLOC) {   // Eq. "10": ω²/κ0 for all 27 neighbours → m·w0 multiplies the u class sums
          cn[i].m1 *= wn;
          cn[i].m2 *= wn;
          cn[i].m3 *= wn;
        }
        m0n[i] = COLLOC ? wn : R(1);
      } else {
        cn[i] = Coef6<R>{R(0), R(0), R(0), R(0), R(0), R(0)};
        m0n[i] = R(0);
      }
    }
  };
  const R w2 = p.w2;
  // centre coefficients from the sum rules (m0 needs the ω² scale: ω²·(1 or w0) in m0s)
  auto c0_of = [](const Coef6<R>& c) { return -fma(R(6), c.c1, fma(R(12), c.c2, R(8) * c.c3)); };
  auto m0_of = [&](const Coef6<R>& c, R m0s) { return fma(w2, m0s, -fma(R(6), c.m1, fma(R(12), c.m2, R(8) * c.m3))); };

  // One input plane pl.  cP: coefficients of output pl-1 (overwritten with those of pl+1);
  // cC: of output pl.  aP: partial of output pl-1 (overwritten with the first partial of pl+1);
  // aC: partial of output pl.  Roles alternate between two slots → no register rotation.
  auto body = [&](PlaneRegs<R, NY>& Pc, PlaneRegs<R, NY>& Pn, Coef6<R> (&cP)[NY], Coef6<R> (&cC)[NY],
                  R (&mP)[NY], R (&mC)[NY], C (&aP)[NY], C (&aC)[NY], R (&wcN)[NY], R (&wcF)[NY], int pl) {
    // wcN: own-row w of plane pl+1 (fetched one iteration ago); wcF receives plane pl+2
    if (pl + 1 <= zc1) fetch(Pn, pl + 1);   // prefetch: in flight while plane pl is consumed
    if (pl + 2 < zc1) fetch_w(wcF, pl + 2);
    // epilogue operands of the outputs finalised in this call (plane pl-1), loaded now so their latency
    // overlaps the plane's arithmetic: r̂0 (DOT1/DOT4/RESID) and s = u (DOT4) or b (RESID)
    C e1[NY], e2[NY];
    const bool fin = (pl - 1 >= zc0) && is_out;
#pragma unroll
    for (int i = 0; i < NY; i++) {
      e1[i] = czv;
      e2[i] = czv;
      if (K > 0 && fin && (INTERIOR || ((rmask >> (i + 1)) & 1u))) {
        const long long o = (long long)rhs * p.fstride + (unsigned)(loff + pl * plane + (i + 1) * lx);
        if (EPI != EPI_RESID || p.rhat != nullptr) e1[i] = to_cx(ldg_c(p.rhat + o), R(0));
        if (EPI == EPI_DOT4) e2[i] = to_cx(ldg_c(p.u + o), R(0));
        if (EPI == EPI_RESID) e2[i] = to_cx(ldg_c(p.bvec + o), R(0));
      }
    }
    const bool do_prev = (pl - 1 >= zc0);
    const bool do_next = (pl + 1 < zc1);
    const int zg = zbase + pl;
    bool zp_prev = false, zp_cur = false, zp_next = false, zcorr = false;
    if (!INTERIOR) {
      zp_prev = do_prev && (zg - 1 < zlo || zg - 1 > zhi);
      zp_cur = (pl >= zc0 && pl < zc1) && (zg < zlo || zg > zhi);
      zp_next = do_next && (zg + 1 < zlo || zg + 1 > zhi);
      zcorr = zp_prev || zp_cur || zp_next;
    }

    // ---- in-plane x sums: X = u(x-1) + u(x+1), Xq = q(x-1) + q(x+1), q = u·w
    C X[NY + 2], q[NY + 2], Xq[NY + 2];
#pragma unroll
    for (int r = 0; r < NY + 2; r++) {
      const C a = shfl_up_c(Pc.u[r], 1);
      const C b = shfl_down_c(Pc.u[r], 1);
      X[r] = cadd(a, b);
      if (!COLLOC) {
        const R wa = __shfl_up_sync(FULL, Pc.w[r], 1);
        const R wbv = __shfl_down_sync(FULL, Pc.w[r], 1);
        q[r] = cscale(Pc.w[r], Pc.u[r]);
        Xq[r] = cfma(wbv, b, cscale(wa, a));
      }
    }
    Coef6<R> cN[NY];
    R mN[NY];
    coefs(cN, mN, wcN, do_next, pl);

#pragma unroll
    for (int i = 0; i < NY; i++) {
      const C u0 = Pc.u[i + 1];
      const C Y = cadd(Pc.u[i], Pc.u[i + 2]);
      const C P1 = cadd(X[i + 1], Y);
      const C P2 = cadd(X[i], X[i + 2]);
      const C Q0 = COLLOC ? u0 : q[i + 1];
      const C Q1 = COLLOC ? P1 : cadd(Xq[i + 1], cadd(q[i], q[i + 2]));
      const C Q2 = COLLOC ? P2 : cadd(Xq[i], Xq[i + 2]);
      // ---- interior class-sum form
      C a = aP[i];
      a = cfma(cP[i].c1, u0, a);
      a = cfma(cP[i].c2, P1, a);
      a = cfma(cP[i].c3, P2, a);
      a = cfma(cP[i].m1, Q0, a);
      a = cfma(cP[i].m2, Q1, a);
      a = cfma(cP[i].m3, Q2, a);
      C b = aC[i];
      b = cfma(c0_of(cC[i]), u0, b);
      b = cfma(cC[i].c1, P1, b);
      b = cfma(cC[i].c2, P2, b);
      b = cfma(m0_of(cC[i], mC[i]), Q0, b);
      b = cfma(cC[i].m1, Q1, b);
      b = cfma(cC[i].m2, Q2, b);
      C c = cscale(cN[i].c1, u0);
      c = cfma(cN[i].c2, P1, c);
      c = cfma(cN[i].c3, P2, c);
      c = cfma(cN[i].m1, Q0, c);
      c = cfma(cN[i].m2, Q1, c);
      c = cfma(cN[i].m3, Q2, c);
      // ---- PML corrections (A8): a± = h⁻² + δ±; warp/plane-uniform branches
      if (!INTERIOR && (gen_col || zcorr)) {
        // transverse weights from the class coefficients: t2 = c3 h²/3, t1 = t2 + c2 h²/2, t0 = c1 h² + 4 t1
        const R pt2 = cP[i].c3 * i3h, pt1 = fma(cP[i].c2, i2h, pt2), pt0 = fma(cP[i].c1, i1h, R(4) * pt1);
        const R ct2 = cC[i].c3 * i3h, ct1 = fma(cC[i].c2, i2h, ct2), ct0 = fma(cC[i].c1, i1h, R(4) * ct1);
        const R nt2 = cN[i].c3 * i3h, nt1 = fma(cN[i].c2, i2h, nt2), nt0 = fma(cN[i].c1, i1h, R(4) * nt1);
        if (gen_col) {
          // ΔL1 = δx(u) + δy(u), ΔL2 = δx(Y) + δy(X): the stretched parts of D_x, D_y; the x part only
          // in warps with x-PML lanes, the y part only for strips with y-PML rows
          C L1 = czv, L2 = czv;
          if (gen_x) {
            const C uL = shfl_up_c(u0, 1), uR = shfl_down_c(u0, 1);
            const C YL = shfl_up_c(Y, 1), YR = shfl_down_c(Y, 1);
            L1 = zmulc(dxm, csub(uL, u0));
            L1 = zfma(dxp, csub(uR, u0), L1);
            L2 = zmulc(dxm, csub(YL, Y));
            L2 = zfma(dxp, csub(YR, Y), L2);
          }
          if (gen_y) {
            C dym = czv, dyp = czv;
            if ((rmask >> (i + 1)) & 1u) {
              dym = p.dm[1][y0 + i];
              dyp = p.dp[1][y0 + i];
            }
            L1 = zfma(dym, csub(Pc.u[i], u0), L1);
            L1 = zfma(dyp, csub(Pc.u[i + 2], u0), L1);
            L2 = zfma(dym, csub(X[i], X[i + 1]), L2);
            L2 = zfma(dyp, csub(X[i + 2], X[i + 1]), L2);
          }
          a = cfma(pt1, L1, a);
          a = cfma(pt2, L2, a);
          b = cfma(ct0, L1, b);
          b = cfma(ct1, L2, b);
          c = cfma(nt1, L1, c);
          c = cfma(nt2, L2, c);
        }
        if (zcorr) {   // δz · (t0 P0 + t1 P1 + t2 P2) of each output plane
          if (zp_prev) {
            C B3 = cscale(pt0, u0);
            B3 = cfma(pt1, P1, B3);
            B3 = cfma(pt2, P2, B3);
            a = zfma(p.dp[2][zg - 1], B3, a);
          }
          if (zp_cur) {
            C B3 = cscale(ct0, u0);
            B3 = cfma(ct1, P1, B3);
            B3 = cfma(ct2, P2, B3);
            const C dz = cadd(p.dm[2][zg], p.dp[2][zg]);
            b = zfma(make_cx(-dz.x, -dz.y), B3, b);
          }
          if (zp_next) {
            C B3 = cscale(nt0, u0);
            B3 = cfma(nt1, P1, B3);
            B3 = cfma(nt2, P2, B3);
            c = zfma(p.dm[2][zg + 1], B3, c);
          }
        }
      }
      aC[i] = b;          // output pl: "prev" of the next plane (slot roles swap)
      aP[i] = c;          // output pl+1: "cur" of the next plane
      cP[i] = cN[i];      // coefficients of pl+1 take the slot of pl-1
      mP[i] = mN[i];
      // ---- finalize output (row i, plane pl-1), epilogue
      if (do_prev && is_out && (INTERIOR || ((rmask >> (i + 1)) & 1u))) {
        const long long o = (long long)rhs * p.fstride + (unsigned)(loff + pl * plane + (i + 1) * lx);
        if (EPI == EPI_RESID) {
          const C rr = csub(e2[i], a);
          p.au[o] = from_cx(rr, S(0));
          part[0] += (double)rr.x * (double)rr.x + (double)rr.y * (double)rr.y;
          if (p.rhat != nullptr) acc_cdot(part[1], part[2], e1[i], rr);
        } else {
          p.au[o] = from_cx(a, S(0));
          if (EPI == EPI_DOT1) {
            acc_cdot(part[0], part[1], e1[i], a);
          } else if (EPI == EPI_DOT4) {
            const C sv = e2[i];
            const C rh = e1[i];
            acc_cdot(part[0], part[1], a, sv);
            part[2] += (double)a.x * (double)a.x + (double)a.y * (double)a.y;
            acc_cdot(part[3], part[4], rh, sv);
            acc_cdot(part[5], part[6], rh, a);
          }
        }
      }
    }
  };

  PlaneRegs<R, NY> A, B;
  Coef6<R> c0s[NY], c1s[NY];
  R m0a[NY], m0b[NY];
  C a0s[NY], a1s[NY];
#pragma unroll
  for (int i = 0; i < NY; i++) {
    c0s[i] = Coef6<R>{R(0), R(0), R(0), R(0), R(0), R(0)};
    c1s[i] = c0s[i];
    m0a[i] = m0b[i] = R(0);
    a0s[i] = czv;
    a1s[i] = czv;
  }
  R w0s[NY], w1s[NY];
  if (zc1 >= zc0) {
    fetch(A, zc0 - 1);
    if (zc0 < zc1) fetch_w(w0s, zc0);
  }
  int pl = zc0 - 1;
  for (; pl + 1 <= zc1; pl += 2) {
    body(A, B, c0s, c1s, m0a, m0b, a0s, a1s, w0s, w1s, pl);
    body(B, A, c1s, c0s, m0b, m0a, a1s, a0s, w1s, w0s, pl + 1);
  }
  if (pl <= zc1) body(A, B, c0s, c1s, m0a, m0b, a0s, a1s, w0s, w1s, pl);

  if (K > 0) {
    // both launches share the partials / ticket: the general one owns blocks [0, nb_gen), the
    // interior one [nb_gen, nb_gen + nb_int); the last block overall reduces in a fixed order
    const int nb_gen = p.gen_blocks;
    const int nblocks = nb_gen + p.box_nbx * (p.box_c1 - p.box_c0);
    const int slot = INTERIOR ? nb_gen + tile : tile;
    block_grid_reduce<K, 32 * W>(part, p.partials + (long long)rhs * nblocks * K, p.dots + (long long)rhs * K,
                                 p.tickets + rhs, nblocks, slot);
  }
}

}  // namespace hz
