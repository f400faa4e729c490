// K2 for complex64, every point of the slab: RHS-fused, cp.async-staged plane tiles sliding in z.
//
// Same operator and per-point operation order as apply27_v2 / apply27_tma (class-sum form, SURVEY
// App. A.5; PML per-axis corrections, reading A8), organised for the BiCGSTAB regime — several RHS,
// grids of ~10⁶ points, 40% of them in the PML — where the register-path launches were latency bound
// (12 warps/SM, one plane of loads in flight) and recomputed the coefficients once per RHS:
//  * One CTA (8 warps) owns a tile of tx × (2·ns) output columns/rows (tx ≤ 64, chosen per grid so
//    that tx·ns ≈ 256 threads: no idle lanes for ragged nx such as 101) for NR right-hand sides and
//    marches a z-chunk.  Thread t owns column t % tx and the 2 rows of strip t / tx.
//  * Each plane's w tile and the NR u tiles (+1 halo row/column) are copied global → shared by
//    cp.async (4/8-byte, zero-filled outside the grid: the Dirichlet boundary costs no branch) into a
//    ring of HZ_CP_STAGES planes; two planes are in flight while one is consumed.
//  * Per plane and point the coefficients (table interpolation, PML transverse weights) are computed
//    once and used for all NR fields; per field the 9 in-plane neighbours come from shared memory.
//  * Two instantiations: PML = true for tiles with any output point in the PML (warp-uniform x / y /
//    plane-uniform z corrections, exactly the register path's), PML = false for the rest.  A
//    correction with δ = 0 adds exact zeros, so both compute bitwise the same value for a point.
//  * Dot epilogues accumulate per thread in fp32 (HZ_CP_DOT_F64 = 1: fp64 as the register path) and
//    reduce per block and grid in fp64 in a fixed order.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "apply27.cuh"

namespace hz {

// Tile geometry is shared by all variants: tx ≤ 64 columns × TY = 2·ns rows with tx·ns ≤ 256.  A
// variant with NY rows per thread runs CP_THREADS(NY) = 512/NY threads; the halo tile
// (TY + 2)·(tx + 2) ≤ 768 elements is copied with CP_SLOTS(NY) elements per thread.
constexpr int CP_NT = 256;        // positions (column, 2-row strip) per tile
constexpr int CP_PMAX = 66;       // shared row pitch (elements): tx ≤ 64 + 2 halo columns
constexpr int CP_NSMAX = 16;      // strips per tile (TY ≤ 32)
constexpr int CP_KS = 3;          // (2·ns + 2)·(tx + 2) ≤ CP_KS·CP_NT
__host__ __device__ constexpr int CP_THREADS(int ny) { return 512 / ny; }
__host__ __device__ constexpr int CP_SLOTS(int ny) { return (CP_KS * CP_NT + CP_THREADS(ny) - 1) / CP_THREADS(ny); }
// PML mode of a work item: 0 none, 1 z-PML output planes only, 2 x/y-PML columns/rows (+ z)
enum { CP_LEAN = 0, CP_PMLZ = 1, CP_PMLXY = 2 };
#ifndef HZ_CP_STAGES
#define HZ_CP_STAGES 4
#endif
constexpr int CP_STAGES = HZ_CP_STAGES;
#ifndef HZ_CP_GX   // experiment switches (register-pressure study); 1 = on
#define HZ_CP_GX 1
#endif
#ifndef HZ_CP_GY
#define HZ_CP_GY 1
#endif
#ifndef HZ_CP_GZ
#define HZ_CP_GZ 1
#endif
#ifndef HZ_CP_DOT_F64
#define HZ_CP_DOT_F64 0
#endif

// bytes of one ring stage: w rows then NR u tiles, ROWS = 2·ns + 2 rows of CP_PMAX elements
__host__ __device__ constexpr size_t cp_stage_bytes(int ns, int nr) {
  return (size_t)(2 * ns + 2) * CP_PMAX * (4 + 8 * nr);
}
__host__ __device__ constexpr size_t cp_smem_bytes(int tab_n, int ns, int nr) {
  return (((size_t)tab_n * 12 * 4 + 127) / 128) * 128 + (size_t)CP_STAGES * cp_stage_bytes(ns, nr);
}

__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, uint32_t n) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src, uint32_t n) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// conj(a)·b accumulated per thread (fp32 or fp64)
#if HZ_CP_DOT_F64
typedef double DotT;
__device__ __forceinline__ void cp_cdot(DotT& re, DotT& im, float2 a, float2 b) { acc_cdot(re, im, a, b); }
__device__ __forceinline__ void cp_norm(DotT& s, float2 a) { s += (double)a.x * (double)a.x + (double)a.y * (double)a.y; }
#else
typedef float DotT;
__device__ __forceinline__ void cp_cdot(DotT& re, DotT& im, float2 a, float2 b) {
  re = fmaf(a.x, b.x, fmaf(a.y, b.y, re));
  im = fmaf(a.x, b.y, fmaf(-a.y, b.x, im));
}
__device__ __forceinline__ void cp_norm(DotT& s, float2 a) { s = fmaf(a.x, a.x, fmaf(a.y, a.y, s)); }
#endif

// complex multiply-add with a per-thread constant d (PML δ): acc + d·b as two packed FMAs,
// dn = (−d.y, d.y) precomputed once so the only per-use operand shuffle is the swap of b
__device__ __forceinline__ float2 zfma_c(float2 d, float2 dn, float2 b, float2 acc) {
  acc = pk_fma(make_float2(d.x, d.x), b, acc);
  return pk_fma(dn, make_float2(b.y, b.x), acc);
}
__device__ __forceinline__ float2 zneg_sw(float2 d) { return make_float2(-d.y, d.y); }

// Work item: tile index (ty·ntx + tx), output planes [z0, z1) of the slab (local indices)
template <int NY, int NR, bool COLLOC, int EPI, int PM>
__global__ void __launch_bounds__(CP_THREADS(NY), 512 / CP_THREADS(NY)) apply27_cp(ApplyParams<float, float> p, int item0) {
  typedef float R;
  typedef float2 C;
  constexpr bool PML = PM != CP_LEAN;
  constexpr bool PXY = PM == CP_PMLXY;
  constexpr int NT = CP_THREADS(NY);
  constexpr int KS = CP_SLOTS(NY);
  constexpr int K = epi_k(EPI);
  constexpr int S = CP_STAGES;
  const unsigned FULL = 0xffffffffu;

  // ---- block → (work item, RHS group)
  const int4 item = p.cp_work[item0 + blockIdx.x];
  const int rhs0 = blockIdx.y * NR;
  bool act[NR];
  bool any = false;
#pragma unroll
  for (int r = 0; r < NR; r++) {
    act[r] = rhs0 + r < p.nrhs && (p.active == nullptr || p.active[rhs0 + r] != 0);
    any = any || act[r];
  }
  if (!any) return;   // uniform per CTA

  const int nx = p.nx, ny = p.ny;
  const int tx = p.cp_tx, ns = p.cp_ns, TY = 2 * ns, ROWS = TY + 2;
  const int ttx = item.x % p.cp_ntx, tty = item.x / p.cp_ntx;
  const int X0n = ttx * tx, Y0n = tty * TY;
  const int X0 = min(X0n, nx - tx), Y0 = min(Y0n, ny - TY);   // clamped tiles (overlap, not stored twice)
  const int zc0 = item.y, zc1 = item.z;
  const int nplanes = zc1 - zc0 + 2;   // input planes zc0-1 .. zc1
  const int plane = (int)p.plane;      // host: (nzl + 2)·plane < 2^31 (32-bit offsets within a field)

  extern __shared__ __align__(1024) unsigned char smem_cp[];
  float* stab = reinterpret_cast<float*>(smem_cp);
  unsigned char* ring = smem_cp + (((size_t)p.tab_n * 12 * 4 + 127) / 128) * 128;
  const uint32_t stage_bytes = (uint32_t)cp_stage_bytes(ns, NR);
  const uint32_t wbytes = (uint32_t)ROWS * CP_PMAX * 4;   // w rows of a stage; the u tiles follow
  const uint32_t ubytes = (uint32_t)ROWS * CP_PMAX * 8;
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);

  // ---- copy slots: element e = tid + k·NT of the (ROWS × (tx+2)) halo tile.  Elements outside the
  // grid copy 0 bytes (zero fill) from a valid address (element 0 of the same plane).
  const int tid = threadIdx.x;
  int goff[KS];        // in-plane element offset y·nx + x (0 outside the grid)
  uint32_t sdst[KS];   // byte offset of the w element in a stage (~0u: no element for this slot)
  bool gin[KS];
#pragma unroll
  for (int k = 0; k < KS; k++) {
    const int e = tid + k * NT;
    const int r = e / (tx + 2), cc = e - r * (tx + 2);
    const int gx = X0 - 1 + cc, gy = Y0 - 1 + r;
    const bool in_tile = r < ROWS;
    sdst[k] = in_tile ? 4u * (uint32_t)(r * CP_PMAX + cc) : ~0u;
    gin[k] = in_tile && gx >= 0 && gx < nx && gy >= 0 && gy < ny;
    goff[k] = gin[k] ? gy * nx + gx : 0;
  }
  const float2* ug[NR];
#pragma unroll
  for (int r = 0; r < NR; r++) ug[r] = p.u + (long long)(rhs0 + r) * p.fstride;
  auto issue = [&](int j) {
    if (j < nplanes) {
      const int pl = zc0 - 1 + j;
      const int zg = p.z0 + pl;
      const bool zin = zg >= 0 && zg < p.nzg;
      const int po = (pl + 1) * plane;
      const uint32_t st = ring_s + (uint32_t)(j % S) * stage_bytes;
#pragma unroll
      for (int k = 0; k < KS; k++) {
        if (sdst[k] == ~0u) continue;
        const bool ok = zin && gin[k];
        const int o = goff[k] + po;
        cp_async4(st + sdst[k], p.w + o, ok ? 4u : 0u);
#pragma unroll
        for (int r = 0; r < NR; r++)
          if (act[r]) cp_async8(st + wbytes + (uint32_t)r * ubytes + 2u * sdst[k], ug[r] + o, ok ? 8u : 0u);
      }
    }
    cp_commit();
  };
  for (int j = 0; j < S - 1; j++) issue(j);

  // stage the coefficient table while the first planes stream in
  for (int e = tid; e < p.tab_n * CTAB_STRIDE; e += NT) stab[e] = p.ctab[(long long)p.tab_lo * CTAB_STRIDE + e];

  // ---- this thread's position (threads past tx·TY/NY duplicate position 0 and never store)
  const bool pos_ok = tid < tx * (TY / NY);
  const int pt = pos_ok ? tid : 0;
  const int s_ = pt / tx, c_ = pt - s_ * tx;
  const int x = X0 + c_;
  const int yl0 = Y0 + NY * s_;
  const bool x_ok = pos_ok && x >= X0n;
  const int sbase = (NY * s_) * CP_PMAX + c_;   // stage element of (row y0-1, column x-1)
  bool st_ok[NY];
#pragma unroll
  for (int i = 0; i < NY; i++) st_ok[i] = x_ok && yl0 + i >= Y0n;

  // PML deltas of this thread's column / rows (warp-uniform use); dn = (−δ.y, δ.y)
  bool gen_x = false, gen_y = false;
  C dxm = make_float2(0.f, 0.f), dxp = dxm, dxmn = dxm, dxpn = dxm, dym[NY], dyp[NY], dymn[NY], dypn[NY];
#pragma unroll
  for (int i = 0; i < NY; i++) dym[i] = dyp[i] = dymn[i] = dypn[i] = dxm;
  if (PXY) {
    const bool xp = pos_ok && (x < p.lo[0] || x > p.hi[0]);
    bool yp = false;
#pragma unroll
    for (int i = 0; i < NY; i++) yp = yp || (pos_ok && (yl0 + i < p.lo[1] || yl0 + i > p.hi[1]));
    gen_x = __any_sync(FULL, xp);
    gen_y = __any_sync(FULL, yp);
    if (gen_x) {
      dxm = p.dm[0][x];
      dxp = p.dp[0][x];
      dxmn = zneg_sw(dxm);
      dxpn = zneg_sw(dxp);
    }
    if (gen_y) {
#pragma unroll
      for (int i = 0; i < NY; i++) {
        dym[i] = p.dm[1][yl0 + i];
        dyp[i] = p.dp[1][yl0 + i];
        dymn[i] = zneg_sw(dym[i]);
        dypn[i] = zneg_sw(dyp[i]);
      }
    }
  }
  const bool gen_col = gen_x || gen_y;
  const int zlo = p.lo[2], zhi = p.hi[2];

  constexpr int SP = SmemPitch<R>::V;
  const R s_k1 = p.inv_fh * p.inv_dg, s_k0 = -p.g_min * p.inv_dg, s_max = (R)(p.n_g - 1);
  const R w2 = p.w2;
  const R i3h = p.inv3ih2, i2h = p.inv2ih2, i1h = p.invih2;
  auto c0_of = [](const Coef6<R>& c) { return -fma(R(6), c.c1, fma(R(12), c.c2, R(8) * c.c3)); };
  auto m0_of = [&](const Coef6<R>& c, R m0s) { return fma(w2, m0s, -fma(R(6), c.m1, fma(R(12), c.m2, R(8) * c.m3))); };

  DotT part[NR][K > 0 ? K : 1];
#pragma unroll
  for (int r = 0; r < NR; r++)
#pragma unroll
    for (int k = 0; k < (K > 0 ? K : 1); k++) part[r][k] = DotT(0);

  // output / epilogue element of (row yl0, column x) in plane storage 0 of each RHS: + pl·plane
  const long long orow = (long long)yl0 * nx + x;

  // One input plane j (local pl = zc0-1+j).  Three register slots per quantity rotate through the
  // roles prev (output pl-1) / cur (output pl) / next (output pl+1) over three consecutive calls, so no
  // values are copied: cX = coefficients (+ m0 scale), aX = partial sums, sX = centre u (DOT4's s).
  auto body = [&](Coef6<R> (&cP)[NY], Coef6<R> (&cC)[NY], Coef6<R> (&cN)[NY], R (&mP)[NY], R (&mC)[NY],
                  R (&mN)[NY], C (&aP)[NR][NY], C (&aC)[NR][NY], C (&aN)[NR][NY], C (&sP)[NR][NY],
                  C (&sC)[NR][NY], int j) {
    const int pl = zc0 - 1 + j;
    const bool do_prev = (pl - 1 >= zc0);
    const bool do_next = (pl + 1 < zc1);
    const int oplane = pl * plane;   // storage plane pl = local output plane pl-1
    // epilogue operand r̂0 of the outputs finalised here (plane pl-1), loaded before the wait
    C e1[NR][NY];
#pragma unroll
    for (int r = 0; r < NR; r++)
#pragma unroll
      for (int i = 0; i < NY; i++) {
        e1[r][i] = make_float2(0.f, 0.f);
        if (K > 0 && act[r] && do_prev && st_ok[i])
          e1[r][i] = ldg_c(p.rhat + (long long)(rhs0 + r) * p.fstride + orow + (oplane + i * nx));
      }
    // planes j and j+1 have landed (own copies), then every thread's copies; the slot of plane j-1
    // is free (all threads are past iteration j-1) and receives plane j+S-1
    cp_wait<S - 3>();
    __syncthreads();
    issue(j + S - 1);

    const unsigned char* st = ring + (size_t)(j % S) * stage_bytes;
    const float* sw = reinterpret_cast<const float*>(st) + sbase;
    const int zg = p.z0 + pl;
    bool zp_prev = false, zp_cur = false, zp_next = false, zcorr = false;
    if (PML) {
      zp_prev = do_prev && (zg - 1 < zlo || zg - 1 > zhi);
      zp_cur = (pl >= zc0 && pl < zc1) && (zg < zlo || zg > zhi);
      zp_next = do_next && (zg + 1 < zlo || zg + 1 > zhi);
      zcorr = zp_prev || zp_cur || zp_next;
    }
    // ---- w of the 3 × (NY+2) in-plane neighbourhood (shared by the NR fields)
    float wa[NY + 2], w0[NY + 2], wb[NY + 2];
#pragma unroll
    for (int r = 0; r < NY + 2; r++) {
      wa[r] = sw[r * CP_PMAX];
      w0[r] = sw[r * CP_PMAX + 1];
      wb[r] = sw[r * CP_PMAX + 2];
    }
    // ---- coefficients of the output rows of plane pl+1 (w from the next stage) into the free slot
    {
      const float* swn = reinterpret_cast<const float*>(ring + (size_t)((j + 1) % S) * stage_bytes) + sbase;
#pragma unroll
      for (int i = 0; i < NY; i++) {
        const R wn = do_next ? swn[(1 + i) * CP_PMAX + 1] : R(1);
        const R vv = rsqrt_r(wn);
        R sidx = fma(vv, s_k1, s_k0);
        sidx = fmin(fmax(sidx, R(0)), s_max);
        const int ii = min((int)sidx, p.n_g - 2);
        const R tau = sidx - (R)ii;
        const int li = min(max(ii - p.tab_lo, 0), p.tab_n - 2);
        const R* row = stab + li * SP;
        const float4 ta = lds4<R>(row), tb = lds4<R>(row + 4), td = lds4<R>(row + 8);
        cN[i].c1 = fma(tau, tb.z, ta.x);
        cN[i].c2 = fma(tau, tb.w, ta.y);
        cN[i].c3 = fma(tau, td.x, ta.z);
        cN[i].m1 = fma(tau, td.y, ta.w);
        cN[i].m2 = fma(tau, td.z, tb.x);
        cN[i].m3 = fma(tau, td.w, tb.y);
        if (COLLOC) {
          cN[i].m1 *= wn;
          cN[i].m2 *= wn;
          cN[i].m3 *= wn;
        }
        mN[i] = COLLOC ? wn : R(1);
      }
    }
    C dzp = make_float2(0.f, 0.f), dzc = dzp, dzn = dzp;
    if (PML && zcorr) {
      if (zp_prev) dzp = p.dp[2][zg - 1];
      if (zp_cur) {
        const C dz = cadd(p.dm[2][zg], p.dp[2][zg]);
        dzc = make_cx(-dz.x, -dz.y);
      }
      if (zp_next) dzn = p.dm[2][zg + 1];
    }

#pragma unroll
    for (int r = 0; r < NR; r++) {
      if (!act[r]) continue;
      const C* su = reinterpret_cast<const C*>(st + wbytes + (size_t)r * ubytes) + sbase;
      C X[NY + 2], q[NY + 2], Xq[NY + 2], U[NY + 2];
#pragma unroll
      for (int k = 0; k < NY + 2; k++) {
        const C a = su[k * CP_PMAX], u0 = su[k * CP_PMAX + 1], b = su[k * CP_PMAX + 2];
        U[k] = u0;
        X[k] = cadd(a, b);
        if (!COLLOC) {
          q[k] = cscale(w0[k], u0);
          Xq[k] = cfma(wb[k], b, cscale(wa[k], a));
        }
      }
#pragma unroll
      for (int i = 0; i < NY; i++) {
        const C u0 = U[i + 1];
        const C Y = cadd(U[i], U[i + 2]);
        const C P1 = cadd(X[i + 1], Y);
        const C P2 = cadd(X[i], X[i + 2]);
        const C Q0 = COLLOC ? u0 : q[i + 1];
        const C Q1 = COLLOC ? P1 : cadd(Xq[i + 1], cadd(q[i], q[i + 2]));
        const C Q2 = COLLOC ? P2 : cadd(Xq[i], Xq[i + 2]);
        C a = aP[r][i];
        a = cfma(cP[i].c1, u0, a);
        a = cfma(cP[i].c2, P1, a);
        a = cfma(cP[i].c3, P2, a);
        a = cfma(cP[i].m1, Q0, a);
        a = cfma(cP[i].m2, Q1, a);
        a = cfma(cP[i].m3, Q2, a);
        C b = aC[r][i];
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
        if (PML && ((PXY && gen_col) || zcorr)) {
          // PML transverse weights of the three output rows (t2 = c3 h²/3, t1 = t2 + c2 h²/2, t0 = c1 h² + 4 t1)
          const R pt2 = cP[i].c3 * i3h, pt1 = fma(cP[i].c2, i2h, pt2);
          const R ct2 = cC[i].c3 * i3h, ct1 = fma(cC[i].c2, i2h, ct2), ct0 = fma(cC[i].c1, i1h, R(4) * ct1);
          const R nt2 = cN[i].c3 * i3h, nt1 = fma(cN[i].c2, i2h, nt2);
          if (PXY && gen_col) {
            // ΔL1 = δx(u) + δy(u), ΔL2 = δx(Y) + δy(X) (A8); x-neighbour columns from shared memory
            C L1 = make_float2(0.f, 0.f), L2 = L1;
            if (gen_x) {
              const C YL = cadd(su[i * CP_PMAX], su[(i + 2) * CP_PMAX]);
              const C YR = cadd(su[i * CP_PMAX + 2], su[(i + 2) * CP_PMAX + 2]);
              L1 = zfma_c(dxm, dxmn, csub(su[(i + 1) * CP_PMAX], u0), L1);
              L1 = zfma_c(dxp, dxpn, csub(su[(i + 1) * CP_PMAX + 2], u0), L1);
              L2 = zfma_c(dxm, dxmn, csub(YL, Y), L2);
              L2 = zfma_c(dxp, dxpn, csub(YR, Y), L2);
            }
            if (gen_y) {
              L1 = zfma_c(dym[i], dymn[i], csub(U[i], u0), L1);
              L1 = zfma_c(dyp[i], dypn[i], csub(U[i + 2], u0), L1);
              L2 = zfma_c(dym[i], dymn[i], csub(X[i], X[i + 1]), L2);
              L2 = zfma_c(dyp[i], dypn[i], csub(X[i + 2], X[i + 1]), L2);
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
              C B3 = cscale(fma(cP[i].c1, i1h, R(4) * pt1), u0);
              B3 = cfma(pt1, P1, B3);
              B3 = cfma(pt2, P2, B3);
              a = zfma_c(dzp, zneg_sw(dzp), B3, a);
            }
            if (zp_cur) {
              C B3 = cscale(ct0, u0);
              B3 = cfma(ct1, P1, B3);
              B3 = cfma(ct2, P2, B3);
              b = zfma_c(dzc, zneg_sw(dzc), B3, b);
            }
            if (zp_next) {
              C B3 = cscale(fma(cN[i].c1, i1h, R(4) * nt1), u0);
              B3 = cfma(nt1, P1, B3);
              B3 = cfma(nt2, P2, B3);
              c = zfma_c(dzn, zneg_sw(dzn), B3, c);
            }
          }
        }
        aC[r][i] = b;   // output pl: "prev" of the next call
        aN[r][i] = c;   // output pl+1: "cur" of the next call (a's slot is free after this call)
        if (EPI == EPI_DOT4) sC[r][i] = u0;   // s of output pl: "prev" s of the next call
        if (do_prev && st_ok[i]) {
          const long long o = (long long)(rhs0 + r) * p.fstride + orow + (oplane + i * nx);
          p.au[o] = a;
          if (EPI == EPI_DOT1) {
            cp_cdot(part[r][0], part[r][1], e1[r][i], a);
          } else if (EPI == EPI_DOT4) {
            const C sv = sP[r][i];
            cp_cdot(part[r][0], part[r][1], a, sv);
            cp_norm(part[r][2], a);
            cp_cdot(part[r][3], part[r][4], e1[r][i], sv);
            cp_cdot(part[r][5], part[r][6], e1[r][i], a);
          }
        }
      }
    }
  };

  Coef6<R> cs0[NY], cs1[NY], cs2[NY];
  R ms0[NY], ms1[NY], ms2[NY];
  C as0[NR][NY], as1[NR][NY], as2[NR][NY], ss0[NR][NY], ss1[NR][NY], ss2[NR][NY];
#pragma unroll
  for (int i = 0; i < NY; i++) {
    cs0[i] = cs1[i] = cs2[i] = Coef6<R>{0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    ms0[i] = ms1[i] = ms2[i] = 0.f;
#pragma unroll
    for (int r = 0; r < NR; r++) as0[r][i] = as1[r][i] = as2[r][i] = ss0[r][i] = ss1[r][i] = ss2[r][i] = make_float2(0.f, 0.f);
  }
  // roles (prev, cur, next) = (0,1,2), (1,2,0), (2,0,1); the s slots (prev, cur) rotate likewise
  int j = 0;
  for (; j + 2 < nplanes; j += 3) {
    body(cs0, cs1, cs2, ms0, ms1, ms2, as0, as1, as2, ss0, ss1, j);
    body(cs1, cs2, cs0, ms1, ms2, ms0, as1, as2, as0, ss1, ss2, j + 1);
    body(cs2, cs0, cs1, ms2, ms0, ms1, as2, as0, as1, ss2, ss0, j + 2);
  }
  if (j < nplanes) body(cs0, cs1, cs2, ms0, ms1, ms2, as0, as1, as2, ss0, ss1, j);
  if (j + 1 < nplanes) body(cs1, cs2, cs0, ms1, ms2, ms0, as1, as2, as0, ss1, ss2, j + 1);
  cp_wait<0>();

  if (K > 0) {
    const int nblocks = p.cp_nblocks;
    const int slot = item0 + blockIdx.x;
#pragma unroll
    for (int r = 0; r < NR; r++) {
      if (!act[r]) continue;   // uniform
      double pd[K > 0 ? K : 1];
#pragma unroll
      for (int k = 0; k < K; k++) pd[k] = (double)part[r][k];
      const int rr = rhs0 + r;
      block_grid_reduce<K, NT>(pd, p.partials + (long long)rr * nblocks * K, p.dots + (long long)rr * K,
                               p.tickets + rr, nblocks, slot);
    }
  }
}

}  // namespace hz
