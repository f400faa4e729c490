// K2 for complex64, every point of the slab: RHS-fused, cp.async-staged plane tiles sliding in z.
//
// Same operator and per-point operation order as apply27_v2 / apply27_tma (class-sum form, SURVEY
// App. A.5; PML per-axis corrections, reading A8), organised for the BiCGSTAB regime — several RHS,
// grids of ~10⁶ points, 40% of them in the PML — where the register-path launches were latency bound
// (12 warps/SM, one plane of loads in flight) and recomputed the coefficients once per RHS:
//  * One CTA owns a tile of tx × ty output columns/rows (tx ≤ 64, tx·ty ≤ 512: 512/NY threads, each
//    owning column t % tx and NY rows of strip t / tx; no idle lanes for ragged widths such as 101)
//    for NR right-hand sides and marches a z-chunk.  The host cuts the grid into x/y bands — the PML
//    slabs of each axis and the interior — and tiles each band separately, so a tile is either wholly
//    in the x/y-PML or wholly outside it.
//  * Each plane's w tile and the NR u tiles (+1 halo row/column) are copied global → shared by
//    cp.async (4/8-byte, zero-filled outside the grid: the Dirichlet boundary costs no branch) into a
//    ring of HZ_CP_STAGES planes; two planes are in flight while one is consumed.
//  * Per plane and point the coefficients (table interpolation, PML transverse weights) are computed
//    once and used for all NR fields; per field the 9 in-plane neighbours come from shared memory.
//  * Three instantiations: x/y-PML tiles (x / y corrections in warp-uniform branches plus the plane-
//    uniform z corrections, the register path's A8 form), z-PML-only tiles, PML-free tiles.  A
//    correction with δ = 0 adds exact zeros, so all compute bitwise the same value for a point.
//  * Dot epilogues accumulate per thread in fp32 (HZ_CP_DOT_F64 = 1: fp64 as the register path) and
//    reduce per block and grid in fp64 in a fixed order.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "apply27.cuh"

namespace hz {

// A CTA has CP_THREADS = 256 threads; with NY rows per thread its tile is tx × ty points (tx ≤ 64,
// tx·ty ≤ 256·NY, (tx+2)·(ty+2) ≤ CP_HALO, ty even), the halo tile copied with CP_SLOTS elements
// per thread.  Shared rows have pitch tx + 2.
constexpr int CP_NTHR = 256;
constexpr int CP_HALO = 768;
__host__ __device__ constexpr int CP_THREADS(int) { return CP_NTHR; }
__host__ __device__ constexpr int CP_TILE_PTS(int ny) { return CP_NTHR * ny; }
__host__ __device__ constexpr int CP_SLOTS(int) { return (CP_HALO + CP_NTHR - 1) / CP_NTHR; }
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

// bytes of one ring stage: the w halo tile then NR u halo tiles, CP_HALO elements each
__host__ __device__ constexpr size_t cp_stage_bytes(int nr) { return (size_t)CP_HALO * (4 + 8 * nr); }
// DOT4 reads its s operand (the centre u of the previous plane) back from the ring, which keeps one
// more plane resident: one more stage, same lookahead
#ifndef HZ_CP_S_SMEM
#define HZ_CP_S_SMEM 0
#endif
__host__ __device__ constexpr int cp_stages(int epi) { return CP_STAGES + ((HZ_CP_S_SMEM && epi == 2) ? 1 : 0); }
__host__ __device__ constexpr size_t cp_smem_bytes(int tab_n, int nr, int epi) {
  return (((size_t)tab_n * 12 * 4 + 127) / 128) * 128 + (size_t)cp_stages(epi) * cp_stage_bytes(nr);
}
// work item {x0 | y0 << 16, tx | ty << 8 | (xs − x0) << 16 | (ys − y0) << 24, z0 | z1 << 16,
// (xe − x0) | (ye − y0) << 8 | mode << 16}: the tile computes [x0, x0+tx) × [y0, y0+ty) and stores
// [xs, xe) × [ys, ye) (tiles overlap where a band is not a multiple of the tile), planes [z0, z1)
__host__ __device__ inline int4 cp_item(int x0, int y0, int tx, int ty, int xs, int ys, int xe, int ye, int z0, int z1, int mode) {
  return make_int4(x0 | (y0 << 16), tx | (ty << 8) | ((xs - x0) << 16) | ((ys - y0) << 24), z0 | (z1 << 16),
                   (xe - x0) | ((ye - y0) << 8) | (mode << 16));
}

// 4 / 8-byte async copies global → shared; zfill = true writes zeros instead (src not read)
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, bool zfill) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n cp.async.ca.shared.global [%0], [%1], 4, p;\n}\n" ::"r"(dst),
      "l"(src), "r"((int)zfill)
      : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src, bool zfill) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n cp.async.ca.shared.global [%0], [%1], 8, p;\n}\n" ::"r"(dst),
      "l"(src), "r"((int)zfill)
      : "memory");
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

// Dot epilogue reduction of one CTA for its NR right-hand sides (all K values at once, fixed order):
// warp shuffles (fp64) → per-warp sums in shared memory → one thread per (RHS, value) writes the
// block's partial; the last CTA of the RHS group (ticket of the group's first RHS) reduces the
// partials of all CTAs with one warp per (RHS, value): lanes stride the blocks, then a shuffle tree.
template <int NR, int K, int NT>
__device__ __forceinline__ void cp_reduce(const DotT (&part)[NR][K], const bool (&act)[NR], const ApplyParams<float, float>& p,
                                          int rhs0, int slot) {
  constexpr int NWARP = NT / 32;
  __shared__ double red[NWARP][NR * K];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nblocks = p.cp_nblocks;
#pragma unroll
  for (int r = 0; r < NR; r++)
#pragma unroll
    for (int k = 0; k < K; k++) {
      double v = (double)part[r][k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[warp][r * K + k] = v;
    }
  __syncthreads();
  if (threadIdx.x < NR * K) {
    const int r = threadIdx.x / K, k = threadIdx.x - r * K;
    if (act[r]) {
      double v = 0.0;
      for (int w = 0; w < NWARP; w++) v += red[w][threadIdx.x];
      p.partials[((long long)(rhs0 + r) * nblocks + slot) * K + k] = v;
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(p.tickets + rhs0, 1u) == (unsigned)nblocks - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int q = warp; q < NR * K; q += NWARP) {
    const int r = q / K, k = q - r * K;
    if (!act[r]) continue;
    const volatile double* pp = p.partials + (long long)(rhs0 + r) * nblocks * K + k;
    double v = 0.0;
    for (int b = lane; b < nblocks; b += 32) v += pp[(long long)b * K];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) p.dots[(long long)(rhs0 + r) * K + k] = v;
  }
  if (threadIdx.x == 0) p.tickets[rhs0] = 0u;
}

// Work item: see cp_item (local plane indices)
template <int NY, int NR, bool COLLOC, int EPI, int PM, bool GAM>
__device__ __forceinline__ void cp_body(const ApplyParams<float, float>& p, int item0) {
  typedef float R;
  typedef float2 C;
  constexpr bool PML = PM != CP_LEAN;
  constexpr bool PXY = PM == CP_PMLXY;
  constexpr int NT = CP_THREADS(NY);
  constexpr int KS = CP_SLOTS(NY);
  constexpr int K = epi_k(EPI);
  constexpr bool SSM = HZ_CP_S_SMEM && EPI == EPI_DOT4;   // s operand from the ring
  constexpr int S = cp_stages(EPI);
  constexpr int L = SSM ? S - 2 : S - 1;                   // planes issued ahead
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
  const int X0 = item.x & 0xffff, Y0 = item.x >> 16;
  const int tx = item.y & 0xff, TY = (item.y >> 8) & 0xff;
  const int X0n = X0 + ((item.y >> 16) & 0xff), Y0n = Y0 + (item.y >> 24);
  const int X1n = X0 + (item.w & 0xff), Y1n = Y0 + ((item.w >> 8) & 0xff);
  const int ROWS = TY + 2, P = tx + 2;   // halo tile rows, shared row pitch
  const int zc0 = item.z & 0xffff, zc1 = item.z >> 16;
  const int nplanes = zc1 - zc0 + 2;   // input planes zc0-1 .. zc1
  const int plane = (int)p.plane;      // host: (nzl + 2)·plane < 2^31 (32-bit offsets within a field)

  extern __shared__ __align__(1024) unsigned char smem_cp[];
  float* stab = reinterpret_cast<float*>(smem_cp);
  unsigned char* ring = smem_cp + (((size_t)p.tab_n * 12 * 4 + 127) / 128) * 128;
  const uint32_t stage_bytes = (uint32_t)cp_stage_bytes(NR);
  const uint32_t wbytes = (uint32_t)CP_HALO * 4;   // w halo tile of a stage; the u tiles follow
  const uint32_t ubytes = (uint32_t)CP_HALO * 8;
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);

  // ---- copy slots: element e = tid + k·NT of the (ROWS × (tx+2)) halo tile.  Elements outside the
  // grid copy 0 bytes (zero fill) from a valid address (element 0 of the same plane).  Addresses are a
  // uniform base + an unsigned 32-bit element offset (host: fstride < 2^31, so r·fstride + offset < 2^32
  // for the NR ≤ 2 fields of a group).
  const int tid = threadIdx.x;
  int goff[KS];        // in-plane element offset y·nx + x (0 outside the grid)
  uint32_t sdst[KS];   // byte offset of the w element in a stage (~0u: no element for this slot)
  bool gout[KS];       // element outside the grid: zero fill
#pragma unroll
  for (int k = 0; k < KS; k++) {
    const int e = tid + k * NT;
    const int r = e / P, cc = e - r * P;
    const int gx = X0 - 1 + cc, gy = Y0 - 1 + r;
    const bool in_tile = r < ROWS;
    const bool gin = in_tile && gx >= 0 && gx < nx && gy >= 0 && gy < ny;
    sdst[k] = in_tile ? 4u * (uint32_t)e : ~0u;
    gout[k] = !gin;
    goff[k] = gin ? gy * nx + gx : 0;
  }
  const uint32_t fs = (uint32_t)p.fstride;
  const float2* __restrict__ ug0 = p.u + (long long)rhs0 * p.fstride;
#ifndef HZ_CP_NO_OPAQUE
  asm("mov.b64 %0, %0;" : "+l"(ug0));   // keep the group's base in a register (not re-derived per use)
#endif
  const float* __restrict__ wg = p.w;
  auto issue = [&](int j) {
    if (j < nplanes) {
      const int pl = zc0 - 1 + j;
      const int zg = p.z0 + pl;
      const bool zout = !(zg >= 0 && zg < p.nzg);
      const int po = (pl + 1) * plane;
      const uint32_t st = ring_s + (uint32_t)(j % S) * stage_bytes;
#pragma unroll
      for (int k = 0; k < KS; k++) {
        if (sdst[k] == ~0u) continue;
        const bool zf = zout || gout[k];
        const uint32_t o = (uint32_t)(goff[k] + po);
        cp_async4(st + sdst[k], wg + o, zf);
#pragma unroll
        for (int r = 0; r < NR; r++)
          if (act[r]) cp_async8(st + wbytes + (uint32_t)r * ubytes + 2u * sdst[k], ug0 + (o + (uint32_t)r * fs), zf);
      }
    }
    cp_commit();
  };
  for (int j = 0; j < L; j++) issue(j);

  // stage the coefficient table while the first planes stream in
  for (int e = tid; e < p.tab_n * CTAB_STRIDE; e += NT) stab[e] = p.ctab[(long long)p.tab_lo * CTAB_STRIDE + e];

  // ---- this thread's position (threads past tx·TY/NY duplicate position 0 and never store)
  const bool pos_ok = tid < tx * (TY / NY);
  const int pt = pos_ok ? tid : 0;
  const int s_ = pt / tx, c_ = pt - s_ * tx;
  const int x = X0 + c_;
  const int yl0 = Y0 + NY * s_;
  const bool x_ok = pos_ok && x >= X0n && x < X1n;
  const int sbase = (NY * s_) * P + c_;   // stage element of (row y0-1, column x-1)
  bool st_ok[NY];
#pragma unroll
  for (int i = 0; i < NY; i++) st_ok[i] = x_ok && yl0 + i >= Y0n && yl0 + i < Y1n;

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
  const uint32_t orow = (uint32_t)(yl0 * nx + x);
  // GAm: the 5 weights of this thread's rows of the next coefficient plane, loaded one call ahead
  R gpf[NY][5];
  auto gam_load = [&](R (&g)[5], int splane, int i) {
    const long long e = (long long)splane * plane + orow + i * nx;
#pragma unroll
    for (int k = 0; k < 5; k++) g[k] = __ldg(p.gam + k * p.fstride + e);
  };
  if (GAM) {
#pragma unroll
    for (int i = 0; i < NY; i++) {
      gam_load(gpf[i], zc0 + 1, i);   // rows of output plane zc0 (storage zc0 + 1), used by call j = 0
    }
  }
  const float2* __restrict__ rh0 = p.rhat + (long long)rhs0 * p.fstride;
  float2* __restrict__ au0 = p.au + (long long)rhs0 * p.fstride;
#ifndef HZ_CP_NO_OPAQUE
  asm("mov.b64 %0, %0;" : "+l"(rh0));
  asm("mov.b64 %0, %0;" : "+l"(au0));
#endif

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
          e1[r][i] = ldg_c(rh0 + ((uint32_t)r * fs + orow + (uint32_t)(oplane + i * nx)));
      }
    // planes j and j+1 have landed (own copies), then every thread's copies; the slot of plane j+L-S
    // (j-1, or j-2 when the previous plane's centre is still read) is free — every thread is past the
    // iteration that last read it — and receives plane j+L
    cp_wait<L - 2>();
    __syncthreads();
    issue(j + L);

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
      wa[r] = sw[r * P];
      w0[r] = sw[r * P + 1];
      wb[r] = sw[r * P + 2];
    }
    // ---- coefficients of the output rows of plane pl+1 (w from the next stage) into the free slot
    {
      const float* swn = reinterpret_cast<const float*>(ring + (size_t)((j + 1) % S) * stage_bytes) + sbase;
#pragma unroll
      for (int i = 0; i < NY; i++) {
        const R wn = do_next ? swn[(1 + i) * P + 1] : R(1);
        if (GAM) {   // GAm: the row's 27-node mean weights (A19), prefetched one plane ahead
          if (do_next) {
            const R t1 = gpf[i][0], t2 = gpf[i][1], mu0 = gpf[i][2], mu1 = gpf[i][3], mu2 = gpf[i][4];
            const R t0 = R(1) - R(4) * (t1 + t2);
            cN[i].c1 = p.ih2 * (t0 - R(4) * t1);
            cN[i].c2 = p.ih2 * (R(2) * (t1 - t2));
            cN[i].c3 = p.ih2 * (R(3) * t2);
            cN[i].m1 = w2 * mu1;
            cN[i].m2 = w2 * mu2;
            cN[i].m3 = w2 * ((R(1) - mu0 - R(6) * mu1 - R(12) * mu2) * R(0.125));
          } else {
            cN[i] = Coef6<R>{R(0), R(0), R(0), R(0), R(0), R(0)};
          }
          if (pl + 2 < zc1) gam_load(gpf[i], pl + 3, i);   // the next call's rows
        } else {
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
        }
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
        const C a = su[k * P], u0 = su[k * P + 1], b = su[k * P + 2];
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
              const C YL = cadd(su[i * P], su[(i + 2) * P]);
              const C YR = cadd(su[i * P + 2], su[(i + 2) * P + 2]);
              L1 = zfma_c(dxm, dxmn, csub(su[(i + 1) * P], u0), L1);
              L1 = zfma_c(dxp, dxpn, csub(su[(i + 1) * P + 2], u0), L1);
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
        if (EPI == EPI_DOT4 && !SSM) sC[r][i] = u0;   // s of output pl: "prev" s of the next call
        if (do_prev && st_ok[i]) {
          au0[(uint32_t)r * fs + orow + (uint32_t)(oplane + i * nx)] = a;
          if (EPI == EPI_DOT1) {
            cp_cdot(part[r][0], part[r][1], e1[r][i], a);
          } else if (EPI == EPI_DOT4) {
            C sv;
            if (SSM)   // centre u of plane pl-1, still resident in the previous stage
              sv = reinterpret_cast<const C*>(ring + (size_t)((j + S - 1) % S) * stage_bytes + wbytes + (size_t)r * ubytes)[sbase + (i + 1) * P + 1];
            else
              sv = sP[r][i];
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
  // (the ragged end is guarded inside the loop: three body copies, not five — instruction cache)
  for (int j = 0; j < nplanes; j += 3) {
    body(cs0, cs1, cs2, ms0, ms1, ms2, as0, as1, as2, ss0, ss1, j);
    if (j + 1 >= nplanes) break;
    body(cs1, cs2, cs0, ms1, ms2, ms0, as1, as2, as0, ss1, ss2, j + 1);
    if (j + 2 >= nplanes) break;
    body(cs2, cs0, cs1, ms2, ms0, ms1, as2, as0, as1, ss2, ss0, j + 2);
  }
  cp_wait<0>();

  if constexpr (K > 0) cp_reduce<NR, K, NT>(part, act, p, rhs0, item0 + blockIdx.x);
}

// One launch for every tile class: the work item's mode selects the x/y-PML body, the body with the
// plane-uniform z corrections (chunks touching the z-PML) or the PML-free body, so CTAs of all classes
// share the GPU; x/y-PML items come first (heavier, scheduled first).  The PML-free body is a separate
// instantiation because the mere presence of the z-PML code costs ~20% (registers / scheduling).
// GAM: rows read their 27-node mean weights (A19) instead of interpolating the table — a separate
// instantiation (a runtime branch alone slowed the GA kernel by ~5%).
template <int NY, int NR, bool COLLOC, int EPI, bool GAM>
__global__ void __launch_bounds__(CP_NTHR, 2) apply27_cp(ApplyParams<float, float> p, int item0) {
  const int mode = p.cp_work[item0 + blockIdx.x].w >> 16;
  if (mode == CP_PMLXY)
    cp_body<NY, NR, COLLOC, EPI, CP_PMLXY, GAM>(p, item0);
  else if (mode == CP_PMLZ)
    cp_body<NY, NR, COLLOC, EPI, CP_PMLZ, GAM>(p, item0);
  else
    cp_body<NY, NR, COLLOC, EPI, CP_LEAN, GAM>(p, item0);
}

}  // namespace hz
