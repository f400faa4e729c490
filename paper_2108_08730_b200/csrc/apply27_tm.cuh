// K2 for complex64 (north-star steps a2–a6): tensor-map TMA plane tiles sliding in z, two x-points
// per thread, RHS-fused.  DESIGN.md §5.
//
//   (Au)_n = ω² Σ_d μ_{|d|}(w_n) u_{n+d} / v²_{n+d}                        Eq. 8, A2, A4
//          + Σ_a Σ_e D_a(n_a, e) Σ_{p,q} T(p,q; w_n) u_{n+e ê_a+p ê_b+q ê_c}   A6 (App. A), A8
//   w_n = clamped linear interpolation of the Tikhonov weight table at G_n = v_n/(f h)  P:36, A13
//
// Design (HBM-bound: 4 + 16·nrhs bytes per point and apply):
//  * Fields are [nrhs][nz+2][ny][ldx] with a 32-byte row pitch (ldx = nx rounded up to 4), so one
//    3-D (w) and one 4-D (u: x, y, plane, RHS) tensor map describe them.  The work list holds items
//    (a tx × ty tile × a z-chunk, tx ∈ {32, 64}); a persistent grid of one CTA per SM walks it
//    round-robin, each CTA for NR right-hand sides.  Per input plane ONE thread issues one TMA box per
//    field — the halo tile of w and of each RHS's u — into a ring of shared-memory stages with one
//    mbarrier each
//    (expect_tx); coordinates outside the grid (x, y, and z where the map is trimmed to the slab's
//    in-grid planes) are zero-filled by the TMA unit: the Dirichlet boundary (A9) costs no code.
//  * A stage is refilled as soon as every warp has finished with it: the consumer warps `bar.arrive` on
//    the stage's named barrier, the last warp `bar.sync`s on it and its lane 0 issues the next plane of the
//    CTA's sequence — across item boundaries, so the ring does not drain between items; no CTA-wide
//    barrier per plane.
//  * Thread (pair c, row r) computes the two points (x0 − 1 + 2c, x0 + 2c) of its row: per halo row it
//    reads the four u columns 2c .. 2c+3 as two 16-byte shared loads and the four w as two 8-byte
//    loads, and the x-neighbour / y-neighbour class sums come from registers:
//    P0 = u, P1 = 4 in-plane faces, P2 = 4 in-plane corners, Q0..Q2 of q = u·w (Eq. 8), scattered into
//    the partial outputs of planes k−1, k, k+1 (18 packed FFMA2 per point).  Row coefficients are
//    built once per point and plane from w (one MUFU.RSQ, clamped linear interpolation of the table
//    staged in shared memory) and shared by the NR fields; c0 and m0 follow from the sum rules.
//  * PML: warp-uniform branches (the same per-axis A8 corrections as the complex128 kernel); a
//    correction with δ = 0 adds exact zeros, so every point is computed with the same operation
//    sequence whichever tile, chunk, launch or slab computes it (bitwise z-slab invariance).
//  * Output: one 8-byte store per point; the pad columns [nx, ldx) are written as zeros.
//  * Epilogues (BiCGSTAB dots): each thread's pair products in fp32, summed over planes in fp64, then
//    an fp64 block and grid reduction in a fixed order (tm_reduce).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "apply27.cuh"

namespace hz {

constexpr int TM_NTHR = 384;     // threads per CTA (12 warps, one CTA per SM, ≤ 168 registers)
constexpr int TM_MAXTX = 64;     // widest tile

// PML mode bits of a work item: TM_PMLZ the chunk holds z-PML planes, TM_PMLXY the tile holds x/y-PML
// columns / rows; TM_LEAN neither
enum { TM_LEAN = 0, TM_PMLZ = 1, TM_PMLXY = 2 };

// work item {x0 | y0 << 16, z0 | z1 << 16, mode, 0}: tile origin (x0, y0), local planes [z0, z1)
__host__ __device__ inline int4 tm_item(int x0, int y0, int z0, int z1, int mode) {
  return make_int4(x0 | (y0 << 16), z0 | (z1 << 16), mode, 0);
}

// tile geometry shared by host and device: box widths and stage sizes (bytes, 128-aligned)
// A tile of tx ∈ {32, 64} columns with origin X0 (a multiple of tx) computes the points
// x ∈ [X0 − 1, X0 + tx − 1): pair c is (X0 − 1 + 2c, X0 + 2c).  The TMA unit needs the box's innermost
// start coordinate 16-byte aligned (a misaligned start faults), so the u box starts at X0 − 2 and the
// w box at X0 − 4 — and with the pair starting one column left of X0, a thread's four columns
// x − 1 .. x + 2 sit at 16-byte (u) / 8-byte (w) aligned shared addresses: two vector loads each.  The
// w box is widened to a row pitch ≡ 16 (mod 32) words so the two rows a half-warp reads hit disjoint
// banks.  A warp covers 8 pairs × 4 rows (so only the warps holding x- or y-PML points take the PML
// corrections), the 12 warps of a CTA tx/16 × 192/tx such blocks: ty = 768/tx rows.
__host__ __device__ constexpr int tm_bxu(int tx) { return tx + 2; }
__host__ __device__ constexpr int tm_bxw(int tx) { return ((tx + 4 + 15) / 32) * 32 + 16; }
__host__ __device__ constexpr uint32_t tm_r128(uint32_t b) { return (b + 127u) & ~127u; }
// bytes one box delivers (the mbarrier's transaction count) and its 128-byte aligned slot in a stage
__host__ __device__ constexpr uint32_t tm_wbox(int tx, int ty) { return (uint32_t)tm_bxw(tx) * (ty + 2) * 4u; }
__host__ __device__ constexpr uint32_t tm_ubox(int tx, int ty) { return (uint32_t)tm_bxu(tx) * (ty + 2) * 8u; }
__host__ __device__ constexpr uint32_t tm_wbytes(int tx, int ty) { return tm_r128(tm_wbox(tx, ty)); }
__host__ __device__ constexpr uint32_t tm_ubytes(int tx, int ty) { return tm_r128(tm_ubox(tx, ty)); }
__host__ __device__ constexpr uint32_t tm_stage_bytes(int tx, int ty, int nr) { return tm_wbytes(tx, ty) + (uint32_t)nr * tm_ubytes(tx, ty); }
__host__ __device__ constexpr uint32_t tm_tab_bytes(int tab_n) { return tm_r128((uint32_t)tab_n * 12u * 4u); }
// rows per CTA for a tile width tx: TM_NTHR threads of tx/2 column pairs per row
__host__ __device__ constexpr int tm_rows(int tx) { return TM_NTHR / (tx / 2); }

// ---- TMA / mbarrier / named-barrier primitives (PTX) -------------------------------------------
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// Wait for the phase with the given parity to complete.  A transfer that never completes (a
// programming error) traps after ~2^30 polls instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  for (uint32_t n = 0;; n++) {
    asm volatile(
        "{\n .reg .pred P1;\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n selp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    if (n > (1u << 30)) __trap();
  }
}
__device__ __forceinline__ void tma_load3(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_load4(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void bar_sync_n(int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(TM_NTHR) : "memory"); }
__device__ __forceinline__ void bar_arrive_n(int id) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "n"(TM_NTHR) : "memory"); }

// conj(a)·b of complex64 data in fp32 (a thread's pair of points; the sums over planes, threads, blocks
// and the grid are fp64)
__device__ __forceinline__ void tm_cdot(float& re, float& im, float2 a, float2 b) {
  re = fmaf(a.x, b.x, fmaf(a.y, b.y, re));
  im = fmaf(a.x, b.y, fmaf(-a.y, b.x, im));
}
__device__ __forceinline__ void tm_norm(float& s, float2 a) { s = fmaf(a.x, a.x, fmaf(a.y, a.y, s)); }

// complex multiply-add with a per-thread constant d (PML δ): acc + d·b as two packed FMAs,
// dn = (−d.y, d.y) precomputed once
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
__device__ __forceinline__ void tm_reduce(const double (&part)[NR][K], const bool (&act)[NR], const ApplyParams<float, float>& p,
                                          int rhs0, int slot) {
  constexpr int NWARP = NT / 32;
  __shared__ double red[NWARP][NR * K];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nblocks = gridDim.x;
#pragma unroll
  for (int r = 0; r < NR; r++)
#pragma unroll
    for (int k = 0; k < K; k++) {
      double v = part[r][k];
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

// ring depth: planes in flight per CTA (one CTA per SM; ≤ 160 KB of stages at tx = 64)
template <int NR> struct TmStages { enum { S = NR == 1 ? 12 : 8 }; };
__host__ __device__ constexpr int tm_stages(int nr) { return nr == 1 ? 12 : 8; }
// shared memory: S mbarriers (128 B), the ring of S stages, then the staged coefficient rows
__host__ __device__ constexpr size_t tm_ring_end(int tx, int ty, int nr) {
  return 128 + (size_t)tm_stages(nr) * tm_stage_bytes(tx, ty, nr);
}
__host__ __device__ constexpr size_t tm_smem_bytes(int tab_n, int tx, int ty, int nr) {
  return tm_ring_end(tx, ty, nr) + tm_tab_bytes(tab_n);
}

// predicated 8- / 16-byte global stores (branch-free)
__device__ __forceinline__ void st_pred(float2* ptr, float2 v, bool pred) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %0, 0;\n @p st.global.v2.f32 [%1], {%2, %3};\n}\n" ::"r"((int)pred),
               "l"(ptr), "f"(v.x), "f"(v.y)
               : "memory");
}
__device__ __forceinline__ void st_pred4(float2* ptr, float2 a, float2 b, bool pred) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %0, 0;\n @p st.global.v4.f32 [%1], {%2, %3, %4, %5};\n}\n" ::"r"((int)pred),
               "l"(ptr), "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y)
               : "memory");
}

// The kernel: a persistent grid of CTAs (one per SM) walks the work list round-robin; blockIdx.y is
// the group of NR right-hand sides.  Lane 0 of the last warp is the producer: it issues the TMA boxes of the CTA's
// planes in order — across item boundaries, so the ring never drains between items — and refills a
// stage as soon as every warp has released it.  Each item (tile × z-chunk) runs the body its mode
// selects: x/y-PML, z-PML or PML-free.
template <int TX, int NR, bool COLLOC, int EPI, bool GAM>
__global__ void __launch_bounds__(TM_NTHR, 1)
    apply27_tm(const __grid_constant__ CUtensorMap tmw, const __grid_constant__ CUtensorMap tmu, ApplyParams<float, float> p) {
  typedef float R;
  typedef float2 C;
  constexpr int K = epi_k(EPI);
  constexpr int KK = K > 0 ? K : 1;
  constexpr int S = TmStages<NR>::S;
  const unsigned FULL = 0xffffffffu;
  // tile geometry (compile time): TX columns × TY rows, box widths, stage layout
  constexpr int tx = TX, ty = tm_rows(TX);
  constexpr int bxu = tm_bxu(TX), bxw = tm_bxw(TX);
  constexpr uint32_t wB = tm_wbytes(TX, tm_rows(TX)), uB = tm_ubytes(TX, tm_rows(TX));
  constexpr uint32_t stB = wB + (uint32_t)NR * uB;

  const int rhs0 = blockIdx.y * NR;
  bool act[NR];
  bool any = false;
#pragma unroll
  for (int r = 0; r < NR; r++) {
    act[r] = rhs0 + r < p.nrhs && (p.active == nullptr || p.active[rhs0 + r] != 0);
    any = any || act[r];
  }
  if (!any) return;   // uniform per CTA (a converged RHS group)

  const int nx = p.nx, ny = p.ny, ldx = p.ldx;
  const int plane = (int)p.plane;      // host: (nzl + 2)·plane < 2^31 (32-bit offsets within a field)
  const int nitems = p.tm_nitems;

  extern __shared__ __align__(1024) unsigned char smem_tm[];
  const uint32_t mbar0 = (uint32_t)__cvta_generic_to_shared(smem_tm);
  unsigned char* ring = smem_tm + 128;
  const uint32_t ring_s = mbar0 + 128u;
  float* stab = reinterpret_cast<float*>(smem_tm + tm_ring_end(TX, tm_rows(TX), NR));
  uint32_t txB = tm_wbox(tx, ty);   // transaction bytes per plane: the boxes exactly, not their slots
#pragma unroll
  for (int r = 0; r < NR; r++)
    if (act[r]) txB += tm_ubox(tx, ty);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // the producer is lane 0 of the LAST warp: the warp schedulers favour higher warp ids, so the warp
  // that waits for every warp's release and refills the ring is not the one left behind
  constexpr int PWARP = TM_NTHR / 32 - 1;

  // ---- producer (lane 0 of warp PWARP): cursor over the CTA's planes, item after item
  int p_it = blockIdx.x, p_j = 0, p_n = 0, p_x0 = 0, p_y0 = 0, p_c2 = 0, p_st = 0;
  auto p_load = [&]() {
    if (p_it < nitems) {
      const int4 it = p.tm_work[p_it];
      p_x0 = it.x & 0xffff;
      p_y0 = it.x >> 16;
      p_c2 = (it.y & 0xffff) - p.tm_org;   // map coordinate of storage plane zc0 (input plane j = 0)
      p_n = (it.y >> 16) - (it.y & 0xffff) + 2;
      p_j = 0;
    }
  };
  auto issue_next = [&]() {
    if (p_it >= nitems) return;
    const uint32_t bar = mbar0 + 8u * p_st;
    const uint32_t dst = ring_s + (uint32_t)p_st * stB;
    mbar_expect_tx(bar, txB);
    tma_load3(dst, &tmw, bar, p_x0 - 4, p_y0 - 1, p_c2 + p_j);
#pragma unroll
    for (int r = 0; r < NR; r++)
      if (act[r]) tma_load4(dst + wB + (uint32_t)r * uB, &tmu, bar, p_x0 - 2, p_y0 - 1, p_c2 + p_j, rhs0 + r);
    if (++p_st == S) p_st = 0;
    if (++p_j == p_n) {
      p_it += gridDim.x;
      p_load();
    }
  };
  if (warp == PWARP && lane == 0) {
    for (int s = 0; s < S; s++) mbar_init(mbar0 + 8u * s, 1u);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    p_load();
    for (int s = 0; s < S; s++) issue_next();
  }
  // stage the coefficient table while the first planes stream in
  for (int e = tid; e < p.tab_n * CTAB_STRIDE; e += TM_NTHR) stab[e] = p.ctab[(long long)p.tab_lo * CTAB_STRIDE + e];
  __syncthreads();

  // ---- consumer ring cursor (every thread): the stage of the plane being consumed, its phase
  int c_st = 0;
  uint32_t c_ph = 0;
  auto wait_stage = [&](int st, uint32_t ph) { mbar_wait(mbar0 + 8u * st, ph); };

  // ---- thread → points: columns x = X0 − 1 + 2c and x + 1 of row y; warp w covers pairs
  // 8·(w mod WX) + 0..7 of rows 4·(w / WX) + 0..3 (WX = tx/16 warp columns)
  const int wx = tx >> 4;
  const int rg = 4 * (warp / wx) + (lane >> 3), c_ = 8 * (warp % wx) + (lane & 7);
  const int sbw = rg * bxw + 2 * c_ + 2;   // stage element (row y-1, column x-1) in the w box
  const int sbu = rg * bxu + 2 * c_;       // ... in a u box
  const C z2 = make_float2(0.f, 0.f);

  constexpr int SP = SmemPitch<R>::V;
  const R s_k1 = p.inv_fh * p.inv_dg, s_k0 = -p.g_min * p.inv_dg, s_max = (R)(p.n_g - 1);
  const int ig_max = p.n_g - 2, tab_lo = p.tab_lo, tab_n2 = p.tab_n - 2;
  const R w2 = p.w2;
  auto c0_of = [](const Coef6<R>& c) { return -fma(R(6), c.c1, fma(R(12), c.c2, R(8) * c.c3)); };
  auto m0_of = [&](const Coef6<R>& c, R m0s) { return fma(w2, m0s, -fma(R(6), c.m1, fma(R(12), c.m2, R(8) * c.m3))); };
  const uint32_t fs = (uint32_t)p.fstride;
  const float2* __restrict__ rh0 = p.rhat + (long long)rhs0 * p.fstride;
  float2* __restrict__ au0 = p.au + (long long)rhs0 * p.fstride;

  double part[NR][KK];
#pragma unroll
  for (int r = 0; r < NR; r++)
#pragma unroll
    for (int k = 0; k < KK; k++) part[r][k] = 0.0;

  // ---- one work item with body PM (mode bits TM_PMLZ | TM_PMLXY)
  auto run_item = [&](auto PMc, const int4 item) {
    constexpr int PM = decltype(PMc)::value;
    constexpr bool PML = PM != TM_LEAN;
    constexpr bool PXY = (PM & TM_PMLXY) != 0;
    constexpr bool PZ = (PM & TM_PMLZ) != 0;
    const int X0 = item.x & 0xffff, Y0 = item.x >> 16;
    const int zc0 = item.y & 0xffff, zc1 = item.y >> 16;
    const int nplanes = zc1 - zc0 + 2;   // input planes zc0-1 .. zc1
    const int x = X0 - 1 + 2 * c_;
    const int y = Y0 + rg;
    const bool yok = y < ny;
    // a point is stored if it lies in the pitched row (a pad column gets a zero), computed if in the grid
    const bool sto[2] = {yok && x >= 0 && x < ldx, yok && x + 1 < ldx};
    const bool in_[2] = {sto[0] && x < nx, sto[1] && x + 1 < nx};
    // output element (row y, column x) in storage plane 0 of the group's first RHS, + plane offsets;
    // 32-bit arithmetic (wraps back for the never-stored x = −1 of row 0)
    const uint32_t orow = (uint32_t)(y * ldx + x);
    // PML: warp-uniform flags for x-PML columns / y-PML rows among the warp's points; the deltas
    // δ± = a± − h⁻² are read from the (L1-resident) 1-D arrays where they are used
    bool gen_x = false, gen_y = false;
    const int xe0 = min(max(x, 0), nx - 1), xe1 = min(x + 1, nx - 1), ye = min(y, ny - 1);
    if (PXY) {
      bool xp = false;
#pragma unroll
      for (int e = 0; e < 2; e++) xp = xp || (in_[e] && (x + e < p.lo[0] || x + e > p.hi[0]));
      const bool yp = yok && (y < p.lo[1] || y > p.hi[1]);
      gen_x = __any_sync(FULL, xp);
      gen_y = __any_sync(FULL, yp);
    }
    const bool gen_col = gen_x || gen_y;
    const int zlo = p.lo[2], zhi = p.hi[2];
    const R i3h = p.inv3ih2, i2h = p.inv2ih2, i1h = p.invih2;
    R gpf[2][5];   // GAm / record: the 5 weights of this thread's points of the next coefficient plane
    auto gam_load = [&](int splane) {
      const uint32_t e = (uint32_t)(splane * plane) + orow;
#pragma unroll
      for (int k = 0; k < 5; k++)
#pragma unroll
        for (int q = 0; q < 2; q++) gpf[q][k] = in_[q] ? __ldg(p.gam + k * p.fstride + (e + (uint32_t)q)) : R(0);
    };
    if (GAM) gam_load(zc0 + 1);   // rows of output plane zc0 (storage zc0 + 1), used by plane j = 0

    // One input plane j (local pl = zc0-1+j).  Three register slots per quantity rotate through the
    // roles prev (output pl-1) / cur (output pl) / next (output pl+1) over three consecutive calls:
    // cX = coefficients (+ m0 scale), aX = partial sums, sX = centre u (DOT4's s).
    auto body = [&](Coef6<R> (&cP)[2], Coef6<R> (&cC)[2], Coef6<R> (&cN)[2], R (&mP)[2], R (&mC)[2], R (&mN)[2],
                    C (&aP)[NR][2], C (&aC)[NR][2], C (&aN)[NR][2], C (&sP)[NR][2], C (&sC)[NR][2], int j) {
      const int pl = zc0 - 1 + j;
      const bool do_prev = (pl - 1 >= zc0);
      const bool do_next = (pl + 1 < zc1);
      const uint32_t oplane = (uint32_t)(pl * plane);   // storage plane pl = local output plane pl-1
      // epilogue operand r̂0 of the outputs finalised here (plane pl-1), loaded before the wait
      C e1[NR][2];
#pragma unroll
      for (int r = 0; r < NR; r++)
#pragma unroll
        for (int q = 0; q < 2; q++) {
          e1[r][q] = z2;
          if (K > 0 && act[r] && do_prev && in_[q]) e1[r][q] = __ldg(rh0 + ((uint32_t)r * fs + orow + oplane + (uint32_t)q));
        }
      int n_st = c_st + 1;
      uint32_t n_ph = c_ph;
      if (n_st == S) {
        n_st = 0;
        n_ph ^= 1u;
      }
      // plane j was waited for as "next" by iteration j-1 — except the item's first plane and its last
      // (iteration nplanes-2 has no next coefficients to build); a stage is never re-armed before the
      // phase its consumers read has completed
      if (j == 0 || j == nplanes - 1) wait_stage(c_st, c_ph);
      if (do_next) wait_stage(n_st, n_ph);

      const unsigned char* st = ring + (size_t)c_st * stB;
      const float* sw = reinterpret_cast<const float*>(st) + sbw;
      const int zg = p.z0 + pl;
      bool zp_prev = false, zp_cur = false, zp_next = false, zcorr = false;
      if (PZ) {
        zp_prev = do_prev && (zg - 1 < zlo || zg - 1 > zhi);
        zp_cur = (pl >= zc0 && pl < zc1) && (zg < zlo || zg > zhi);
        zp_next = do_next && (zg + 1 < zlo || zg + 1 > zhi);
        zcorr = zp_prev || zp_cur || zp_next;
      }
      // ---- coefficients of the output points of plane pl+1 (w from the next stage) into the free slot
      {
        const float* swn = reinterpret_cast<const float*>(ring + (size_t)n_st * stB) + sbw + bxw;
#pragma unroll
        for (int e = 0; e < 2; e++) {
          const R wn = do_next ? swn[1 + e] : R(1);
          if (GAM) {   // GAm: the row's 27-node mean weights (A19), prefetched one plane ahead
            if (do_next) {
              const R t1 = gpf[e][0], t2 = gpf[e][1], mu0 = gpf[e][2], mu1 = gpf[e][3], mu2 = gpf[e][4];
              const R t0 = R(1) - R(4) * (t1 + t2);
              cN[e].c1 = p.ih2 * (t0 - R(4) * t1);
              cN[e].c2 = p.ih2 * (R(2) * (t1 - t2));
              cN[e].c3 = p.ih2 * (R(3) * t2);
              cN[e].m1 = w2 * mu1;
              cN[e].m2 = w2 * mu2;
              cN[e].m3 = w2 * ((R(1) - mu0 - R(6) * mu1 - R(12) * mu2) * R(0.125));
            } else {
              cN[e] = Coef6<R>{R(0), R(0), R(0), R(0), R(0), R(0)};
            }
          } else {
            // a2 + a3: G = 1/(√w f h) → clamped table index → linear interpolation (A13); the staged
            // rows [tab_lo, tab_lo + tab_n) cover every G of the model; packed FMAs on coefficient pairs
            const R vv = rsqrt_r(fmax(wn, R(1e-30)));
            R sidx = fma(vv, s_k1, s_k0);
            sidx = fmin(fmax(sidx, R(0)), s_max);
            const int ii = min((int)sidx, ig_max);
            const R tau = sidx - (R)ii;
            // staged row index; points outside the model's G range (pad columns, the w = 1 stand-in past
            // the chunk) read an in-range row: one unsigned min keeps every index inside the staging
            const int li = (int)min((unsigned)(ii - tab_lo), (unsigned)tab_n2);
            const R* row = stab + li * SP;
            const float4 ta = lds4<R>(row), tb = lds4<R>(row + 4), td = lds4<R>(row + 8);
            const float2 tt = make_float2(tau, tau);
            const float2 c12 = pk_fma(tt, make_float2(tb.z, tb.w), make_float2(ta.x, ta.y));
            const float2 c3m1 = pk_fma(tt, make_float2(td.x, td.y), make_float2(ta.z, ta.w));
            const float2 m23 = pk_fma(tt, make_float2(td.z, td.w), make_float2(tb.x, tb.y));
            cN[e] = Coef6<R>{c12.x, c12.y, c3m1.x, c3m1.y, m23.x, m23.y};
          }
          if (COLLOC) {
            cN[e].m1 *= wn;
            cN[e].m2 *= wn;
            cN[e].m3 *= wn;
          }
          mN[e] = COLLOC ? wn : R(1);
        }
        if (GAM && pl + 2 < zc1) gam_load(pl + 3);   // the next call's rows
      }
      C dzp = z2, dzc = z2, dzn = z2;
      if (PZ && zcorr) {
        if (zp_prev) dzp = p.dp[2][zg - 1];
        if (zp_cur) {
          const C dz = cadd(p.dm[2][zg], p.dp[2][zg]);
          dzc = make_cx(-dz.x, -dz.y);
        }
        if (zp_next) dzn = p.dm[2][zg + 1];
      }

      // ---- per RHS: in-plane class sums of the two points, accumulated halo row by halo row:
      // P0 = u0, P1 = 4 faces (x-neighbours in the centre row + centre column of the rows below /
      // above), P2 = 4 corners, Q0..Q2 of q = u·w (Eq. 8).  Rows in the order below, centre, above; the
      // x/y-PML body takes the centre row first so that the stretched parts ΔL1 = δx(u) + δy(u),
      // ΔL2 = δx(Y) + δy(X) (A8) accumulate from each row directly (a tile is always computed by the
      // same body, so each point's operation sequence is fixed).
      float Wall[3][4];   // w of the three halo rows (loaded once per plane for NR = 2)
      auto load_w = [&](int k, float (&Wr)[4]) {
        const float2 wa = *reinterpret_cast<const float2*>(sw + k * bxw);
        const float2 wb = *reinterpret_cast<const float2*>(sw + k * bxw + 2);
        Wr[0] = wa.x;
        Wr[1] = wa.y;
        Wr[2] = wb.x;
        Wr[3] = wb.y;
      };
      if (!COLLOC && NR > 1) {
#pragma unroll
        for (int k = 0; k < 3; k++) load_w(k, Wall[k]);
      }
      // the x/y-PML body handles its two points one after the other (rows read twice): the stretched
      // parts' state then fits the register budget
      constexpr int EP = PXY ? 1 : 2;
#pragma unroll
      for (int r = 0; r < NR; r++) {
        if (!act[r]) continue;
        const C* su0 = reinterpret_cast<const C*>(st + wB + (size_t)r * uB) + sbu;
        C outv[2];
#pragma unroll
        for (int eb = 0; eb < 2; eb += EP) {
        C u0[2], P1[2], P2[2], Q0[2], Q1[2], Q2[2], L1[2], L2[2], Xc[2];
        C dmx = z2, dpx = z2, dmy = z2, dpy = z2;   // this point's δ∓ (x) and the row's δ∓ (y), read once a plane
        if (PXY && gen_x) {
          dmx = __ldg(p.dm[0] + (eb ? xe1 : xe0));
          dpx = __ldg(p.dp[0] + (eb ? xe1 : xe0));
        }
        if (PXY && gen_y) {
          dmy = __ldg(p.dm[1] + ye);
          dpy = __ldg(p.dp[1] + ye);
        }
#pragma unroll
        for (int kk = 0; kk < 3; kk++) {
          const int k = PXY ? (kk == 0 ? 1 : (kk == 1 ? 0 : 2)) : kk;   // halo row: 0 below, 1 centre, 2 above
          const bool first = kk == 0;
          float Wr[4];
          if (!COLLOC) {
            if (NR > 1) {
#pragma unroll
              for (int m = 0; m < 4; m++) Wr[m] = Wall[k][m];
            } else {
              load_w(k, Wr);
            }
          }
          const C* su = su0 + k * bxu;
          const float4 A4 = *reinterpret_cast<const float4*>(su);
          const float4 B4 = *reinterpret_cast<const float4*>(su + 2);
          const C U[4] = {make_float2(A4.x, A4.y), make_float2(A4.z, A4.w), make_float2(B4.x, B4.y), make_float2(B4.z, B4.w)};
          C q[4];
          if (!COLLOC) {
#pragma unroll
            for (int m = 0; m < 4; m++) q[m] = cscale(Wr[m], U[m]);
          }
#pragma unroll
          for (int e = eb; e < eb + EP; e++) {
            const C X = cadd(U[e], U[e + 2]);
            const C Xq = COLLOC ? z2 : cadd(q[e], q[e + 2]);
            if (k == 1) {   // centre row: the centre, 2 faces (x-neighbours)
              u0[e] = U[e + 1];
              P1[e] = first ? X : cadd(P1[e], X);
              if (!COLLOC) {
                Q0[e] = q[e + 1];
                Q1[e] = first ? Xq : cadd(Q1[e], Xq);
              }
              if (PXY && gen_col) {
                Xc[e] = X;
                L1[e] = z2;
                L2[e] = z2;
                if (gen_x) {   // δx(u)
                  L1[e] = zfma_c(dmx, zneg_sw(dmx), csub(U[e], U[e + 1]), L1[e]);
                  L1[e] = zfma_c(dpx, zneg_sw(dpx), csub(U[e + 2], U[e + 1]), L1[e]);
                }
              }
            } else {   // row below / above: a face (centre column), 2 corners (x-neighbours)
              P1[e] = first ? U[e + 1] : cadd(P1[e], U[e + 1]);
              P2[e] = k == 0 ? X : cadd(P2[e], X);   // row below: the first side row in both orders
              if (!COLLOC) {
                Q1[e] = first ? q[e + 1] : cadd(Q1[e], q[e + 1]);
                Q2[e] = k == 0 ? Xq : cadd(Q2[e], Xq);
              }
              if (PXY && gen_col) {
                if (gen_x) {   // δx(Y): this row's part
                  L2[e] = zfma_c(dmx, zneg_sw(dmx), csub(U[e], U[e + 1]), L2[e]);
                  L2[e] = zfma_c(dpx, zneg_sw(dpx), csub(U[e + 2], U[e + 1]), L2[e]);
                }
                if (gen_y) {   // δy(u), δy(X): this row's part
                  const C d = k == 0 ? dmy : dpy;
                  L1[e] = zfma_c(d, zneg_sw(d), csub(U[e + 1], u0[e]), L1[e]);
                  L2[e] = zfma_c(d, zneg_sw(d), csub(X, Xc[e]), L2[e]);
                }
              }
            }
          }
        }

#pragma unroll
        for (int e = eb; e < eb + EP; e++) {
          const C c0u = u0[e];
          const C p1 = P1[e], p2 = P2[e];
          const C q0 = COLLOC ? c0u : Q0[e];
          const C q1 = COLLOC ? p1 : Q1[e];
          const C q2 = COLLOC ? p2 : Q2[e];
          const Coef6<R>& cp = cP[e];
          const Coef6<R>& cc = cC[e];
          const Coef6<R>& cn = cN[e];
          C a = aP[r][e];
          a = cfma(cp.c1, c0u, a);
          a = cfma(cp.c2, p1, a);
          a = cfma(cp.c3, p2, a);
          a = cfma(cp.m1, q0, a);
          a = cfma(cp.m2, q1, a);
          a = cfma(cp.m3, q2, a);
          C b = aC[r][e];
          b = cfma(c0_of(cc), c0u, b);
          b = cfma(cc.c1, p1, b);
          b = cfma(cc.c2, p2, b);
          b = cfma(m0_of(cc, mC[e]), q0, b);
          b = cfma(cc.m1, q1, b);
          b = cfma(cc.m2, q2, b);
          C c = cscale(cn.c1, c0u);
          c = cfma(cn.c2, p1, c);
          c = cfma(cn.c3, p2, c);
          c = cfma(cn.m1, q0, c);
          c = cfma(cn.m2, q1, c);
          c = cfma(cn.m3, q2, c);
          if (PML && ((PXY && gen_col) || zcorr)) {
            // PML transverse weights of the three output rows (t2 = c3 h²/3, t1 = t2 + c2 h²/2, t0 = c1 h² + 4 t1)
            const R pt2 = cp.c3 * i3h, pt1 = fma(cp.c2, i2h, pt2);
            const R ct2 = cc.c3 * i3h, ct1 = fma(cc.c2, i2h, ct2), ct0 = fma(cc.c1, i1h, R(4) * ct1);
            const R nt2 = cn.c3 * i3h, nt1 = fma(cn.c2, i2h, nt2);
            if (PXY && gen_col) {   // t1 ΔL1 + t2 ΔL2 (planes ±1), t0 ΔL1 + t1 ΔL2 (own plane)
              a = cfma(pt1, L1[e], a);
              a = cfma(pt2, L2[e], a);
              b = cfma(ct0, L1[e], b);
              b = cfma(ct1, L2[e], b);
              c = cfma(nt1, L1[e], c);
              c = cfma(nt2, L2[e], c);
            }
            if (PZ && zcorr) {   // δz · (t0 P0 + t1 P1 + t2 P2) of each output plane
              if (zp_prev) {
                C B3 = cscale(fma(cp.c1, i1h, R(4) * pt1), c0u);
                B3 = cfma(pt1, p1, B3);
                B3 = cfma(pt2, p2, B3);
                a = zfma_c(dzp, zneg_sw(dzp), B3, a);
              }
              if (zp_cur) {
                C B3 = cscale(ct0, c0u);
                B3 = cfma(ct1, p1, B3);
                B3 = cfma(ct2, p2, B3);
                b = zfma_c(dzc, zneg_sw(dzc), B3, b);
              }
              if (zp_next) {
                C B3 = cscale(fma(cn.c1, i1h, R(4) * nt1), c0u);
                B3 = cfma(nt1, p1, B3);
                B3 = cfma(nt2, p2, B3);
                c = zfma_c(dzn, zneg_sw(dzn), B3, c);
              }
            }
          }
          aC[r][e] = b;   // output pl: "prev" of the next call
          aN[r][e] = c;   // output pl+1: "cur" of the next call (a's slot is free after this call)
          outv[e] = in_[e] ? a : z2;
          if (EPI == EPI_DOT4) sC[r][e] = u0[e];   // s of output pl: "prev" s of the next call
        }
        }
        // ---- outputs of plane pl-1 (predicated 8-byte stores; measured faster than pairing them into
        // aligned 16-byte stores through a shuffle), then the dot epilogue
        {
          float2* o = au0 + ((uint32_t)r * fs + orow + oplane);
          st_pred(o, outv[0], do_prev && sto[0]);
          st_pred(o + 1, outv[1], do_prev && sto[1]);
        }
        if (EPI != EPI_PLAIN) {
          // the pair's products in fp32 (the same operations whichever tile / chunk / slab computes the
          // pair), accumulated per thread in fp64: the dot products then depend on the decomposition
          // only at the 1e-16 level
          float pp[KK];
#pragma unroll
          for (int k = 0; k < KK; k++) pp[k] = 0.f;
#pragma unroll
          for (int e = 0; e < 2; e++) {
            const C a = do_prev ? outv[e] : z2;
            const C rh = e1[r][e];
            if (EPI == EPI_DOT1) {
              tm_cdot(pp[0], pp[1], rh, a);
            } else if (EPI == EPI_DOT4) {
              const C sv = (do_prev && in_[e]) ? sP[r][e] : z2;
              tm_cdot(pp[0], pp[1], a, sv);
              tm_norm(pp[2], a);
              tm_cdot(pp[3], pp[4], rh, sv);
              tm_cdot(pp[5], pp[6], rh, a);
            }
          }
#pragma unroll
          for (int k = 0; k < KK; k++) part[r][k] += (double)pp[k];
        }
      }
      // ---- release this plane's stage: the producer warp waits for every warp, then refills it
      if (warp == PWARP) {
        bar_sync_n(1 + c_st);
        if (lane == 0) issue_next();
      } else {
        bar_arrive_n(1 + c_st);
      }
      c_st = n_st;
      c_ph = n_ph;
    };

    Coef6<R> cs0[2], cs1[2], cs2[2];
    R ms0[2], ms1[2], ms2[2];
    C as0[NR][2], as1[NR][2], as2[NR][2], ss0[NR][2], ss1[NR][2], ss2[NR][2];
#pragma unroll
    for (int e = 0; e < 2; e++) {
      cs0[e] = cs1[e] = cs2[e] = Coef6<R>{0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      ms0[e] = ms1[e] = ms2[e] = 0.f;
#pragma unroll
      for (int r = 0; r < NR; r++) as0[r][e] = as1[r][e] = as2[r][e] = ss0[r][e] = ss1[r][e] = ss2[r][e] = z2;
    }
    // roles (prev, cur, next) = (0,1,2), (1,2,0), (2,0,1); the s slots (prev, cur) rotate likewise
    for (int j = 0; j < nplanes; j += 3) {
      body(cs0, cs1, cs2, ms0, ms1, ms2, as0, as1, as2, ss0, ss1, j);
      if (j + 1 >= nplanes) break;
      body(cs1, cs2, cs0, ms1, ms2, ms0, as1, as2, as0, ss1, ss2, j + 1);
      if (j + 2 >= nplanes) break;
      body(cs2, cs0, cs1, ms2, ms0, ms1, as2, as0, as1, ss2, ss0, j + 2);
    }
  };

  (void)ty;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const int4 item = p.tm_work[it];
    // the body is chosen per WARP: in a tile touching the x/y-PML only the warps holding x- or y-PML
    // points run the x/y-PML body (a point is always computed by the same warp of the same tile, so its
    // operation sequence stays fixed); the others run the z-PML or the PML-free body
    bool xyw = false;
    if (item.z & TM_PMLXY) {
      const int X0 = item.x & 0xffff, Y0 = item.x >> 16;
      const int x = X0 - 1 + 2 * c_, y = Y0 + rg;
      bool xp = false;
#pragma unroll
      for (int e = 0; e < 2; e++) xp = xp || (x + e >= 0 && x + e < nx && (x + e < p.lo[0] || x + e > p.hi[0]));
      const bool yp = y < ny && (y < p.lo[1] || y > p.hi[1]);
      xyw = __any_sync(FULL, (xp || yp) && y < ny);
    }
    const bool zm = (item.z & TM_PMLZ) != 0;
    if (xyw) {   // (one x/y body handles its chunk's z-PML planes too: a fourth body costs spills)
      run_item(std::integral_constant<int, TM_PMLXY | TM_PMLZ>(), item);
    } else if (zm) {
      run_item(std::integral_constant<int, TM_PMLZ>(), item);
    } else {
      run_item(std::integral_constant<int, TM_LEAN>(), item);
    }
  }

  if constexpr (K > 0) tm_reduce<NR, K, TM_NTHR>(part, act, p, rhs0, blockIdx.x);
}

}  // namespace hz
