// K2 for complex64 (north-star steps a2–a6): tensor-map TMA plane tiles sliding in z, class sums
// gathered in registers, a dedicated producer warp, dynamically scheduled work items.  DESIGN.md §5.
//
//   (Au)_n = ω² Σ_d μ_{|d|}(w_n) u_{n+d} / v²_{n+d}                        Eq. 8, A2, A4
//          + Σ_a Σ_e D_a(n_a, e) Σ_{p,q} T(p,q; w_n) u_{n+e ê_a+p ê_b+q ê_c}   A6 (App. A), A8
//   w_n = clamped linear interpolation of the Tikhonov weight table at G_n = v_n/(f h)  P:36, A13
//
// Design (HBM-bound: 4 + 16 bytes per point and RHS):
//  * Fields are [nrhs][nz+2][ny][ldx] with a 32-byte row pitch (ldx = nx rounded up to 4), so one
//    3-D (w) and one 4-D (u: x, y, plane, RHS) tensor map describe them.  A work item is a tile of
//    tx × ty points (tx ∈ {32, 64}) × a z-chunk × one RHS.  A persistent grid of one CTA per SM takes
//    items from a global counter; the CTA's producer warp (one lane) issues, per input plane, one TMA
//    box of w and one of u — the halo tile, columns [x0 − 2, x0 + tx) — into a ring of
//    shared-memory stages (full / empty mbarrier pair per stage).  Coordinates outside the grid are
//    zero-filled by the TMA unit: the Dirichlet boundary (A9) costs no code.
//  * Consumer thread (column pair c, row r) owns the points (x0 − 1 + 2c, x0 + 2c) of row y0 + r.
//    Per input plane it reads, for the three halo rows, the four u columns 2c .. 2c+3 (two 16-byte
//    shared loads) and the four w (two 8-byte loads) and forms the in-plane class sums P0 = u,
//    P1 = 4 faces, P2 = 4 corners of u and of q = u·w (Eq. 8).  The sums of the last three planes stay
//    in registers (three rotating slots); output plane k is gathered when plane k+1 arrives:
//    U1 = P1(k) + P0(k−1) + P0(k+1), U2 = P2(k) + P1(k±1), U3 = P2(k±1), likewise for q, then
//    Au = c0·u + c1 U1 + c2 U2 + c3 U3 + m0·q + m1 Q1 + m2 Q2 + m3 Q3 with the row's coefficients built
//    from its own w (one MUFU.RSQ, clamped linear interpolation of the table staged in shared memory);
//    c0 and m0 follow from the sum rules.  Every point is computed by the same operation sequence
//    whichever item, chunk, launch or slab computes it (bitwise z-slab invariance).
//  * PML (A8): the z corrections δ∓_z (B(k∓1) − B(k)), B = t0 P0 + t1 P1 + t2 P2, from the register
//    sums (plane-uniform branch); the x/y corrections re-read the 3 × 3 × 3 window from the three
//    stages still held (warp-uniform branch, only in warps holding x/y-PML points; a δ = 0 adds
//    exact zeros).  A stage is released when the output plane above it is done.
//  * Output: two 8-byte stores per thread; the pad columns [nx, ldx) are written as zeros.
//  * Epilogues (BiCGSTAB dots): per-point products in fp32, accumulated per thread in fp64, reduced
//    per ITEM (warp shuffles, then the consumer warps in a fixed order) into a partial slot per item;
//    the last CTA sums the slots in item order — deterministic whatever CTA ran which item.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "apply27.cuh"

namespace hz {

constexpr int TM_NCW = 11;                    // consumer warps per CTA (+ producer: 12 warps, 3 per SMSP → ≤ 168 registers)
constexpr int TM_NTHR = 32 * (TM_NCW + 1);    // + one producer warp (one CTA per SM)
constexpr int TM_MAXTX = 64;                  // widest tile
#ifndef HZ_TM_STAGES
#define HZ_TM_STAGES 10
#endif
#ifndef HZ_TM_SLEEP_NS
#define HZ_TM_SLEEP_NS 64
#endif
constexpr int TM_STAGES = HZ_TM_STAGES;       // ring depth (planes in flight per CTA)

// PML mode bits of a work item: TM_PMLZ the chunk holds z-PML output planes, TM_PMLXY the tile holds
// x/y-PML columns / rows; TM_LEAN neither
enum { TM_LEAN = 0, TM_PMLZ = 1, TM_PMLXY = 2 };

// work item {x0 | y0 << 16, z0 | z1 << 16, mode, 0}: tile origin (x0, y0), local output planes [z0, z1)
__host__ __device__ inline int4 tm_item(int x0, int y0, int z0, int z1, int mode) {
  return make_int4(x0 | (y0 << 16), z0 | (z1 << 16), mode, 0);
}

// Tile geometry shared by host and device.  A tile of tx columns with origin X0 (a multiple of tx)
// computes the points x ∈ [X0 − 1, X0 + tx − 1).  The TMA unit needs the box's innermost start
// coordinate 16-byte aligned (a misaligned start faults: tools/tma_odd), so the u box is
// [X0 − 2, X0 + tx) (tx + 2 complex columns) and the w box [X0 − 4, X0 + tx) (tx + 4 floats); a thread's
// four columns x − 1 .. x + 2 then sit at 16-byte (u) / 8-byte (w) aligned shared addresses.
// A warp covers whole tile rows (tx/2 column pairs each): the TM_NCW consumer warps TM_NCW·64/tx rows.
__host__ __device__ constexpr int tm_bxu(int tx) { return tx + 2; }
__host__ __device__ constexpr int tm_bxw(int tx) { return tx + 4; }
__host__ __device__ constexpr int tm_rows(int tx) { return TM_NCW * 64 / tx; }
__host__ __device__ constexpr uint32_t tm_r128(uint32_t b) { return (b + 127u) & ~127u; }
// bytes one box delivers (the mbarrier's transaction count) and its 128-byte aligned slot in a stage
__host__ __device__ constexpr uint32_t tm_wbox(int tx, int ty) { return (uint32_t)tm_bxw(tx) * (ty + 2) * 4u; }
__host__ __device__ constexpr uint32_t tm_ubox(int tx, int ty) { return (uint32_t)tm_bxu(tx) * (ty + 2) * 8u; }
__host__ __device__ constexpr uint32_t tm_wbytes(int tx, int ty) { return tm_r128(tm_wbox(tx, ty)); }
__host__ __device__ constexpr uint32_t tm_ubytes(int tx, int ty) { return tm_r128(tm_ubox(tx, ty)); }
// a stage: the w box, the u box, and (dot epilogues) an r̂₀ box of the u box's shape (rh)
__host__ __device__ constexpr uint32_t tm_stage_bytes(int tx, int ty, bool rh = false) {
  return tm_wbytes(tx, ty) + (rh ? 2u : 1u) * tm_ubytes(tx, ty);
}
// staged table rows: TM_TP floats apart (80 B: 8 consecutive rows start on distinct 16-byte bank groups)
constexpr int TM_TP = 20;
__host__ __device__ constexpr uint32_t tm_tab_bytes(int tab_n) { return tm_r128((uint32_t)tab_n * TM_TP * 4u); }
// shared memory: header (full / empty mbarriers, per-stage item ids, the item reduction scratch),
// the ring of stages, then the staged coefficient rows
constexpr uint32_t TM_HDR = 1024;
__host__ __device__ constexpr size_t tm_ring_end(int tx, int ty, bool rh) { return TM_HDR + (size_t)TM_STAGES * tm_stage_bytes(tx, ty, rh); }
__host__ __device__ constexpr size_t tm_smem_bytes(int tab_n, int tx, int ty, bool rh) { return tm_ring_end(tx, ty, rh) + tm_tab_bytes(tab_n); }

// ---- TMA / mbarrier / named-barrier primitives (PTX) -------------------------------------------
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// Wait for the phase with the given parity to complete.  A transfer that never completes (a
// programming error) traps after ~2^30 polls instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  for (uint32_t n = 0;; n++) {
    uint32_t done;
    asm volatile(
        "{\n .reg .pred P1;\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n selp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    if (n > (1u << 30)) __trap();
  }
}
// the producer's wait for a free stage: back off between polls (its spinning would take issue slots
// from the consumer warps of its SM sub-partition)
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
  for (uint32_t n = 0;; n++) {
    uint32_t done;
    asm volatile(
        "{\n .reg .pred P1;\n mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n selp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    if (n > (1u << 28)) __trap();
    __nanosleep(HZ_TM_SLEEP_NS);
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
// named barrier 1: the consumer warps only
__device__ __forceinline__ void bar_consumers() { asm volatile("bar.sync 1, %0;" ::"n"(32 * TM_NCW) : "memory"); }

// conj(a)·b of complex64 data in fp32
__device__ __forceinline__ void tm_cdot(float& re, float& im, float2 a, float2 b) {
  re = fmaf(a.x, b.x, fmaf(a.y, b.y, re));
  im = fmaf(a.x, b.y, fmaf(-a.y, b.x, im));
}
__device__ __forceinline__ void tm_norm(float& s, float2 a) { s = fmaf(a.x, a.x, fmaf(a.y, a.y, s)); }

// predicated 8-byte global store (branch-free)
__device__ __forceinline__ void st_pred(float2* ptr, float2 v, bool pred) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %0, 0;\n @p st.global.v2.f32 [%1], {%2, %3};\n}\n" ::"r"((int)pred),
               "l"(ptr), "f"(v.x), "f"(v.y)
               : "memory");
}

// the in-plane class sums of one input plane at a thread's two points, and their w
struct TmSlot {
  float2 u0[2], u1[2], u2[2];   // P0, P1, P2 of u
  float2 q1[2], q2[2];          // P1, P2 of q = u·w (Eq. 8; P0 = w·u0); unused for the Eq. "10" mass
  float w[2];                   // w at the points (the output's coefficients and P0 of q)
};
// ... in an x/y-PML tile, plus the stretched parts of the plane (A8): ΔL1 = δx(u) + δy(u) on the row's
// own line, ΔL2 = δx(Y) + δy(X) on the 4 transverse neighbours' lines
struct TmSlotX : TmSlot {
  float2 L1[2], L2[2];
};

// The kernel.  Work items g = item · nrhs + rhs (all RHS of a tile × chunk run back to back, so w is
// read from HBM once); the global counter p.tm_ctr[0] hands them out, p.tm_ctr[1] counts finished
// CTAs (the last one reduces the dot partials and resets both counters for the next launch).
template <int TX, bool COLLOC, int EPI, bool GAM>
__global__ void __launch_bounds__(TM_NTHR, 1)
    apply27_tm(const __grid_constant__ CUtensorMap tmw, const __grid_constant__ CUtensorMap tmu,
               const __grid_constant__ CUtensorMap tmr, ApplyParams<float, float> p) {
  typedef float R;
  typedef float2 C;
  constexpr int K = epi_k(EPI);
  constexpr int KK = K > 0 ? K : 1;
  constexpr int S = TM_STAGES;
  constexpr int tx = TX, ty = tm_rows(TX);
  constexpr int bxu = tm_bxu(TX), bxw = tm_bxw(TX);
  // dot epilogues: r̂₀ at the output plane comes through the stage too (a TMA box, not a per-thread
  // global load whose DRAM latency the 11 consumer warps cannot hide)
  constexpr bool RH = K > 0;
  constexpr uint32_t wB = tm_wbytes(TX, ty), uB = tm_ubytes(TX, ty);
  constexpr uint32_t stB = tm_stage_bytes(TX, ty, RH);
  constexpr uint32_t txB = tm_wbox(tx, ty) + (RH ? 2u : 1u) * tm_ubox(tx, ty);   // transaction bytes per plane

  const int nx = p.nx, ny = p.ny, ldx = p.ldx;
  const int plane = (int)p.plane;   // host: (nzl + 2)·plane < 2^31 (32-bit offsets within a field)
  const int nrhs = p.nrhs;
  const int total = p.tm_nitems * nrhs;

  extern __shared__ __align__(1024) unsigned char smem_tm[];
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_tm);
  const uint32_t full0 = sbase, empty0 = sbase + 8u * S;
  volatile int* meta = reinterpret_cast<volatile int*>(smem_tm + 16 * S);        // item id per stage
  // header: full[S], empty[S] mbarriers, meta[S], then the item reduction scratch [TM_NCW][KK]
  constexpr uint32_t RED_OFF = (20u * S + 7u) & ~7u;
  static_assert(RED_OFF + 8u * TM_NCW * KK <= TM_HDR, "apply27_tm: shared header overflow");
  double* red = reinterpret_cast<double*>(smem_tm + RED_OFF);
  unsigned char* ring = smem_tm + TM_HDR;
  const uint32_t ring_s = sbase + TM_HDR;
  float* stab = reinterpret_cast<float*>(smem_tm + tm_ring_end(TX, ty, RH));

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < S; s++) {
      mbar_init(full0 + 8u * s, 1u);
      mbar_init(empty0 + 8u * s, (uint32_t)TM_NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int e = tid; e < p.tab_n * TMTAB_STRIDE; e += TM_NTHR) {
    const int rw = e / TMTAB_STRIDE, k = e - rw * TMTAB_STRIDE;
    stab[rw * TM_TP + k] = p.ctm[(long long)(p.tab_lo + rw) * TMTAB_STRIDE + k];
  }
  __syncthreads();

  // ---- producer: lane 0 of the last warp
  if (warp == TM_NCW) {
    if (lane != 0) return;
    int s = 0;
    uint32_t ph = 0;
    for (;;) {
      const int g = (int)atomicAdd(p.tm_ctr, 1u);
      if (g < total) {
        const int r = g % nrhs;
        if (p.active != nullptr && p.active[r] == 0) continue;   // converged RHS: no work
        const int4 it = p.tm_work[p.tm_item0 + g / nrhs];
        const int x0 = it.x & 0xffff, y0 = it.x >> 16;
        const int c2 = (it.y & 0xffff) - p.tm_org;   // map coordinate of input plane 0 (storage plane z0)
        const int n = (it.y >> 16) - (it.y & 0xffff) + 2;
        for (int j = 0; j < n; j++) {
          mbar_wait_sleep(empty0 + 8u * s, ph ^ 1u);
          if (j == 0) meta[s] = g + p.tm_item0 * nrhs;   // list-wide id: item = g / nrhs
          const uint32_t bar = full0 + 8u * s, dst = ring_s + (uint32_t)s * stB;
          mbar_expect_tx(bar, txB);
          tma_load3(dst, &tmw, bar, x0 - 4, y0 - 1, c2 + j);
          tma_load4(dst + wB, &tmu, bar, x0 - 2, y0 - 1, c2 + j, r);
          // r̂₀ of the output plane computed when input plane j arrives (storage plane z0 + j − 1; the
          // first two input planes fetch a plane no output reads, outside the map's range for j = 0)
          if (RH) tma_load4(dst + wB + uB, &tmr, bar, x0 - 2, y0 - 1, c2 + j - 1, r);
          if (++s == S) { s = 0; ph ^= 1u; }
        }
      } else {
        mbar_wait(empty0 + 8u * s, ph ^ 1u);
        meta[s] = -1;
        mbar_arrive(full0 + 8u * s);
        break;
      }
    }
    return;
  }

  // ---- consumers: thread → points (x0 − 1 + 2c, x0 + 2c) of row y0 + rr; a warp covers whole tile rows
  // (TX/2 column pairs each), so in a tile holding x-PML columns every warp holds some
  constexpr int PR = TX / 2;
  const int cw = warp;
  const int c_ = lane % PR;
  const int rr = (32 / PR) * cw + lane / PR;
  const int sbw = rr * bxw + 2 * c_ + 2;   // stage element (row y − 1, column x − 1) in the w box
  const int sbu = rr * bxu + 2 * c_;   // ... in the u box
  const C z2 = make_float2(0.f, 0.f);
  // staged-row index of a row: (G − g_min)/ΔG − tab_lo, clamped to the staged rows (which cover every G
  // of the model and the global clamp at both table ends, api.cu)
  const R s_k1 = p.inv_fh * p.inv_dg, s_k0 = -p.g_min * p.inv_dg - (R)p.tab_lo, s_hi = (R)(p.tab_n - 1);
  const R w2 = p.w2;
  const int zlo = p.lo[2], zhi = p.hi[2];
  const R i3h = p.inv3ih2, i2h = p.inv2ih2, i1h = p.invih2;

  int s = 0;          // stage of the next plane to wait for
  uint32_t ph = 0;    // its phase parity
  int rs = 0;         // next stage to release
  // release the oldest held stage: lane 0 arrives (predicated, no branch) once the warp is done with it
  const uint32_t lead = lane == 0 ? 1u : 0u;
  auto release = [&]() {
    __syncwarp();
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %0, 0;\n @p mbarrier.arrive.shared::cta.b64 _, [%1];\n}\n" ::"r"(lead),
                 "r"(empty0 + 8u * rs)
                 : "memory");
    if (++rs == S) rs = 0;
  };

  for (;;) {
    mbar_wait(full0 + 8u * s, ph);
    const int g = meta[s];
    if (g < 0) break;
    const int r = g % nrhs;
    const int4 item = p.tm_work[g / nrhs];
    const int X0 = item.x & 0xffff, Y0 = item.x >> 16;
    const int zc0 = item.y & 0xffff, zc1 = item.y >> 16;
    const int n = zc1 - zc0 + 2;   // input planes zc0−1 .. zc1
    const bool PZ = (item.z & TM_PMLZ) != 0;
    const int x = X0 - 1 + 2 * c_, y = Y0 + rr;
    const bool yok = y < ny;
    // a point is stored if it lies in the pitched row (a pad column gets a zero), computed if in the grid
    const bool sto[2] = {yok && x >= 0 && x < ldx, yok && x + 1 < ldx};
    const bool in_[2] = {sto[0] && x < nx, sto[1] && x + 1 < nx};
    // 32-bit element offsets (wrap back for the never-stored x = −1 of row 0)
    const uint32_t orow = (uint32_t)(y * ldx + x);
    float2* __restrict__ au0 = p.au + (long long)r * p.fstride;
    double part[KK];
#pragma unroll
    for (int k = 0; k < KK; k++) part[k] = 0.0;

    auto march = [&](auto XYc) {
    constexpr bool XY = decltype(XYc)::value;
    typedef typename std::conditional<XY, TmSlotX, TmSlot>::type Slot;
    // x/y-PML tiles: the δ∓ of this thread's columns and row (zero off the PML)
    C dmx[2] = {z2, z2}, dpx[2] = {z2, z2}, dmy = z2, dpy = z2;
    if constexpr (XY) {
#pragma unroll
      for (int e = 0; e < 2; e++) {
        const int xe = min(max(x + e, 0), nx - 1);
        dmx[e] = __ldg(p.dm[0] + xe);
        dpx[e] = __ldg(p.dp[0] + xe);
      }
      const int ye = min(y, ny - 1);
      dmy = __ldg(p.dm[1] + ye);
      dpy = __ldg(p.dp[1] + ye);
    }
    // ---- in-plane class sums of the plane in stage st into slot N
    auto step = [&](Slot& N, int st) {
      const unsigned char* sp = ring + (size_t)st * stB;
      const float* sw = reinterpret_cast<const float*>(sp) + sbw;
      const C* su = reinterpret_cast<const C*>(sp + wB) + sbu;
      C cr0[2], hr0[2], cr1[2], hr1[2], xm[2], xp[2];   // x/y-PML row temporaries
#pragma unroll
      for (int k = 0; k < 3; k++) {
        const float4 A4 = *reinterpret_cast<const float4*>(su + k * bxu);
        const float4 B4 = *reinterpret_cast<const float4*>(su + k * bxu + 2);
        const C U[4] = {make_float2(A4.x, A4.y), make_float2(A4.z, A4.w), make_float2(B4.x, B4.y), make_float2(B4.z, B4.w)};
        float W[4];
        {
          const float2 wa = *reinterpret_cast<const float2*>(sw + k * bxw);
          const float2 wb = *reinterpret_cast<const float2*>(sw + k * bxw + 2);
          W[0] = wa.x; W[1] = wa.y; W[2] = wb.x; W[3] = wb.y;
        }
        C q[4];
        if (!COLLOC) {
#pragma unroll
          for (int m = 0; m < 4; m++) q[m] = cscale(W[m], U[m]);
        }
#pragma unroll
        for (int e = 0; e < 2; e++) {
          const C hu = cadd(U[e], U[e + 2]);
          if constexpr (XY) {   // the stretched parts, row by row (A8)
            if (k == 0) {
              cr0[e] = U[e + 1];
              hr0[e] = hu;
              xm[e] = csub(U[e], U[e + 1]);
              xp[e] = csub(U[e + 2], U[e + 1]);
            } else if (k == 1) {
              cr1[e] = U[e + 1];
              hr1[e] = hu;
              N.L1[e] = zfma(dmx[e], csub(U[e], U[e + 1]), z2);
              N.L1[e] = zfma(dpx[e], csub(U[e + 2], U[e + 1]), N.L1[e]);
            } else {
              xm[e] = cadd(xm[e], csub(U[e], U[e + 1]));
              xp[e] = cadd(xp[e], csub(U[e + 2], U[e + 1]));
              N.L1[e] = zfma(dmy, csub(cr0[e], cr1[e]), N.L1[e]);
              N.L1[e] = zfma(dpy, csub(U[e + 1], cr1[e]), N.L1[e]);
              N.L2[e] = zfma(dmx[e], xm[e], z2);
              N.L2[e] = zfma(dpx[e], xp[e], N.L2[e]);
              N.L2[e] = zfma(dmy, csub(hr0[e], hr1[e]), N.L2[e]);
              N.L2[e] = zfma(dpy, csub(hu, hr1[e]), N.L2[e]);
            }
          }
          const C hq = COLLOC ? z2 : cadd(q[e], q[e + 2]);
          if (k == 0) {          // row below: a face (centre column), 2 corners
            N.u1[e] = U[e + 1];
            N.u2[e] = hu;
            if (!COLLOC) { N.q1[e] = q[e + 1]; N.q2[e] = hq; }
          } else if (k == 1) {   // centre row: the centre, 2 faces
            N.u0[e] = U[e + 1];
            N.u1[e] = cadd(N.u1[e], hu);
            if (!COLLOC) N.q1[e] = cadd(N.q1[e], hq);
            N.w[e] = W[e + 1];
          } else {               // row above: a face, 2 corners
            N.u1[e] = cadd(N.u1[e], U[e + 1]);
            N.u2[e] = cadd(N.u2[e], hu);
            if (!COLLOC) { N.q1[e] = cadd(N.q1[e], q[e + 1]); N.q2[e] = cadd(N.q2[e], hq); }
          }
        }
      }
    };

    // ---- output plane ol (local) from the slots of planes ol−1 (A), ol (B), ol+1 (N); st = stage of ol+1
    auto output = [&](const Slot& A, const Slot& B, const Slot& N, int ol, int st) {
      const uint32_t oel = (uint32_t)((ol + 1) * plane) + orow;   // element in this RHS's field
      C rh[2] = {z2, z2};
      if (K > 0) {   // r̂₀ box of stage st: row rr + 1, columns 2c + 1, 2c + 2 (points x, x + 1)
        const C* sr = reinterpret_cast<const C*>(ring + (size_t)st * stB + wB + uB) + sbu + bxu + 1;
#pragma unroll
        for (int e = 0; e < 2; e++) rh[e] = in_[e] ? sr[e] : z2;
      }
      const int zg = p.z0 + ol;
      const bool zpml = PZ && (zg < zlo || zg > zhi);
      C outv[2];
#pragma unroll
      for (int e = 0; e < 2; e++) {
        // a2 + a3: the row coefficients from its own w: G = 1/(√w f h) → clamped index into the staged
        // rows → linear interpolation (A13); GAm: the row's 27-node mean weights (A19)
        const R wn = B.w[e];
        R cf[8];   // c0 c1 c2 c3 m0 m1 m2 m3
        if (GAM) {
          const uint32_t ge = oel + (uint32_t)e;
          R t1 = 0, t2 = 0, mu0 = 0, mu1 = 0, mu2 = 0;
          if (in_[e]) {
            t1 = __ldg(p.gam + ge);
            t2 = __ldg(p.gam + p.fstride + ge);
            mu0 = __ldg(p.gam + 2 * p.fstride + ge);
            mu1 = __ldg(p.gam + 3 * p.fstride + ge);
            mu2 = __ldg(p.gam + 4 * p.fstride + ge);
          }
          const R t0 = R(1) - R(4) * (t1 + t2);
          cf[1] = p.ih2 * (t0 - R(4) * t1);
          cf[2] = p.ih2 * (R(2) * (t1 - t2));
          cf[3] = p.ih2 * (R(3) * t2);
          cf[5] = w2 * mu1;
          cf[6] = w2 * mu2;
          cf[7] = w2 * ((R(1) - mu0 - R(6) * mu1 - R(12) * mu2) * R(0.125));
          cf[0] = -fma(R(6), cf[1], fma(R(12), cf[2], R(8) * cf[3]));
          cf[4] = fma(w2, R(1), -fma(R(6), cf[5], fma(R(12), cf[6], R(8) * cf[7])));
        } else {
          // w = 0 (outside the grid) gives +inf: clamped to the last staged row like any G above the range
          R sidx = fma(rsqrt_r(wn), s_k1, s_k0);
          sidx = fmin(fmax(sidx, R(0)), s_hi);
          const int ii = (int)sidx;
          const R tau = sidx - (R)ii;
          const R* row = stab + ii * TM_TP;
          const float4 a0 = lds4<R>(row), a1 = lds4<R>(row + 4), d0 = lds4<R>(row + 8), d1 = lds4<R>(row + 12);
          cf[0] = fma(tau, d0.x, a0.x);
          cf[1] = fma(tau, d0.y, a0.y);
          cf[2] = fma(tau, d0.z, a0.z);
          cf[3] = fma(tau, d0.w, a0.w);
          cf[4] = fma(tau, d1.x, a1.x);
          cf[5] = fma(tau, d1.y, a1.y);
          cf[6] = fma(tau, d1.z, a1.z);
          cf[7] = fma(tau, d1.w, a1.w);
        }
        const C U1 = cadd(B.u1[e], cadd(A.u0[e], N.u0[e]));
        const C U2 = cadd(B.u2[e], cadd(A.u1[e], N.u1[e]));
        const C U3 = cadd(A.u2[e], N.u2[e]);
        C acc;
        if (COLLOC) {   // Eq. "10": the mass takes the row's own 1/v² (q sums = u sums × w_n)
          acc = cscale(fma(cf[4], wn, cf[0]), B.u0[e]);
          acc = cfma(fma(cf[5], wn, cf[1]), U1, acc);
          acc = cfma(fma(cf[6], wn, cf[2]), U2, acc);
          acc = cfma(fma(cf[7], wn, cf[3]), U3, acc);
        } else {
          const C Q1 = cadd(B.q1[e], cfma(N.w[e], N.u0[e], cscale(A.w[e], A.u0[e])));
          const C Q2 = cadd(B.q2[e], cadd(A.q1[e], N.q1[e]));
          const C Q3 = cadd(A.q2[e], N.q2[e]);
          acc = cscale(fma(cf[4], wn, cf[0]), B.u0[e]);   // c0 u + m0 q0, q0 = w u
          acc = cfma(cf[1], U1, acc);
          acc = cfma(cf[2], U2, acc);
          acc = cfma(cf[3], U3, acc);
          acc = cfma(cf[5], Q1, acc);
          acc = cfma(cf[6], Q2, acc);
          acc = cfma(cf[7], Q3, acc);
        }
        if (zpml || XY) {
          // transverse weights of the row (t2 = c3 h²/3, t1 = t2 + c2 h²/2, t0 = c1 h² + 4 t1)
          const R t2 = cf[3] * i3h, t1 = fma(cf[2], i2h, t2), t0 = fma(cf[1], i1h, R(4) * t1);
          if (zpml) {   // δ∓_z (B(k∓1) − B(k)), B = t0 P0 + t1 P1 + t2 P2 (A8)
            C Bm = cscale(t0, A.u0[e]);
            Bm = cfma(t1, A.u1[e], Bm);
            Bm = cfma(t2, A.u2[e], Bm);
            C Bc = cscale(t0, B.u0[e]);
            Bc = cfma(t1, B.u1[e], Bc);
            Bc = cfma(t2, B.u2[e], Bc);
            C Bp = cscale(t0, N.u0[e]);
            Bp = cfma(t1, N.u1[e], Bp);
            Bp = cfma(t2, N.u2[e], Bp);
            acc = zfma(p.dm[2][zg], csub(Bm, Bc), acc);
            acc = zfma(p.dp[2][zg], csub(Bp, Bc), acc);
          }
          if constexpr (XY) {   // x/y: t0 ΔL1(k) + t1 ΔL2(k) + t1 ΔL1(k±1) + t2 ΔL2(k±1)
            acc = cfma(t0, B.L1[e], acc);
            acc = cfma(t1, B.L2[e], acc);
            acc = cfma(t1, cadd(A.L1[e], N.L1[e]), acc);
            acc = cfma(t2, cadd(A.L2[e], N.L2[e]), acc);
          }
        }
        outv[e] = acc;
      }
#pragma unroll
      for (int e = 0; e < 2; e++) outv[e] = in_[e] ? outv[e] : z2;
      st_pred(au0 + oel, outv[0], sto[0]);
      st_pred(au0 + oel + 1u, outv[1], sto[1]);
      if (EPI != EPI_PLAIN) {
        float pp[KK];
#pragma unroll
        for (int k = 0; k < KK; k++) pp[k] = 0.f;
#pragma unroll
        for (int e = 0; e < 2; e++) {
          const C a = outv[e];
          if (EPI == EPI_DOT1) {
            tm_cdot(pp[0], pp[1], rh[e], a);
          } else if (EPI == EPI_DOT4) {
            // s = the apply's input, or (right-preconditioned solve: the input is M⁻¹s) p.bvec
            const C sv = in_[e] ? (p.bvec != nullptr ? __ldg(p.bvec + oel + (uint32_t)e) : B.u0[e]) : z2;
            tm_cdot(pp[0], pp[1], a, sv);
            tm_norm(pp[2], a);
            tm_cdot(pp[3], pp[4], rh[e], sv);
            tm_cdot(pp[5], pp[6], rh[e], a);
          }
        }
#pragma unroll
        for (int k = 0; k < KK; k++) part[k] += (double)pp[k];
      }
    };

    // ---- march the planes: three slots rotate through the roles (ol−1, ol, ol+1)
    Slot S0, S1, S2;
    auto advance = [&]() {
      const int st = s;
      if (++s == S) { s = 0; ph ^= 1u; }
      return st;
    };
    step(S0, advance());   // plane 0 (waited for above)
    {
      mbar_wait(full0 + 8u * s, ph);
      step(S1, advance());
    }
    for (int j = 2;;) {
      int st;
      mbar_wait(full0 + 8u * s, ph);
      st = advance();
      step(S2, st);
      output(S0, S1, S2, zc0 + j - 2, st);
      release();
      if (++j >= n) break;
      mbar_wait(full0 + 8u * s, ph);
      st = advance();
      step(S0, st);
      output(S1, S2, S0, zc0 + j - 2, st);
      release();
      if (++j >= n) break;
      mbar_wait(full0 + 8u * s, ph);
      st = advance();
      step(S1, st);
      output(S2, S0, S1, zc0 + j - 2, st);
      release();
      if (++j >= n) break;
    }
    release();   // the item's last two planes
    release();

    };
    if (item.z & TM_PMLXY) march(std::true_type());
    else march(std::false_type());

    if constexpr (K > 0) {   // the item's partials: warps (fixed order) → slot g
#pragma unroll
      for (int k = 0; k < K; k++) {
        double v = part[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[cw * KK + k] = v;
      }
      bar_consumers();
      if (tid < K) {
        double v = 0.0;
        for (int w = 0; w < TM_NCW; w++) v += red[w * KK + tid];
        p.partials[(long long)g * K + tid] = v;
      }
      bar_consumers();
    }
  }

  // ---- CTA done: the last CTA sums the item partials in item order and resets the counters
  __shared__ bool last;
  bar_consumers();
  if (tid == 0) {
    __threadfence();
    last = atomicAdd(p.tm_ctr + 1, 1u) == gridDim.x - 1;
  }
  bar_consumers();
  if (!last) return;
  __threadfence();
  if constexpr (K > 0) {
    const int nit = p.tm_nred;
    for (int q = nit > 0 ? cw : nrhs * K; q < nrhs * K; q += TM_NCW) {
      const int rq = q / K, k = q - rq * K;
      if (p.active != nullptr && p.active[rq] == 0) continue;
      const volatile double* pp = p.partials;
      double v = 0.0;
      for (int i = lane; i < nit; i += 32) v += pp[((long long)i * nrhs + rq) * K + k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) p.dots[(long long)rq * K + k] = v;
    }
  }
  if (tid == 0) {
    p.tm_ctr[0] = 0u;
    p.tm_ctr[1] = 0u;
  }
}

}  // namespace hz
