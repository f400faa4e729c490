// K2 interior launch, complex64: bulk-copy (TMA engine) staged plane tiles sliding in z.
//
// Same per-point arithmetic as apply27_v2 (class-sum form; coefficients from the
// staged table; identical operation order so a point's value does not depend on which launch computed
// it — the z-slab decomposition stays bitwise invariant), different data movement:
//  * A CTA owns a TX × TY = (32·WX) × (NY·WY) tile of the interior box and marches a z-chunk.  Each
//    plane's u and w tile rows (+1 halo row/column) are copied global → shared by cp.async.bulk (one
//    instruction per row, issued by lanes of warp 0; no registers, no per-element address math) into
//    a ring of STAGES planes guarded by full/empty mbarriers, so ~STAGES planes are in flight per CTA.
//  * 1-D bulk copies need 16-byte aligned sources: each row copy starts at the 16-byte boundary at or
//    before its first element and the consumers add the (warp-uniform) shift — this works for any nx,
//    where a 2-D tensor map would need an nx·8 row pitch divisible by 16.
//  * Consumers read their column and its x-neighbours from shared memory (no shuffles, no halo
//    lanes: all 32 lanes produce outputs) and scatter into the outputs of planes k−1, k, k+1.
// Interior only: every row/column/plane of the footprint is inside the grid and outside the PML.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "apply27.cuh"

namespace hz {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int NY, int WX, int WY>
struct TmaTile {
  enum {
    TX = 32 * WX,
    TY = NY * WY,
    ROWS = TY + 2,
    UP = TX + 4,       // u row pitch (complex): TX + 2 halo + ≤1 alignment shift, rounded to 16 B
    WP = TX + 8,       // w row pitch (float):   TX + 2 halo + ≤3 alignment shift, rounded to 16 B
    UBYTES = UP * 8,
    WBYTES = WP * 4,
    STAGE = ROWS * (UBYTES + WBYTES),
  };
};

#ifndef HZ_TMA_STAGES
#define HZ_TMA_STAGES 4
#endif
constexpr int TMA_STAGES = HZ_TMA_STAGES;

// dynamic smem: [table tab_n × 12 floats][STAGES × stage][2·STAGES mbarriers]
template <int NY, int WX, int WY>
__host__ __device__ constexpr size_t tma_smem_bytes(int tab_n) {
  return (((size_t)tab_n * 12 * 4 + 127) / 128) * 128 + (size_t)TMA_STAGES * TmaTile<NY, WX, WY>::STAGE +
         2 * TMA_STAGES * 8;
}

#ifndef HZ_TMA_MINB
#define HZ_TMA_MINB 2
#endif
template <int NY, int WX, int WY, bool COLLOC, int EPI>
__global__ void __launch_bounds__(32 * WX * WY, HZ_TMA_MINB) apply27_tma(ApplyParams<float, float> p) {
  typedef float R;
  typedef float2 C;
  typedef TmaTile<NY, WX, WY> T;
  constexpr int K = epi_k(EPI);
  constexpr int NW = WX * WY;
  constexpr int S = TMA_STAGES;

  // ---- block → (rhs, tile, chunk)
  const int nrhs = p.nrhs;
  const int rhs = blockIdx.x % nrhs;
  const int tile = blockIdx.x / nrhs;
  const int ntx = p.tma_ntx;                    // tiles along x of the box
  const int tiles_per_chunk = ntx * p.tma_nty;
  const int chunk = p.box_c0 + tile / tiles_per_chunk;
  const int trem = tile % tiles_per_chunk;
  // tiles are clamped inside the box (the last tile of a row/column overlaps its neighbour; the
  // outputs it shares with the neighbour are not stored twice), so every copied row/column is in the grid
  const int X0n = p.tma_x0 + (trem % ntx) * T::TX, Y0n = p.tma_y0 + (trem / ntx) * T::TY;
  const int X0 = min(X0n, p.tma_x1 - T::TX), Y0 = min(Y0n, p.tma_y1 - T::TY);
  if (p.active != nullptr && p.active[rhs] == 0) return;

  extern __shared__ __align__(1024) unsigned char smem_tma[];   // own symbol: alignment not shared with other kernels
  float* stab = reinterpret_cast<float*>(smem_tma);
  unsigned char* ring = smem_tma + (((size_t)p.tab_n * 12 * 4 + 127) / 128) * 128;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)S * T::STAGE);
  uint64_t* empty = full + S;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wx = warp % WX, wy = warp / WX;
  const int nx = p.nx;
  int zc0, zc1;
  chunk_range(p, chunk, zc0, zc1);
  const int nplanes = zc1 - zc0 + 2;            // planes zc0-1 .. zc1
  const long long plane = p.plane;
  const float2* ubase = p.u + (long long)rhs * p.fstride;
  const float* wbase = p.w;

  // producer: the 2·ROWS row copies of plane j go into slot j % S; copy c is issued by lane 0 of warp
  // c % NW (the bulk-copy instruction takes uniform operands, so spreading the copies over the warps
  // keeps any one warp from lagging behind the others)
  auto issue_copies = [&](int j) {
    const int s = j % S;
    unsigned char* st = ring + (size_t)s * T::STAGE;
    const int pl = zc0 - 1 + j;
    if (lane == 0) {
      for (int c = warp; c < 2 * T::ROWS; c += NW) {
        const int r = c < T::ROWS ? c : c - T::ROWS;
        const long long e = (long long)(pl + 1) * plane + (long long)(Y0 - 1 + r) * nx + (X0 - 1);
        if (c < T::ROWS) {
          const uintptr_t a = reinterpret_cast<uintptr_t>(ubase + e) & ~(uintptr_t)15;
          bulk_g2s(st + (size_t)r * T::UBYTES, reinterpret_cast<const void*>(a), T::UBYTES, &full[s]);
        } else {
          const uintptr_t a = reinterpret_cast<uintptr_t>(wbase + e) & ~(uintptr_t)15;
          bulk_g2s(st + (size_t)T::ROWS * T::UBYTES + (size_t)r * T::WBYTES, reinterpret_cast<const void*>(a),
                   T::WBYTES, &full[s]);
        }
      }
    }
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // stage the coefficient table (generic proxy) while the first planes stream in
  for (int e = threadIdx.x; e < p.tab_n * CTAB_STRIDE; e += 32 * NW) stab[e] = p.ctab[(long long)p.tab_lo * CTAB_STRIDE + e];
  if (threadIdx.x == 0)
    for (int j = 0; j < S && j < nplanes; j++) mbar_expect_tx(&full[j], (uint32_t)T::STAGE);
  __syncthreads();
  for (int j = 0; j < S && j < nplanes; j++) issue_copies(j);

  // ---- per-lane geometry
  const int x = X0 + 32 * wx + lane;
  const int yl0 = Y0 + NY * wy;                 // first output row of this lane
  const bool x_ok = x >= X0n;                   // x < tma_x1 by the clamp
  // alignment shift (elements) of each row's first element x = X0-1 relative to the 16-byte aligned
  // start its bulk copy used: warp-uniform, affine in the plane and row index
  //   u: ((ubase_addr/8) + e) mod 2,  w: ((wbase_addr/4) + e) mod 4,  e = (pl+1)·plane + (Y0-1+r)·nx + X0-1
  const long long e00 = (long long)(Y0 - 1) * nx + (X0 - 1);
  const int ub0 = (int)((reinterpret_cast<uintptr_t>(ubase) >> 3) & 1) + (int)(e00 & 1);
  const int wb0 = (int)((reinterpret_cast<uintptr_t>(wbase) >> 2) & 3) + (int)(e00 & 3);
  const int plane1 = (int)(plane & 1), plane3 = (int)(plane & 3);
  constexpr int SP = SmemPitch<R>::V;
  const R s_k1 = p.inv_fh * p.inv_dg, s_k0 = -p.g_min * p.inv_dg, s_max = (R)(p.n_g - 1);
  const R w2 = p.w2;
  double part[K > 0 ? K : 1];
#pragma unroll
  for (int k = 0; k < (K > 0 ? K : 1); k++) part[k] = 0.0;

  auto c0_of = [](const Coef6<R>& c) { return -fma(R(6), c.c1, fma(R(12), c.c2, R(8) * c.c3)); };
  auto m0_of = [&](const Coef6<R>& c, R m0s) { return fma(w2, m0s, -fma(R(6), c.m1, fma(R(12), c.m2, R(8) * c.m3))); };
  // per-row constants: parity (u) and residue mod 4 (w) of sr·nx, sr = NY·wy + r
  int rpar[NY + 2], rmod[NY + 2];
#pragma unroll
  for (int r = 0; r < NY + 2; r++) {
    const int sr = NY * wy + r;
    rpar[r] = (sr * nx) & 1;
    rmod[r] = (sr * nx) & 3;
  }
  const int lane_u = 32 * wx + lane;                    // element x-1 of this lane within a row
  // output pointer of this lane's first row at local plane -1 (advanced by one plane per iteration)
  const long long obase0 = (long long)rhs * p.fstride + (long long)yl0 * nx + x;

  // one plane j (local pl = zc0-1+j); slots alternate (cP ↔ cC, aP ↔ aC) between calls: no moves
  auto body = [&](Coef6<R> (&cP)[NY], Coef6<R> (&cC)[NY], R (&mP)[NY], R (&mC)[NY], C (&aP)[NY], C (&aC)[NY],
                  int j) {
    const int pl = zc0 - 1 + j;
    const int s = j % S;
    const bool do_prev = (pl - 1 >= zc0);
    const bool do_next = (pl + 1 < zc1);
    // epilogue operands of the outputs finalised in this call (plane pl-1), loaded before the wait and
    // the arithmetic so their latency is hidden
    C e1[NY], e2[NY];
#pragma unroll
    for (int i = 0; i < NY; i++) {
      e1[i] = make_float2(0.f, 0.f);
      e2[i] = make_float2(0.f, 0.f);
      if (K > 0 && do_prev && x_ok && yl0 + i >= Y0n) {
        const long long o = obase0 + (long long)pl * plane + (long long)i * nx;
        if (EPI != EPI_RESID || p.rhat != nullptr) e1[i] = ldg_c(p.rhat + o);
        if (EPI == EPI_DOT4) e2[i] = ldg_c(p.u + o);
        if (EPI == EPI_RESID) e2[i] = ldg_c(p.bvec + o);
      }
    }
    if (j + 1 < nplanes) mbar_wait(&full[(j + 1) % S], ((j + 1) / S) & 1);
    const unsigned char* st = ring + (size_t)s * T::STAGE;
    const C* su = reinterpret_cast<const C*>(st);
    const float* sw = reinterpret_cast<const float*>(st + (size_t)T::ROWS * T::UBYTES);
    const int us_p = ub0 + (pl + 1) * plane1, ws_p = wb0 + (pl + 1) * plane3;   // row-0 shifts

#ifdef HZ_TMA_NOCOMPUTE
    // data-movement ceiling experiment: consume the stage, write the centre value, no arithmetic
    {
      const C* ur = su + (NY * wy + 1) * T::UP + ((us_p + rpar[1]) & 1) + lane_u;
      const C u0 = ur[1];
      __syncwarp();
      if (j + S < nplanes && threadIdx.x == 0) mbar_expect_tx(&full[s], (uint32_t)T::STAGE);
      if (lane == 0) mbar_arrive(&empty[s]);
      if (do_prev && x_ok) p.au[obase0 + (long long)pl * plane] = u0;
      if (j + S < nplanes) {
        mbar_wait(&empty[s], (j / S) & 1);
        issue_copies(j + S);
      }
      return;
    }
#endif
    C X[NY + 2], q[NY + 2], Xq[NY + 2], U[NY + 2];
#pragma unroll
    for (int r = 0; r < NY + 2; r++) {
      const int sr = NY * wy + r;
      const C* ur = su + sr * T::UP + ((us_p + rpar[r]) & 1) + lane_u;   // element x-1
      const float* wr = sw + sr * T::WP + ((ws_p + rmod[r]) & 3) + lane_u;
      const C a = ur[0], u0 = ur[1], b = ur[2];
      U[r] = u0;
      X[r] = cadd(a, b);
      if (!COLLOC) {
        const float wa = wr[0], w0 = wr[1], wbv = wr[2];
        q[r] = cscale(w0, u0);
        Xq[r] = cfma(wbv, b, cscale(wa, a));
      }
    }
    // ---- coefficients of the output rows of plane pl+1 (w from the next stage)
    Coef6<R> cN[NY];
    R mN[NY];
    {
      const unsigned char* sn = ring + (size_t)((j + 1) % S) * T::STAGE;
      const float* swn = reinterpret_cast<const float*>(sn + (size_t)T::ROWS * T::UBYTES);
#pragma unroll
      for (int i = 0; i < NY; i++) {
        const int sr = NY * wy + 1 + i;
        const R wn = do_next ? swn[sr * T::WP + ((ws_p + plane3 + rmod[1 + i]) & 3) + lane_u + 1] : R(1);
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
    // stage s is no longer needed by this warp (the next stage stays until the next iteration); the
    // refill's byte count is registered before the slot can be released, i.e. before any of its copies
    __syncwarp();
    if (j + S < nplanes && threadIdx.x == 0) mbar_expect_tx(&full[s], (uint32_t)T::STAGE);
    if (lane == 0) mbar_arrive(&empty[s]);

    const long long ob = obase0 + (long long)pl * plane;   // output row yl0 of local plane pl-1
#pragma unroll
    for (int i = 0; i < NY; i++) {
      const C u0 = U[i + 1];
      const C Y = cadd(U[i], U[i + 2]);
      const C P1 = cadd(X[i + 1], Y);
      const C P2 = cadd(X[i], X[i + 2]);
      const C Q0 = COLLOC ? u0 : q[i + 1];
      const C Q1 = COLLOC ? P1 : cadd(Xq[i + 1], cadd(q[i], q[i + 2]));
      const C Q2 = COLLOC ? P2 : cadd(Xq[i], Xq[i + 2]);
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
      aC[i] = b;      // output pl: "prev" of the next plane (slot roles swap)
      aP[i] = c;      // output pl+1: "cur" of the next plane
      cP[i] = cN[i];  // coefficients of pl+1 take the slot of pl-1
      mP[i] = mN[i];
      if (do_prev && x_ok && yl0 + i >= Y0n) {
        const long long o = ob + (long long)i * nx;
        if (EPI == EPI_RESID) {
          const C rr = csub(e2[i], a);
          p.au[o] = rr;
          part[0] += (double)rr.x * (double)rr.x + (double)rr.y * (double)rr.y;
          if (p.rhat != nullptr) acc_cdot(part[1], part[2], e1[i], rr);
        } else {
          p.au[o] = a;
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
    // refill slot s with plane j + S once every warp has released it (each warp issues its copies)
    if (j + S < nplanes) {
      mbar_wait(&empty[s], (j / S) & 1);
      issue_copies(j + S);
    }
  };

  Coef6<R> c0s[NY], c1s[NY];
  R m0a[NY], m0b[NY];
  C a0s[NY], a1s[NY];
#pragma unroll
  for (int i = 0; i < NY; i++) {
    c0s[i] = c1s[i] = Coef6<R>{0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    m0a[i] = m0b[i] = 0.f;
    a0s[i] = a1s[i] = make_float2(0.f, 0.f);
  }
  mbar_wait(&full[0], 0);
  int j = 0;
  for (; j + 1 < nplanes; j += 2) {
    body(c0s, c1s, m0a, m0b, a0s, a1s, j);
    body(c1s, c0s, m0b, m0a, a1s, a0s, j + 1);
  }
  if (j < nplanes) body(c0s, c1s, m0a, m0b, a0s, a1s, j);

  if (K > 0) {
    const int nb_gen = p.gen_blocks;
    const int nblocks = nb_gen + p.box_nbx * (p.box_c1 - p.box_c0);
    block_grid_reduce<K, 32 * NW>(part, p.partials + (long long)rhs * nblocks * K, p.dots + (long long)rhs * K,
                                  p.tickets + rhs, nblocks, nb_gen + tile);
  }
}

}  // namespace hz
