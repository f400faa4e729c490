// Visco-acoustic, variable-density impedance apply (NEXT-2; Eqs. 1.1-1.4 and 2; DESIGN.md
// readings A24, A25):
//
//   (Au)_n = ω² Σ_d μ_{|d|}(w_n) κ⁻¹_{n+d} u_{n+d}                                  (Eq. 8, κ complex)
//          + Σ_a Σ_{p,q} T(p,q; w_n) [β⁺ a⁺_a (u_{+} − u_{0}) + β⁻ a⁻_a (u_{−} − u_{0})]_{line (p,q)}
//   β± = ½(b±(n) + b±(n + d⊥)),  b±(m) = ½(b_m + b_{m ± e_a})         (staggered-midpoint buoyancy)
//   κ⁻¹ = b / (v² (1 − i/(2Q))²)                                      (complex velocity, A24)
//
// b breaks the transverse symmetry the class-sum kernels rely on (apply27_tm / apply27), so this path
// builds the row's 27 complex coefficients in registers — row weights from the table (or the GAm
// field), the per-axis PML a± of the row, b and κ⁻¹ of the 27 nodes — and applies them to every RHS
// of the launch.  One thread per output point, 256-thread CTAs of 32 × 8 points, one z-plane per
// grid z-index; neighbours come through L1 / L2 (each u value is read by 27 threads of ≤ 3 CTAs).
// It is a correctness-first gather kernel, not a roofline kernel.  Epilogues (the
// solver's dots) are the register path's: fp64 per-thread products, deterministic block + grid
// reduction.
#include <cuda_runtime.h>

#include "kernels.h"

namespace hz {

namespace {

constexpr int MED_NT = 256;   // 32 × 8 points

template <typename C, typename R>
__device__ __forceinline__ C rcm(R s, C a, C acc) {   // acc + s·a (s real)
  acc.x = fma(s, a.x, acc.x);
  acc.y = fma(s, a.y, acc.y);
  return acc;
}
template <typename C>
__device__ __forceinline__ C ccm(C a, C b, C acc) {   // acc + a·b (complex)
  acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
  return acc;
}

template <typename R, typename S, int EPI, bool COLLOC>
__global__ void __launch_bounds__(MED_NT) apply_medium_kernel(const ApplyParams<R, S> p, const S* __restrict__ bmed,
                                                              const typename Cx<S>::T* __restrict__ kinv, int nrhs) {
  typedef typename Cx<R>::T C;
  constexpr int K = epi_k(EPI);
  const int x = blockIdx.x * 32 + (threadIdx.x & 31);
  const int y = blockIdx.y * (MED_NT / 32) + (threadIdx.x >> 5);
  const int kz = blockIdx.z;                   // local output plane; storage plane kz + 1
  const int zg = p.z0 + kz;
  const bool sto = x < p.ldx && y < p.ny;     // stored (pad columns get zeros for complex64 storage)
  const bool in_ = x < p.nx && y < p.ny;      // computed
  const long long row = (long long)(kz + 1) * p.plane + (long long)(in_ ? y : 0) * p.ldx + (in_ ? x : 0);
  const C z2 = {R(0), R(0)};

  C cf[27];   // coefficient of node n + d, d = (dz, dy, dx) ↦ (dz+1)·9 + (dy+1)·3 + (dx+1)
#pragma unroll
  for (int d = 0; d < 27; d++) cf[d] = z2;
  // node offsets (storage elements) and in-grid flags of the 27 nodes; b / κ⁻¹ at clamped nodes
  bool ok[27];
  long long off[27];
  if (in_) {
    R t1, t2, mu0, mu1, mu2;
    if (p.gam != nullptr) {   // GAm / recorded row weights (t1, t2, μ0, μ1, μ2), stride fstride
      t1 = (R)p.gam[row];
      t2 = (R)p.gam[p.fstride + row];
      mu0 = (R)p.gam[2 * p.fstride + row];
      mu1 = (R)p.gam[3 * p.fstride + row];
      mu2 = (R)p.gam[4 * p.fstride + row];
    } else {                  // GA: the row's G = v/(f h), clamped lookup + interpolation (A13)
      interp_weights<R>((R)p.v[row], p.tab, p.n_g, p.g_min, p.g_max, p.inv_dg, p.inv_fh, t1, t2, mu0, mu1, mu2);
    }
    const R t0 = R(1) - R(4) * (t1 + t2);
    const R mu3 = (R(1) - mu0 - R(6) * mu1 - R(12) * mu2) * R(0.125);
    const R mu[4] = {mu0, mu1, mu2, mu3};
    const R T[3] = {t0, t1, t2};
    // PML: a± = h⁻² + δ± of the row along each axis (A8)
    const C dmx = p.dm[0][x], dpx = p.dp[0][x], dmy = p.dm[1][y], dpy = p.dp[1][y];
    const C dmz = p.dm[2][zg], dpz = p.dp[2][zg];
    const C am[3] = {{p.ih2 + dmx.x, dmx.y}, {p.ih2 + dmy.x, dmy.y}, {p.ih2 + dmz.x, dmz.y}};
    const C ap[3] = {{p.ih2 + dpx.x, dpx.y}, {p.ih2 + dpy.x, dpy.y}, {p.ih2 + dpz.x, dpz.y}};
    R bb[27];
#pragma unroll
    for (int dz = -1; dz <= 1; dz++)
#pragma unroll
      for (int dy = -1; dy <= 1; dy++)
#pragma unroll
        for (int dx = -1; dx <= 1; dx++) {
          const int d = (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1);
          const int xx = x + dx, yy = y + dy, zz = zg + dz;
          ok[d] = xx >= 0 && xx < p.nx && yy >= 0 && yy < p.ny && zz >= 0 && zz < p.nzg;
          off[d] = (long long)dz * p.plane + (long long)dy * p.ldx + dx;
          // clamped node (a row inside the grid clamps an outside neighbour onto its own line)
          const int xc = min(max(xx, 0), p.nx - 1), yc = min(max(yy, 0), p.ny - 1);
          const int zc = (zz >= 0 && zz < p.nzg) ? kz + 1 + dz : kz + 1;
          const long long e = (long long)zc * p.plane + (long long)yc * p.ldx + xc;
          bb[d] = (R)__ldg(bmed + e);
          // mass (Eq. 8): ω² μ_{|d|} κ⁻¹ of the node; the collocation mass (Eq. "10") takes the row's
          const C k = to_cx(ldg_c(kinv + (COLLOC ? row : e)), R(0));
          const R m = p.w2 * mu[(dz != 0) + (dy != 0) + (dx != 0)];
          cf[d] = C{m * k.x, m * k.y};
        }
    // b-weighted per-axis second differences on the 9 lines of each axis (A25)
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
      for (int pp = -1; pp <= 1; pp++)
#pragma unroll
        for (int qq = -1; qq <= 1; qq++) {
          // node index of (line offset s ∈ {−1, 0, 1} along axis a) on the line (pp, qq) ⊥ a
          auto nd = [&](int s, int lp, int lq) {
            int dx, dy, dz;
            if (a == 0) { dx = s; dy = lp; dz = lq; }
            else if (a == 1) { dy = s; dx = lp; dz = lq; }
            else { dz = s; dx = lp; dy = lq; }
            return (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1);
          };
          const R Tw = T[(pp != 0) + (qq != 0)];
          const R bp_row = R(0.5) * (bb[nd(0, 0, 0)] + bb[nd(1, 0, 0)]);
          const R bm_row = R(0.5) * (bb[nd(0, 0, 0)] + bb[nd(-1, 0, 0)]);
          const R bp_line = R(0.5) * (bb[nd(0, pp, qq)] + bb[nd(1, pp, qq)]);
          const R bm_line = R(0.5) * (bb[nd(0, pp, qq)] + bb[nd(-1, pp, qq)]);
          const R betap = Tw * (R(0.5) * (bp_row + bp_line));
          const R betam = Tw * (R(0.5) * (bm_row + bm_line));
          const int np = nd(1, pp, qq), nm = nd(-1, pp, qq), n0 = nd(0, pp, qq);
          cf[np] = rcm(betap, ap[a], cf[np]);
          cf[nm] = rcm(betam, am[a], cf[nm]);
          cf[n0] = rcm(-betap, ap[a], cf[n0]);
          cf[n0] = rcm(-betam, am[a], cf[n0]);
        }
  }

  const int nblocks = gridDim.x * gridDim.y * gridDim.z;
  const int bid = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  for (int r = 0; r < nrhs; r++) {
    if (p.active != nullptr && p.active[r] == 0) continue;   // converged RHS (uniform over the grid)
    const long long rb = (long long)r * p.fstride;
    const typename Cx<S>::T* ub = p.u + rb;
    const typename Cx<S>::T* ulb = p.ulo != nullptr ? p.ulo + rb : nullptr;
    C acc = z2, s0 = z2;
    if (in_) {
#pragma unroll
      for (int d = 0; d < 27; d++)
        if (ok[d]) {
          const C uu = load_u<R, S>(ub, ulb, row + off[d]);
          if (d == 13) s0 = uu;
          acc = ccm(cf[d], uu, acc);
        }
    }
    double part[K > 0 ? K : 1];
#pragma unroll
    for (int k = 0; k < (K > 0 ? K : 1); k++) part[k] = 0.0;
    C outv = acc;
    if (in_) {
      if (EPI == EPI_RESID) {
        const C bv = to_cx(ldg_c(p.bvec + rb + row), R(0));
        outv = csub(bv, acc);
        part[0] += (double)outv.x * (double)outv.x + (double)outv.y * (double)outv.y;
        if (p.rhat != nullptr) acc_cdot(part[1], part[2], to_cx(ldg_c(p.rhat + rb + row), R(0)), outv);
      } else if (EPI == EPI_DOT1) {
        acc_cdot(part[0], part[1], to_cx(ldg_c(p.rhat + rb + row), R(0)), acc);
      } else if (EPI == EPI_DOT4) {
        const C rh = to_cx(ldg_c(p.rhat + rb + row), R(0));
        acc_cdot(part[0], part[1], acc, s0);
        part[2] += (double)acc.x * (double)acc.x + (double)acc.y * (double)acc.y;
        acc_cdot(part[3], part[4], rh, s0);
        acc_cdot(part[5], part[6], rh, acc);
      }
      p.au[rb + row] = from_cx(outv, S(0));
    } else if (sto && sizeof(S) == 4) {
      p.au[rb + (long long)(kz + 1) * p.plane + (long long)y * p.ldx + x] = from_cx(z2, S(0));
    }
    if constexpr (K > 0)
      block_grid_reduce<K, MED_NT>(part, p.partials + (long long)r * nblocks * K, p.dots + (long long)r * K,
                                   p.tickets + r, nblocks, bid);
  }
}

// κ⁻¹ = b / (v² (1 − i/(2Q))²) at every storage element (0 where v = 0: pads, planes outside the grid)
template <typename S>
__global__ void medium_kinv_kernel(const S* __restrict__ v, const S* __restrict__ b, const S* __restrict__ q,
                                   typename Cx<S>::T* __restrict__ out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double vv = (double)v[i];
    typename Cx<S>::T o;
    o.x = S(0);
    o.y = S(0);
    if (vv > 0.0) {
      const double bv = (double)b[i];
      const double iq = q != nullptr ? 1.0 / (double)q[i] : 0.0;   // 1/Q (Q = ∞ → 0)
      const double re = 1.0 - 0.25 * iq * iq, im = -iq;            // (1 − i/(2Q))²
      const double den = re * re + im * im;
      const double s = bv / (vv * vv);
      o.x = (S)(s * re / den);
      o.y = (S)(-s * im / den);
    }
    out[i] = o;
  }
}

// domain check of b (> 0, finite) and Q (> 0; +∞ allowed) over the owned elements x < nx
template <typename S>
__global__ void medium_check_kernel(const S* __restrict__ b, const S* __restrict__ q, long long n, int nx, int ldx,
                                    unsigned long long* bad) {
  unsigned long long c = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    if ((int)(i % ldx) >= nx) continue;
    const double bv = (double)b[i];
    if (!(bv > 0.0) || !isfinite(bv)) c++;
    if (q != nullptr) {
      const double qv = (double)q[i];
      if (!(qv > 0.0)) c++;   // NaN or ≤ 0
    }
  }
  if (c) atomicAdd(bad, c);
}

template <typename S>
__global__ void medium_fill_kernel(S* __restrict__ out, long long n, S val) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = val;
}

}  // namespace

template <typename S>
cudaError_t launch_medium_fill(S* out, long long n, S val, cudaStream_t s) {
  medium_fill_kernel<S><<<592, 256, 0, s>>>(out, n, val);
  return cudaGetLastError();
}
template cudaError_t launch_medium_fill<float>(float*, long long, float, cudaStream_t);
template cudaError_t launch_medium_fill<double>(double*, long long, double, cudaStream_t);

template <typename R, typename S>
long long launch_apply_medium(const ApplyParams<R, S>& p, const S* bmed, const typename Cx<S>::T* kinv, int nrhs,
                              bool colloc, int epi, cudaStream_t s, cudaError_t* err) {
  const dim3 grid((p.ldx + 31) / 32, (p.ny + MED_NT / 32 - 1) / (MED_NT / 32), p.nzl);
  const long long nb = (long long)grid.x * grid.y * grid.z;
  if (err == nullptr) return nb;   // geometry query: partial slots per RHS
#define HZ_MED(E, CO) apply_medium_kernel<R, S, E, CO><<<grid, MED_NT, 0, s>>>(p, bmed, kinv, nrhs)
  if (colloc) {
    switch (epi) {
      case EPI_PLAIN: HZ_MED(EPI_PLAIN, true); break;
      case EPI_DOT1: HZ_MED(EPI_DOT1, true); break;
      case EPI_DOT4: HZ_MED(EPI_DOT4, true); break;
      default: HZ_MED(EPI_RESID, true); break;
    }
  } else {
    switch (epi) {
      case EPI_PLAIN: HZ_MED(EPI_PLAIN, false); break;
      case EPI_DOT1: HZ_MED(EPI_DOT1, false); break;
      case EPI_DOT4: HZ_MED(EPI_DOT4, false); break;
      default: HZ_MED(EPI_RESID, false); break;
    }
  }
#undef HZ_MED
  *err = cudaGetLastError();
  return nb;
}

template long long launch_apply_medium<float, float>(const ApplyParams<float, float>&, const float*, const float2*, int,
                                                     bool, int, cudaStream_t, cudaError_t*);
template long long launch_apply_medium<double, double>(const ApplyParams<double, double>&, const double*,
                                                       const double2*, int, bool, int, cudaStream_t, cudaError_t*);
template long long launch_apply_medium<double, float>(const ApplyParams<double, float>&, const float*, const float2*,
                                                      int, bool, int, cudaStream_t, cudaError_t*);

template <typename S>
cudaError_t launch_medium_kinv(const S* v, const S* b, const S* q, typename Cx<S>::T* out, long long n, cudaStream_t s) {
  medium_kinv_kernel<S><<<592, 256, 0, s>>>(v, b, q, out, n);
  return cudaGetLastError();
}
template cudaError_t launch_medium_kinv<float>(const float*, const float*, const float*, float2*, long long, cudaStream_t);
template cudaError_t launch_medium_kinv<double>(const double*, const double*, const double*, double2*, long long,
                                                cudaStream_t);

template <typename S>
cudaError_t launch_medium_check(const S* b, const S* q, long long n, int nx, int ldx, unsigned long long* bad,
                                cudaStream_t s) {
  medium_check_kernel<S><<<592, 256, 0, s>>>(b, q, n, nx, ldx, bad);
  return cudaGetLastError();
}
template cudaError_t launch_medium_check<float>(const float*, const float*, long long, int, int, unsigned long long*,
                                                cudaStream_t);
template cudaError_t launch_medium_check<double>(const double*, const double*, long long, int, int,
                                                 unsigned long long*, cudaStream_t);

}  // namespace hz
