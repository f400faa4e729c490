// sm_100a kernels of libhz: fused coefficient + 27-point apply (with optional BiCGSTAB dot
// epilogues), coefficient-record export, point sources, BiCGSTAB vector updates.
// See apply.cuh for the apply design; DESIGN.md §5 for rooflines.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <type_traits>

#include "apply.cuh"
#include "apply27.cuh"
#include "apply27_tm.cuh"
#include "kernels.h"

namespace hz {

// storage element (halo plane 0 first, row pitch ldx) of owned point idx = (zl·ny + y)·nx + x
template <typename R, typename S>
__device__ __forceinline__ long long st_elem(const ApplyParams<R, S>& p, long long idx, int& zl, int& y, int& x) {
  const long long pl = (long long)p.nx * p.ny;
  zl = (int)(idx / pl);
  const int rem = (int)(idx - (long long)zl * pl);
  y = rem / p.nx;
  x = rem - y * p.nx;
  return (long long)(zl + 1) * p.plane + (long long)y * p.ldx + x;
}

// =============================================================================================
// K1 record export: (k², t0, t1, t2, μ0, μ1, μ2, μ3) per point
// =============================================================================================
template <typename R>
__global__ void record_kernel(ApplyParams<R> p, R w2_over_1, R* __restrict__ rec) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* tab = reinterpret_cast<R*>(smem_raw);
  for (int i = threadIdx.x; i < p.n_g * TAB_STRIDE; i += blockDim.x) tab[i] = p.tab[i];
  __syncthreads();
  const long long n = (long long)p.nzl * p.ny * p.nx;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (long long)gridDim.x * blockDim.x) {
    int zl, y, x;
    const long long e = st_elem(p, idx, zl, y, x);
    const R v = p.v[e];
    R t1, t2, mu0, mu1, mu2;
    if (p.gam != nullptr) {   // GAm: the row's 27-node mean weights (A19)
      t1 = p.gam[e], t2 = p.gam[p.fstride + e], mu0 = p.gam[2 * p.fstride + e];
      mu1 = p.gam[3 * p.fstride + e], mu2 = p.gam[4 * p.fstride + e];
    } else {
      interp_weights<R>(v, tab, p.n_g, p.g_min, p.g_max, p.inv_dg, p.inv_fh, t1, t2, mu0, mu1, mu2);
    }
    rec[0 * n + idx] = w2_over_1 / (v * v);              // k² = ω²/v²
    rec[1 * n + idx] = R(1) - R(4) * (t1 + t2);          // t0
    rec[2 * n + idx] = t1;
    rec[3 * n + idx] = t2;
    rec[4 * n + idx] = mu0;
    rec[5 * n + idx] = mu1;
    rec[6 * n + idx] = mu2;
    rec[7 * n + idx] = (R(1) - mu0 - R(6) * mu1 - R(12) * mu2) * R(0.125);
  }
}

// =============================================================================================
// GAm rule (reading A19): per owned point, the mean of the interpolated free weights
// (t1, t2, μ0, μ1, μ2) over the in-grid nodes of its 27-point stencil (v halo planes carry the
// neighbouring slabs).  One-time, at assemble; out: [5][nzl+2][ny][ldx] (halo planes not written).
// radius 0 stores the row's own weights: the "record mode" of the GA rule.
// =============================================================================================
template <typename R>
__global__ void gam_field_kernel(ApplyParams<R> p, R* __restrict__ out, int radius) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* tab = reinterpret_cast<R*>(smem_raw);
  for (int i = threadIdx.x; i < p.n_g * TAB_STRIDE; i += blockDim.x) tab[i] = p.tab[i];
  __syncthreads();
  const long long n = (long long)p.nzl * p.ny * p.nx;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (long long)gridDim.x * blockDim.x) {
    int zl, y, x;
    const long long e = st_elem(p, idx, zl, y, x);
    R a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0;
    int cnt = 0;
    for (int dz = -radius; dz <= radius; dz++) {
      const int zg = p.z0 + zl + dz;
      if (zg < 0 || zg >= p.nzg) continue;
      for (int dy = -radius; dy <= radius; dy++) {
        if (y + dy < 0 || y + dy >= p.ny) continue;
        for (int dx = -radius; dx <= radius; dx++) {
          if (x + dx < 0 || x + dx >= p.nx) continue;
          R t1, t2, mu0, mu1, mu2;
          interp_weights<R>(p.v[e + (long long)dz * p.plane + (long long)dy * p.ldx + dx], tab, p.n_g,
                            p.g_min, p.g_max, p.inv_dg, p.inv_fh, t1, t2, mu0, mu1, mu2);
          a0 += t1;
          a1 += t2;
          a2 += mu0;
          a3 += mu1;
          a4 += mu2;
          cnt++;
        }
      }
    }
    const R ic = R(1) / (R)cnt;
    out[e] = a0 * ic;
    out[p.fstride + e] = a1 * ic;
    out[2 * p.fstride + e] = a2 * ic;
    out[3 * p.fstride + e] = a3 * ic;
    out[4 * p.fstride + e] = a4 * ic;
  }
}

// =============================================================================================
// K6 point sources (consistent: row n's own mass weights; nodal: 1/h³)
// =============================================================================================
template <typename R>
__global__ void sources_kernel(ApplyParams<R> p, int nsrc, const long long* __restrict__ nodes,
                               const double* __restrict__ amps, int consistent, R ih3,
                               typename Cx<R>::T* __restrict__ b) {
  typedef typename Cx<R>::T C;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* tab = reinterpret_cast<R*>(smem_raw);
  for (int i = threadIdx.x; i < p.n_g * TAB_STRIDE; i += blockDim.x) tab[i] = p.tab[i];
  __syncthreads();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nsrc * 27) return;
  const int s = t / 27, d = t % 27;
  const int dx = d % 3 - 1, dy = (d / 3) % 3 - 1, dz = d / 9 - 1;
  if (!consistent && (dx | dy | dz) != 0) return;
  const long long X = nodes[3 * s] + dx, Y = nodes[3 * s + 1] + dy, Z = nodes[3 * s + 2] + dz;
  if (X < 0 || X >= p.nx || Y < 0 || Y >= p.ny || Z < p.z0 || Z >= (long long)p.z0 + p.nzl) return;
  const int zl = (int)(Z - p.z0);
  const long long o = (long long)s * p.fstride + (long long)(zl + 1) * p.plane + Y * p.ldx + X;
  R w = ih3;
  if (consistent) {
    R t1, t2, mu0, mu1, mu2;
    const long long e = (long long)(zl + 1) * p.plane + Y * p.ldx + X;
    if (p.gam != nullptr) {   // GAm: the row's 27-node mean weights (A19)
      t1 = p.gam[e], t2 = p.gam[p.fstride + e], mu0 = p.gam[2 * p.fstride + e];
      mu1 = p.gam[3 * p.fstride + e], mu2 = p.gam[4 * p.fstride + e];
    } else {
      interp_weights<R>(p.v[e], tab, p.n_g, p.g_min, p.g_max, p.inv_dg, p.inv_fh, t1, t2, mu0, mu1, mu2);
    }
    const int cls = (dx != 0) + (dy != 0) + (dz != 0);
    const R mu3 = (R(1) - mu0 - R(6) * mu1 - R(12) * mu2) * R(0.125);
    const R mu = cls == 0 ? mu0 : (cls == 1 ? mu1 : (cls == 2 ? mu2 : mu3));
    w = mu * ih3;
  }
  const double ar = amps ? amps[2 * s] : 1.0, ai = amps ? amps[2 * s + 1] : 0.0;
  C val;
  val.x = (R)(ar * (double)w);
  val.y = (R)(ai * (double)w);
  b[o] = val;
}

// =============================================================================================
// w = 1/v² (the apply's per-point model input), all planes incl. halos
// =============================================================================================
template <typename R>
__global__ void winv_kernel(const R* __restrict__ v, R* __restrict__ w, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const R a = v[i];
    w[i] = a > R(0) ? R(1) / (a * a) : R(0);   // pad columns (v = 0) get w = 0
  }
}

template <typename R>
cudaError_t launch_winv(const R* v, R* w, long long n, cudaStream_t s) {
  winv_kernel<R><<<592, 256, 0, s>>>(v, w, n);
  return cudaGetLastError();
}
template cudaError_t launch_winv<float>(const float*, float*, long long, cudaStream_t);
template cudaError_t launch_winv<double>(const double*, double*, long long, cudaStream_t);

// =============================================================================================
// velocity validation / statistics: min, max, non-finite count, clamped count
// =============================================================================================
template <typename R>
__global__ void vstats_kernel(const R* __restrict__ v, long long n, int nx, int ldx, R inv_fh, R g_min, R g_max,
                              unsigned long long* __restrict__ out /* [4]: minbits,maxbits,bad,clamped */) {
  R lmin = R(3.0e38), lmax = R(0);
  unsigned long long bad = 0, clamped = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long row = i / nx;
    const R x = v[row * ldx + (i - row * nx)];
    if (!(x > R(0)) || !isfinite((double)x)) { bad++; continue; }
    lmin = x < lmin ? x : lmin;
    lmax = x > lmax ? x : lmax;
    const R G = x * inv_fh;
    if (G < g_min || G > g_max) clamped++;
  }
  for (int o = 16; o > 0; o >>= 1) {
    lmin = fmin(lmin, __shfl_xor_sync(0xffffffffu, lmin, o));
    lmax = fmax(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
    clamped += __shfl_xor_sync(0xffffffffu, clamped, o);
  }
  if ((threadIdx.x & 31) == 0) {
    const double dmin = (double)lmin, dmax = (double)lmax;   // positive doubles order like their bits
    atomicMin(&out[0], (unsigned long long)__double_as_longlong(dmin));
    atomicMax(&out[1], (unsigned long long)__double_as_longlong(dmax));
    atomicAdd(&out[2], bad);
    atomicAdd(&out[3], clamped);
  }
}

// =============================================================================================
// K3: BiCGSTAB vector kernels (per RHS in blockIdx.y).  Scalars come from the fp64 dot buffers
// written by the previous kernels; every CTA recomputes them identically, CTA 0 records them.
// =============================================================================================
__device__ __forceinline__ double2 zdiv(double2 a, double2 b) {
  const double d = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}
// error-free sum (Knuth TwoSum): s = fl(a + b), e = (a + b) − s exactly
__device__ __forceinline__ void two_sum(float a, float b, float& s, float& e) {
  s = __fadd_rn(a, b);
  const float bp = __fsub_rn(s, a);
  e = __fadd_rn(__fsub_rn(a, __fsub_rn(s, bp)), __fsub_rn(b, bp));
}
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  const double bp = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bp)), __dsub_rn(b, bp));
}
__device__ __forceinline__ double2 zmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ bool tiny(double2 a, double scale) {
  const double m = fabs(a.x) + fabs(a.y);
  return !(m > 1e-300 * scale) || !isfinite(m);
}

template <typename R>
__device__ __forceinline__ typename Cx<R>::T to_c(double2 a) {
  typename Cx<R>::T r;
  r.x = (R)a.x;
  r.y = (R)a.y;
  return r;
}

// p = r̂0 = r, rho = (r̂0, r) = ‖r‖²  (after the initial residual)
template <typename R>
__global__ void bicg_init_kernel(VecParams<R> q) {
  typedef typename Cx<R>::T C;
  const int rhs = blockIdx.y;
  if (q.active[rhs] == 0) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    SolverState& st = q.state[rhs];
    const double rr = q.dotR[3 * rhs + 0];
    st.rho_next[0] = rr;
    st.rho_next[1] = 0.0;
    st.flags = 0;
  }
  const long long off = (long long)rhs * q.fstride + q.plane;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < q.n; i += (long long)gridDim.x * blockDim.x) {
    const C r = q.r[off + i];
    q.rhat[off + i] = r;
    q.p[off + i] = r;
  }
}

// after a residual replacement: rho = (r̂0, r)
__global__ void bicg_rho_reset_kernel(const double* __restrict__ dotR, SolverState* state, const int* active, int nrhs) {
  const int rhs = threadIdx.x + blockIdx.x * blockDim.x;
  if (rhs >= nrhs || active[rhs] == 0) return;
  state[rhs].rho_next[0] = dotR[3 * rhs + 1];
  state[rhs].rho_next[1] = dotR[3 * rhs + 2];
}

// s = r − α v, α = ρ/(r̂0, v)   (s overwrites r)
template <typename R>
__global__ void bicg_s_kernel(VecParams<R> q) {
  typedef typename Cx<R>::T C;
  const int rhs = blockIdx.y;
  if (q.active[rhs] == 0) return;
  SolverState& st = q.state[rhs];
  const double2 rho = make_double2(st.rho_next[0], st.rho_next[1]);
  const double2 den = make_double2(q.dotA[2 * rhs], q.dotA[2 * rhs + 1]);
  double2 alpha = make_double2(0.0, 0.0);
  const bool brk = tiny(den, 1.0) || tiny(rho, 1.0);
  if (!brk) alpha = zdiv(rho, den);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st.alpha[0] = alpha.x;
    st.alpha[1] = alpha.y;
    st.rho_used[0] = rho.x;
    st.rho_used[1] = rho.y;
    if (brk) st.flags |= 1;
  }
  const C a = to_c<R>(alpha);
  const long long off = (long long)rhs * q.fstride + q.plane;
  // 4 independent elements per thread and step: 8 loads in flight per thread (the kernel is HBM-bound)
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < q.n; i0 += 4 * stride) {
    C r[4], v[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const long long i = i0 + k * stride;
      if (i < q.n) {
        r[k] = q.r[off + i];
        v[k] = q.v[off + i];
      }
    }
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const long long i = i0 + k * stride;
      if (i < q.n) {
        C s;
        s.x = r[k].x - (a.x * v[k].x - a.y * v[k].y);
        s.y = r[k].y - (a.x * v[k].y + a.y * v[k].x);
        q.r[off + i] = s;
      }
    }
  }
}

// ω = (t,s)/(t,t); ρ' = (r̂0,s) − ω (r̂0,t); β = (ρ'/ρ)(α/ω);
// x += α p + ω s; r = s − ω t; p = r + β (p − ω v); partial ‖r‖²
template <typename R, int NT>
__global__ void __launch_bounds__(NT) bicg_update_kernel(VecParams<R> q) {
  typedef typename Cx<R>::T C;
  const int rhs = blockIdx.y;
  if (q.active[rhs] == 0) return;
  SolverState& st = q.state[rhs];
  const double* dB = q.dotB + 7 * rhs;
  const double2 ts = make_double2(dB[0], dB[1]);
  const double tt = dB[2];
  const double2 rs = make_double2(dB[3], dB[4]);
  const double2 rt = make_double2(dB[5], dB[6]);
  double2 alpha = make_double2(st.alpha[0], st.alpha[1]);
  const double2 rho = make_double2(st.rho_used[0], st.rho_used[1]);
  double2 omega = make_double2(0.0, 0.0), beta = make_double2(0.0, 0.0), rho_new = make_double2(0.0, 0.0);
  bool brk = (st.flags & 1) != 0 || !(tt > 0.0) || !isfinite(tt);
  if (!brk) {
    omega = make_double2(ts.x / tt, ts.y / tt);
    const double2 wrt = zmul(omega, rt);
    rho_new = make_double2(rs.x - wrt.x, rs.y - wrt.y);
    if (tiny(omega, 1.0) || tiny(rho, 1.0)) brk = true;
    else beta = zmul(zdiv(rho_new, rho), zdiv(alpha, omega));
  }
  if (brk) { alpha.x = alpha.y = 0.0; omega.x = omega.y = 0.0; beta.x = beta.y = 0.0; }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st.omega[0] = omega.x;
    st.omega[1] = omega.y;
    st.rho_next[0] = rho_new.x;
    st.rho_next[1] = rho_new.y;
    if (brk) st.flags |= 1;
  }
  const C a = to_c<R>(alpha), w = to_c<R>(omega), bt = to_c<R>(beta);
  const long long off = (long long)rhs * q.fstride + q.plane;
  double part[1] = {0.0};
  // two independent elements per thread and step (12 loads in flight per thread; HBM-bound)
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < q.n; i0 += 2 * stride) {
  C S_[2], T_[2], P_[2], V_[2], X_[2], L_[2];
#pragma unroll
  for (int k = 0; k < 2; k++) {
    const long long i = i0 + k * stride;
    if (i < q.n) {
      S_[k] = q.r[off + i];
      T_[k] = q.t[off + i];
      P_[k] = q.p[off + i];
      V_[k] = q.v[off + i];
      X_[k] = q.x[off + i];
      if (q.xlo != nullptr) L_[k] = q.xlo[off + i];
    }
  }
#pragma unroll
  for (int k = 0; k < 2; k++) {
    const long long i = i0 + k * stride;
    if (i >= q.n) continue;
    const C s = S_[k], t = T_[k], pp = P_[k], vv = V_[k];
    C xx = X_[k];
    // x += α p + ω s; with q.xlo the iterate is the double-word x + xlo (compensated update)
    C dx;
    const C dp_ = q.ph != nullptr ? q.ph[off + i] : pp;   // right preconditioning: M⁻¹p, M⁻¹s
    const C ds_ = q.sh != nullptr ? q.sh[off + i] : s;
    dx.x = (a.x * dp_.x - a.y * dp_.y) + (w.x * ds_.x - w.y * ds_.y);
    dx.y = (a.x * dp_.y + a.y * dp_.x) + (w.x * ds_.y + w.y * ds_.x);
    if (q.xlo != nullptr) {
      C lo = L_[k];
      two_sum(xx.x, dx.x + lo.x, xx.x, lo.x);
      two_sum(xx.y, dx.y + lo.y, xx.y, lo.y);
      q.xlo[off + i] = lo;
    } else {
      xx.x += dx.x;
      xx.y += dx.y;
    }
    // r = s − ω t
    C r;
    r.x = s.x - (w.x * t.x - w.y * t.y);
    r.y = s.y - (w.x * t.y + w.y * t.x);
    // p = r + β (p − ω v)
    C d;
    d.x = pp.x - (w.x * vv.x - w.y * vv.y);
    d.y = pp.y - (w.x * vv.y + w.y * vv.x);
    C pn;
    pn.x = r.x + (bt.x * d.x - bt.y * d.y);
    pn.y = r.y + (bt.x * d.y + bt.y * d.x);
    q.x[off + i] = xx;
    q.r[off + i] = r;
    q.p[off + i] = pn;
    part[0] += (double)r.x * (double)r.x + (double)r.y * (double)r.y;
  }
  }
  const int nblocks = gridDim.x;
  block_grid_reduce<1, NT>(part, q.partials + (long long)rhs * nblocks, q.dotR + 3 * rhs, q.tickets + rhs, nblocks,
                           blockIdx.x);
}

// ‖f‖² per RHS over the owned points (used for ‖b‖: the caller's pad columns are not read)
template <typename R, int NT>
__global__ void __launch_bounds__(NT) norm2_kernel(const typename Cx<R>::T* __restrict__ f, long long fstride,
                                                   long long plane, long long n, int nx, int ldx, double* partials,
                                                   double* out, unsigned int* tickets) {
  const int rhs = blockIdx.y;
  const long long off = (long long)rhs * fstride + plane;
  double part[1] = {0.0};
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long row = i / nx;
    const typename Cx<R>::T a = f[off + row * ldx + (i - row * nx)];
    part[0] += (double)a.x * (double)a.x + (double)a.y * (double)a.y;
  }
  block_grid_reduce<1, NT>(part, partials + (long long)rhs * gridDim.x, out + rhs, tickets + rhs, gridDim.x, blockIdx.x);
}

// =============================================================================================
// K3': BiCGStab(2) vector steps (Sleijpen & Fokkema 1993, ℓ = 2, reading A23) — a
// solver option for the models where BiCGSTAB stagnates (its ω → 0 on strongly indefinite
// Helmholtz systems).  One outer step = two BiCGSTAB iterations' worth of applies (four):
//   A: ρ0 ← −ω ρ0; ρ1 = (r̂0, r0); β = α ρ1/ρ0; ρ0 ← ρ1;            u0 = r0 − β u0
//      u1 = A u0, σ = (r̂0, u1)                                          [apply, DOT1]
//   B: α = ρ0/σ;                                                        r0 −= α u1
//      r1 = A r0, ρ1 = (r̂0, r1)                                         [apply, DOT1]
//   C: β = α ρ1/ρ0; ρ0 ← ρ1;                  x += α u0; u0 = r0 − β u0; u1 = r1 − β u1
//      u2 = A u1, σ = (r̂0, u2)                                          [apply, DOT1]
//   D: α = ρ0/σ;                                   r0 −= α u1; r1 −= α u2; ‖r1‖² → dotG
//      r2 = A r1; (r2,r1), ‖r2‖², (r0,r1), (r0,r2)                      [apply, DOT4, r̂ := r0]
//   E: (γ1, γ2) = argmin ‖r0 − γ1 r1 − γ2 r2‖ (2×2 normal equations in fp64); ω = γ2;
//      x += α u0 + γ1 r0 + γ2 r1; r0 −= γ1 r1 + γ2 r2; u0 −= γ1 u1 + γ2 u2;  ‖r0‖², (r̂0, r0) → dotR
// (a, b) = Σ conj(a) b.  Fields: r0 = q.r, r1 = q.r1, r2 = q.r2, u0 = q.p, u1 = q.v, u2 = q.t.
// The BiCG part's x += α u0 is deferred from B to C and from D to E, the next kernels that read u0
// before changing it: 40 fewer B/pt per outer step (x and its compensation word are read and
// written twice instead of three times), same arithmetic.
// State: rho_used = ρ0 after A (read by B, C), rho_next = ρ0 after C (read by D, next A), alpha
// (B, D), omega (E); no kernel reads a field it writes (every CTA derives the scalars itself).
// =============================================================================================
// x += dx in registers; with comp the iterate is the double-word x + lo (compensated update, as
// bicg_update_kernel)
template <typename R>
__device__ __forceinline__ void x_upd(typename Cx<R>::T& xx, typename Cx<R>::T& lo, typename Cx<R>::T dx, bool comp) {
  if (comp) {
    two_sum(xx.x, dx.x + lo.x, xx.x, lo.x);
    two_sum(xx.y, dx.y + lo.y, xx.y, lo.y);
  } else {
    xx.x += dx.x;
    xx.y += dx.y;
  }
}

template <typename R, int NT, int STEP>
__global__ void __launch_bounds__(NT) bicgl_kernel(VecParams<R> q) {
  typedef typename Cx<R>::T C;
  const int rhs = blockIdx.y;
  if (q.active[rhs] == 0) return;
  SolverState& st = q.state[rhs];
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  bool brk = STEP != BCL_INIT && (st.flags & 1) != 0;
  double2 s1 = make_double2(0.0, 0.0), s2 = s1, s3 = s1;   // the step's complex scalars
  if constexpr (STEP == BCL_INIT) {
    if (lead) {   // ρ0 = α = ω = 1... (α = 0 so that the first β vanishes); (r̂0, r0) = ‖r0‖² as r̂0 = r0
      st.rho_next[0] = 1.0;
      st.rho_next[1] = 0.0;
      st.alpha[0] = st.alpha[1] = 0.0;
      st.omega[0] = 1.0;
      st.omega[1] = 0.0;
      st.flags = 0;
      q.dotR[3 * rhs + 1] = q.dotR[3 * rhs + 0];
      q.dotR[3 * rhs + 2] = 0.0;
    }
  } else if constexpr (STEP == BCL_A) {
    const double2 om = make_double2(st.omega[0], st.omega[1]);
    const double2 r0p = zmul(make_double2(-om.x, -om.y), make_double2(st.rho_next[0], st.rho_next[1]));
    const double2 rho1 = make_double2(q.dotR[3 * rhs + 1], q.dotR[3 * rhs + 2]);
    if (tiny(r0p, 1.0) || tiny(rho1, 1.0)) brk = true;
    else s1 = zdiv(zmul(make_double2(st.alpha[0], st.alpha[1]), rho1), r0p);   // β
    if (lead) {
      st.rho_used[0] = rho1.x;
      st.rho_used[1] = rho1.y;
    }
  } else if constexpr (STEP == BCL_B || STEP == BCL_D) {
    const double2 rho = STEP == BCL_B ? make_double2(st.rho_used[0], st.rho_used[1])
                                      : make_double2(st.rho_next[0], st.rho_next[1]);
    const double2 sig = make_double2(q.dotA[2 * rhs], q.dotA[2 * rhs + 1]);
    if (brk || tiny(sig, 1.0) || tiny(rho, 1.0)) brk = true;
    else s1 = zdiv(rho, sig);   // α
    if (lead) {
      st.alpha[0] = s1.x;
      st.alpha[1] = s1.y;
    }
  } else if constexpr (STEP == BCL_C) {
    const double2 rho0 = make_double2(st.rho_used[0], st.rho_used[1]);
    const double2 rho1 = make_double2(q.dotA[2 * rhs], q.dotA[2 * rhs + 1]);
    s2 = make_double2(st.alpha[0], st.alpha[1]);                                  // α of B
    if (brk || tiny(rho0, 1.0)) brk = true;
    else s1 = zdiv(zmul(s2, rho1), rho0);                                         // β
    if (lead) {
      st.rho_next[0] = rho1.x;
      st.rho_next[1] = rho1.y;
    }
  } else {   // BCL_E: normal equations [a11 a12; a21 a22] γ = c of the 2-term minimal residual
    const double* dB = q.dotB + 7 * rhs;
    const double a11 = q.dotG[rhs], a22 = dB[2];
    const double2 a21 = make_double2(dB[0], dB[1]);          // (r2, r1)
    const double2 a12 = make_double2(a21.x, -a21.y);         // (r1, r2)
    const double2 c1 = make_double2(dB[3], -dB[4]);          // (r1, r0) = conj((r0, r1))
    const double2 c2 = make_double2(dB[5], -dB[6]);          // (r2, r0)
    const double det = a11 * a22 - (a21.x * a21.x + a21.y * a21.y);
    s3 = make_double2(st.alpha[0], st.alpha[1]);   // α of D
    if (brk || !(det > 1e-14 * a11 * a22) || !isfinite(det)) {
      brk = true;
    } else {
      const double2 n1 = csub(cscale(a22, c1), cmul(a12, c2));
      const double2 n2 = csub(cscale(a11, c2), cmul(a21, c1));
      s1 = cscale(1.0 / det, n1);   // γ1
      s2 = cscale(1.0 / det, n2);   // γ2 = ω
    }
    if (lead) {
      st.omega[0] = s2.x;
      st.omega[1] = s2.y;
    }
  }
  // on breakdown the step's own scalars vanish; the deferred α u0 (C: s2, E: s3) is still applied
  // (its α was stored as 0 if its own step broke down), keeping x consistent with r
  if (brk) {
    s1 = make_double2(0.0, 0.0);
    if (STEP != BCL_C) s2 = s1;
  }
  if (lead && brk) st.flags |= 1;
  const C a = to_c<R>(s1), b = to_c<R>(s2), g = to_c<R>(s3);
  const long long off = (long long)rhs * q.fstride + q.plane;
  constexpr int K = STEP == BCL_E ? 3 : (STEP == BCL_D ? 1 : 0);
  double part[K > 0 ? K : 1];
#pragma unroll
  for (int k = 0; k < (K > 0 ? K : 1); k++) part[k] = 0.0;
  // U elements per thread and pass: every operand of the U elements is loaded before the first store
  // (the fields may alias as far as the compiler knows), so 2U..9U loads are in flight (HBM-bound)
  constexpr int U = sizeof(R) == 4 ? 4 : 2;
  const bool comp = q.xlo != nullptr;
  C f0[U], f1[U], f2[U], f3[U], f4[U], f5[U], f6[U], f7[U], f8[U];
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < q.n; i0 += U * stride) {
#pragma unroll
    for (int k = 0; k < U; k++) {
      const long long i = i0 + k * stride;
      if (i >= q.n) continue;
      const long long e = off + i;
      if constexpr (STEP == BCL_INIT) {
        f0[k] = q.r[e];
      } else if constexpr (STEP == BCL_A) {
        f0[k] = q.r[e];
        f1[k] = q.p[e];
      } else if constexpr (STEP == BCL_B) {
        f0[k] = q.r[e];
        f1[k] = q.v[e];
      } else if constexpr (STEP == BCL_C) {
        f0[k] = q.p[e];
        f1[k] = q.x[e];
        if (comp) f2[k] = q.xlo[e];
        f3[k] = q.r[e];
        f4[k] = q.r1[e];
        f5[k] = q.v[e];
      } else if constexpr (STEP == BCL_D) {
        f0[k] = q.r[e];
        f1[k] = q.v[e];
        f2[k] = q.r1[e];
        f3[k] = q.t[e];
      } else {
        f0[k] = q.r[e];
        f1[k] = q.r1[e];
        f2[k] = q.p[e];
        f3[k] = q.x[e];
        if (comp) f4[k] = q.xlo[e];
        f5[k] = q.r2[e];
        f6[k] = q.v[e];
        f7[k] = q.t[e];
        f8[k] = q.rhat[e];
      }
    }
#pragma unroll
    for (int k = 0; k < U; k++) {
      const long long i = i0 + k * stride;
      if (i >= q.n) continue;
      const long long e = off + i;
      if constexpr (STEP == BCL_INIT) {
        q.rhat[e] = f0[k];
        q.p[e] = czero(R(0));
      } else if constexpr (STEP == BCL_A) {   // u0 = r0 − β u0
        q.p[e] = csub(f0[k], cmul(a, f1[k]));
      } else if constexpr (STEP == BCL_B) {   // r0 −= α u1
        q.r[e] = csub(f0[k], cmul(a, f1[k]));
      } else if constexpr (STEP == BCL_C) {   // x += α u0 (of B); u0 = r0 − β u0; u1 = r1 − β u1
        const C u0 = f0[k];
        x_upd<R>(f1[k], f2[k], cmul(b, u0), comp);
        q.x[e] = f1[k];
        if (comp) q.xlo[e] = f2[k];
        q.p[e] = csub(f3[k], cmul(a, u0));
        q.v[e] = csub(f4[k], cmul(a, f5[k]));
      } else if constexpr (STEP == BCL_D) {   // r0 −= α u1; r1 −= α u2
        q.r[e] = csub(f0[k], cmul(a, f1[k]));
        const C r1 = csub(f2[k], cmul(a, f3[k]));
        q.r1[e] = r1;
        part[0] += (double)r1.x * (double)r1.x + (double)r1.y * (double)r1.y;
      } else {   // E: x += α u0 (of D) + γ1 r0 + γ2 r1; r0 −= γ1 r1 + γ2 r2; u0 −= γ1 u1 + γ2 u2
        const C r0 = f0[k], r1 = f1[k], u0 = f2[k];
        x_upd<R>(f3[k], f4[k], cadd(cmul(g, u0), cadd(cmul(a, r0), cmul(b, r1))), comp);
        q.x[e] = f3[k];
        if (comp) q.xlo[e] = f4[k];
        const C rn = csub(r0, cadd(cmul(a, r1), cmul(b, f5[k])));
        q.r[e] = rn;
        q.p[e] = csub(u0, cadd(cmul(a, f6[k]), cmul(b, f7[k])));
        part[0] += (double)rn.x * (double)rn.x + (double)rn.y * (double)rn.y;
        acc_cdot(part[1], part[2], f8[k], rn);
      }
    }
  }
  if constexpr (K > 0) {
    const int nblocks = gridDim.x;
    double* out = STEP == BCL_E ? q.dotR + 3 * rhs : q.dotG + rhs;
    block_grid_reduce<K, NT>(part, q.partials + (long long)rhs * nblocks * K, out, q.tickets + rhs, nblocks,
                             blockIdx.x);
  }
}

// =============================================================================================
// host-side launchers (kernels.h)
// =============================================================================================
// register path: R = double only (complex128, and the fp64 residual of the complex64 solver)
template <typename R> struct ApplyCfg;
template <> struct ApplyCfg<double> { enum { NY = 1, WARPS = 4 }; };

template <typename R>
long long apply_nblocks_x(int nx, int ny) {   // CTAs covering one z-chunk of the (strip, x-tile) space
  constexpr int NY = ApplyCfg<R>::NY, W = ApplyCfg<R>::WARPS;
  const long long nwarps = (long long)((ny + NY - 1) / NY) * ((nx + XT - 1) / XT);
  return (nwarps + W - 1) / W;
}
template long long apply_nblocks_x<double>(int, int);

// Register-path launches (apply27_v2): the general launch (everything) and the interior box launch;
// returns the total number of CTAs per RHS (partials of the dot epilogues).
template <typename R, typename S>
long long apply_plan(ApplyParams<R, S>& p) {
  constexpr int NY = ApplyCfg<R>::NY, W = ApplyCfg<R>::WARPS;
  p.nbx = (int)apply_nblocks_x<R>(p.nx, p.ny);
  // tiles whose outputs lie in [max(lo,1), min(hi, hmax)] (footprint inside the grid, no PML)
  auto range = [](int lo, int hi, int hmax, int T, int& a, int& b) {
    const int l = std::max(lo, 1), h = std::min(hi, hmax);
    a = (l + T - 1) / T;
    b = (h - (T - 1) >= 0) ? (h - (T - 1)) / T + 1 : 0;
    if (b < a) b = a;
  };
  range(p.lo[0], p.hi[0], p.nx - 2, XT, p.box_t0, p.box_t1);
  range(p.lo[1], p.hi[1], p.ny - 2, NY, p.box_s0, p.box_s1);
  // z-chunks: planes whose outputs lie in [max(lo,1), min(hi, nzg-2)] (global) are cut into chunks of
  // ≤ zc planes (the interior chunks); the planes below / above form one chunk each
  {
    const int zl = std::min(std::max(std::max(p.lo[2], 1) - p.z0, 0), p.nzl);
    const int zh = std::max(std::min(std::min(p.hi[2], p.nzg - 2) - p.z0 + 1, p.nzl), zl);   // exclusive
    if (zh > zl) {
      p.zlo = zl;
      p.zhi = zh;
      p.nlow = zl > 0 ? 1 : 0;
      p.nint = (zh - zl + p.zc - 1) / p.zc;
      p.nchunks = p.nlow + p.nint + (zh < p.nzl ? 1 : 0);
      p.box_c0 = p.nlow;
      p.box_c1 = p.nlow + p.nint;
    } else {   // no interior planes: plain chunks, no box
      p.zlo = 0;
      p.zhi = p.nzl;
      p.nlow = 0;
      p.nint = (p.nzl + p.zc - 1) / p.zc;
      p.nchunks = p.nint;
      p.box_c0 = p.box_c1 = 0;
    }
  }
  const long long bw = (long long)(p.box_s1 - p.box_s0) * (p.box_t1 - p.box_t0);
  p.box_nbx = (int)((bw + W - 1) / W);
  if (bw == 0 || p.box_c1 <= p.box_c0) {
    p.box_nbx = 0;
    p.box_c0 = p.box_c1 = 0;
    p.box_s0 = p.box_s1 = p.box_t0 = p.box_t1 = 0;
  }
  // general work list
  const int ntx = (p.nx + XT - 1) / XT, nstrips = (p.ny + NY - 1) / NY;
  const int nhigh = p.nchunks - p.nlow - p.nint;
  if (p.box_nbx > 0) {
    p.nbound = p.nlow + nhigh;
    p.frame_warps = nstrips * ntx - (p.box_s1 - p.box_s0) * (p.box_t1 - p.box_t0);
    p.nbx_frame = (p.frame_warps + W - 1) / W;
  } else {   // no box: every chunk is processed whole by the general launch
    p.nbound = p.nchunks;
    p.frame_warps = nstrips * ntx;
    p.nbx_frame = p.nbx;
  }
  p.gen_blocks = p.nbound == p.nchunks ? p.nbx * p.nchunks : p.nbound * p.nbx + p.nint * p.nbx_frame;
  return (long long)p.gen_blocks + (long long)p.box_nbx * (p.box_c1 - p.box_c0);
}
template long long apply_plan<double, double>(ApplyParams<double, double>&);
template long long apply_plan<double, float>(ApplyParams<double, float>&);

template <typename R, typename S, bool COLLOC, int EPI, bool INTERIOR>
static cudaError_t launch_one(const ApplyParams<R, S>& p, long long nb, cudaStream_t s) {
  constexpr int NY = ApplyCfg<R>::NY, W = ApplyCfg<R>::WARPS;
  auto kern = apply27_v2<R, S, NY, W, COLLOC, EPI, INTERIOR>;
  if (nb <= 0) return cudaSuccess;
  if (nb >= (1LL << 31)) return cudaErrorInvalidConfiguration;
  const size_t smem = (size_t)p.tab_n * SmemPitch<R>::V * sizeof(R);
  static size_t attr = 0;
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  kern<<<(unsigned)nb, 32 * W, smem, s>>>(p);
  return cudaGetLastError();
}

static thread_local int g_last_apply_launches = 0;
int apply_last_launches() { return g_last_apply_launches; }

// the tile-width instantiations live in their own translation units (tm64.cu, tm32.cu)
cudaError_t launch_apply_tm(const TmLaunch& L, const ApplyParams<float, float>& p, int nrhs, bool colloc, int epi,
                            cudaStream_t s) {
  g_last_apply_launches = p.tm_nitems > 0 ? 1 : 0;
  if (p.tm_nitems <= 0) return cudaSuccess;
  if (p.tm_tx == 64) return launch_apply_tm_tx<64>(L, p, nrhs, colloc, epi, s);
  if (p.tm_tx == 32) return launch_apply_tm_tx<32>(L, p, nrhs, colloc, epi, s);
  return cudaErrorInvalidValue;
}

template <typename R, typename S, bool COLLOC, int EPI>
static cudaError_t launch_apply_t(ApplyParams<R, S> p, int nrhs, cudaStream_t s) {
  apply_plan(p);
  p.nrhs = nrhs;
  const long long ngen = (long long)p.gen_blocks * nrhs;
  const long long nbox = (long long)p.box_nbx * (p.box_c1 - p.box_c0) * nrhs;
  g_last_apply_launches = (ngen > 0) + (nbox > 0);
  cudaError_t e = launch_one<R, S, COLLOC, EPI, false>(p, ngen, s);
  if (e != cudaSuccess) return e;
  return launch_one<R, S, COLLOC, EPI, true>(p, nbox, s);
}

// register path: complex128 (every epilogue)
template <>
cudaError_t launch_apply<double, double>(const ApplyParams<double, double>& p, int nrhs, bool colloc, int epi,
                                         cudaStream_t s) {
  if (!colloc) {
    switch (epi) {
      case EPI_PLAIN: return launch_apply_t<double, double, false, EPI_PLAIN>(p, nrhs, s);
      case EPI_DOT1: return launch_apply_t<double, double, false, EPI_DOT1>(p, nrhs, s);
      case EPI_DOT4: return launch_apply_t<double, double, false, EPI_DOT4>(p, nrhs, s);
      case EPI_RESID: return launch_apply_t<double, double, false, EPI_RESID>(p, nrhs, s);
    }
  } else {
    switch (epi) {
      case EPI_PLAIN: return launch_apply_t<double, double, true, EPI_PLAIN>(p, nrhs, s);
      case EPI_DOT1: return launch_apply_t<double, double, true, EPI_DOT1>(p, nrhs, s);
      case EPI_DOT4: return launch_apply_t<double, double, true, EPI_DOT4>(p, nrhs, s);
      case EPI_RESID: return launch_apply_t<double, double, true, EPI_RESID>(p, nrhs, s);
    }
  }
  return cudaErrorInvalidValue;
}

// mixed precision (c64 storage, fp64 arithmetic): the residual of the complex64 solver
template <>
cudaError_t launch_apply<double, float>(const ApplyParams<double, float>& p, int nrhs, bool colloc, int epi,
                                        cudaStream_t s) {
  if (epi == EPI_RESID) return colloc ? launch_apply_t<double, float, true, EPI_RESID>(p, nrhs, s)
                                      : launch_apply_t<double, float, false, EPI_RESID>(p, nrhs, s);
  return cudaErrorInvalidValue;
}

template <typename R>
int apply_occupancy(bool colloc) {
  constexpr int NY = ApplyCfg<R>::NY, W = ApplyCfg<R>::WARPS;
  int nb = 0;
  if (colloc)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, apply27_v2<R, R, NY, W, true, EPI_DOT4, true>, 32 * W, 16 * 1024);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, apply27_v2<R, R, NY, W, false, EPI_DOT4, true>, 32 * W, 16 * 1024);
  return nb > 0 ? nb : 1;
}
template int apply_occupancy<double>(bool);

template <typename R>
cudaError_t launch_record(const ApplyParams<R>& p, R* rec, cudaStream_t s) {
  const size_t smem = (size_t)p.n_g * TAB_STRIDE * sizeof(R);
  cudaFuncSetAttribute(record_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  record_kernel<R><<<1024, 256, smem, s>>>(p, p.w2, rec);
  return cudaGetLastError();
}
template cudaError_t launch_record<float>(const ApplyParams<float>&, float*, cudaStream_t);
template cudaError_t launch_record<double>(const ApplyParams<double>&, double*, cudaStream_t);

// =============================================================================================
// eqerror (reading A20): per-block partial sums (fp64) of W|Re d|, W|Im d|, W|Re ref|,
// W|Im ref| over the owned points at least `npml` nodes from every face and more than `ball` nodes
// from the source, W = h · distance; a fixed-order host sum finishes the reduction.
// =============================================================================================
template <typename R>
__global__ void eqerror_kernel(const typename Cx<R>::T* __restrict__ uref, const typename Cx<R>::T* __restrict__ u,
                               int nx, int ny, int ldx, int nzl, int z0, int nzg, long long xs, long long ys,
                               long long zs, double h, int npml, double ball, double* __restrict__ partials) {
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const long long plane = (long long)nx * ny;
  const long long n = (long long)nzl * plane;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (long long)gridDim.x * blockDim.x) {
    const int zl = (int)(idx / plane);
    const int rem = (int)(idx - (long long)zl * plane);
    const int y = rem / nx, x = rem - y * nx;
    const int zg = z0 + zl;
    if (x < npml || x >= nx - npml || y < npml || y >= ny - npml || zg < npml || zg >= nzg - npml) continue;
    const double dx = (double)(x - xs), dy = (double)(y - ys), dz = (double)(zg - zs);
    const double d = sqrt(dx * dx + dy * dy + dz * dz);
    if (!(d > ball)) continue;
    const double W = h * d;
    const long long e = (long long)(zl + 1) * ny * ldx + (long long)y * ldx + x;
    const typename Cx<R>::T a = uref[e], b = u[e];
    acc[0] += fabs(W * ((double)a.x - (double)b.x));
    acc[1] += fabs(W * ((double)a.y - (double)b.y));
    acc[2] += fabs(W * (double)a.x);
    acc[3] += fabs(W * (double)a.y);
  }
  __shared__ double red[8][4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    double v = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    double v = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) v += red[w][threadIdx.x];
    partials[blockIdx.x * 4 + threadIdx.x] = v;
  }
}

template <typename R>
cudaError_t launch_eqerror(const typename Cx<R>::T* uref, const typename Cx<R>::T* u, int nx, int ny, int ldx, int nzl,
                           int z0, int nzg, const long long* src, double h, int npml, double ball, double* partials,
                           int nblocks, cudaStream_t s) {
  eqerror_kernel<R><<<nblocks, 256, 0, s>>>(uref, u, nx, ny, ldx, nzl, z0, nzg, src[0], src[1], src[2], h, npml, ball,
                                            partials);
  return cudaGetLastError();
}
template cudaError_t launch_eqerror<float>(const float2*, const float2*, int, int, int, int, int, int, const long long*,
                                           double, int, double, double*, int, cudaStream_t);
template cudaError_t launch_eqerror<double>(const double2*, const double2*, int, int, int, int, int, int, const long long*,
                                            double, int, double, double*, int, cudaStream_t);

// =============================================================================================
// Explicit matrix export (the paper's direct-solver setting): the 27 entries of
// every owned row in the per-axis form of the oracle (readings A6, A8; Eq. 8 / Eq. "10" mass; GA or
// GAm weights) — ELL layout, column = global node index or -1 outside the grid (Dirichlet, A9).
//   A[n, n+d] = ω² μ_class(d) w_{n+d}  (Eq. 8; w_n for Eq. "10")  +  Σ_a D_a(n_a, d_a) T(d⊥; t(n))
// =============================================================================================
template <typename R>
__global__ void matrix_kernel(ApplyParams<R> p, bool colloc, long long* __restrict__ cols,
                              typename Cx<R>::T* __restrict__ vals) {
  typedef typename Cx<R>::T C;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* tab = reinterpret_cast<R*>(smem_raw);
  for (int i = threadIdx.x; i < p.n_g * TAB_STRIDE; i += blockDim.x) tab[i] = p.tab[i];
  __syncthreads();
  const long long n = (long long)p.nzl * p.ny * p.nx;
  const R ih2 = p.ih2;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (long long)gridDim.x * blockDim.x) {
    int zl, y, x;
    const long long e = st_elem(p, idx, zl, y, x);   // storage element of the row
    const int zg = p.z0 + zl;
    R t1, t2, mu0, mu1, mu2;
    if (p.gam != nullptr) {
      t1 = p.gam[e], t2 = p.gam[p.fstride + e], mu0 = p.gam[2 * p.fstride + e];
      mu1 = p.gam[3 * p.fstride + e], mu2 = p.gam[4 * p.fstride + e];
    } else {
      interp_weights<R>(p.v[e], tab, p.n_g, p.g_min, p.g_max, p.inv_dg, p.inv_fh, t1, t2, mu0, mu1, mu2);
    }
    const R t0 = R(1) - R(4) * (t1 + t2);
    const R mu[4] = {mu0, mu1, mu2, (R(1) - mu0 - R(6) * mu1 - R(12) * mu2) * R(0.125)};
    const R tw[3] = {t0, t1, t2};
    // stretched 1-D second differences: a± = h⁻² + δ± (the device holds δ)
    const int ia[3] = {x, y, zg};
    C am[3], ap[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
      const C dm = p.dm[a][ia[a]], dpp = p.dp[a][ia[a]];
      am[a] = make_cx(dm.x + ih2, dm.y);
      ap[a] = make_cx(dpp.x + ih2, dpp.y);
    }
    const R wn = p.w[e];
    for (int d = 0; d < 27; d++) {
      const int dx = d % 3 - 1, dy = (d / 3) % 3 - 1, dz = d / 9 - 1;
      const long long o = idx * 27 + d;
      const int xx = x + dx, yy = y + dy, zz = zg + dz;
      if (xx < 0 || xx >= p.nx || yy < 0 || yy >= p.ny || zz < 0 || zz >= p.nzg) {
        cols[o] = -1;
        vals[o] = make_cx(R(0), R(0));
        continue;
      }
      const int cls = (dx != 0) + (dy != 0) + (dz != 0);
      const R wnb = colloc ? wn : p.w[e + (long long)dz * p.plane + (long long)dy * p.ldx + dx];
      C v = make_cx(p.w2 * mu[cls] * wnb, R(0));
      const int dd[3] = {dx, dy, dz};
#pragma unroll
      for (int a = 0; a < 3; a++) {
        const int pa = dd[(a + 1) % 3], qa = dd[(a + 2) % 3];
        const R T = tw[(pa != 0) + (qa != 0)];
        const C D = dd[a] < 0 ? am[a] : (dd[a] > 0 ? ap[a] : make_cx(-am[a].x - ap[a].x, -am[a].y - ap[a].y));
        v.x += D.x * T;
        v.y += D.y * T;
      }
      cols[o] = ((long long)zz * p.ny + yy) * p.nx + xx;
      vals[o] = v;
    }
  }
}

template <typename R>
cudaError_t launch_matrix(const ApplyParams<R>& p, bool colloc, long long* cols, typename Cx<R>::T* vals, cudaStream_t s) {
  const size_t smem = (size_t)p.n_g * TAB_STRIDE * sizeof(R);
  cudaFuncSetAttribute(matrix_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  matrix_kernel<R><<<148 * 4, 256, smem, s>>>(p, colloc, cols, vals);
  return cudaGetLastError();
}
template cudaError_t launch_matrix<float>(const ApplyParams<float>&, bool, long long*, float2*, cudaStream_t);
template cudaError_t launch_matrix<double>(const ApplyParams<double>&, bool, long long*, double2*, cudaStream_t);

// =============================================================================================
// Plane-wave dispersion of the stencil: vtilde = G/(√(2J) π) √R with
//   R = ws1(3−C) + (ws2/3)(6−C−B) + (ws3/2)(3−3A+B−C),  J = μ0 + 2μ1 C + 4μ2 B + 8μ3 A
//   A = cos a cos b cos c, B = Σ pairwise products, C = Σ cosines; (a, b, c) = 2π/G (cosφ cosθ,
//   cosφ sinθ, sinφ).  w7[i] = (ws1, ws2, ws3, wm0, wm1, wm2, wm3) at G[i]; fp64.
// =============================================================================================
__global__ void dispersion_kernel(const double* __restrict__ w7, const double* __restrict__ G, int nG,
                                  const double* __restrict__ theta, const double* __restrict__ phi, int nang,
                                  double* __restrict__ out) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)nG * nang) return;
  const int i = (int)(t / nang), j = (int)(t - (long long)i * nang);
  const double g = G[i], k = 2.0 * M_PI / g;
  const double a = k * cos(phi[j]) * cos(theta[j]), b = k * cos(phi[j]) * sin(theta[j]), c = k * sin(phi[j]);
  const double ca = cos(a), cb = cos(b), cc = cos(c);
  const double A = ca * cb * cc, B = ca * cb + ca * cc + cb * cc, C = ca + cb + cc;
  const double* w = w7 + 7 * i;
  const double Rr = w[0] * (3.0 - C) + w[1] / 3.0 * (6.0 - C - B) + 0.5 * w[2] * (3.0 - 3.0 * A + B - C);
  const double mu0 = w[3], mu1 = w[4] / 6.0, mu2 = w[5] / 12.0, mu3 = w[6] / 8.0;
  const double J = mu0 + 2.0 * mu1 * C + 4.0 * mu2 * B + 8.0 * mu3 * A;
  out[t] = g / (sqrt(2.0 * J) * M_PI) * sqrt(Rr);
}
cudaError_t launch_dispersion(const double* w7, const double* G, int nG, const double* theta, const double* phi, int nang,
                              double* out, cudaStream_t s) {
  const long long n = (long long)nG * nang;
  dispersion_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(w7, G, nG, theta, phi, nang, out);
  return cudaGetLastError();
}

template <typename R>
cudaError_t launch_gam_field(const ApplyParams<R>& p, R* out, int radius, cudaStream_t s) {
  const size_t smem = (size_t)p.n_g * TAB_STRIDE * sizeof(R);
  cudaFuncSetAttribute(gam_field_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  gam_field_kernel<R><<<148 * 8, 256, smem, s>>>(p, out, radius);
  return cudaGetLastError();
}
template cudaError_t launch_gam_field<float>(const ApplyParams<float>&, float*, int, cudaStream_t);
template cudaError_t launch_gam_field<double>(const ApplyParams<double>&, double*, int, cudaStream_t);

template <typename R>
cudaError_t launch_sources(const ApplyParams<R>& p, int nsrc, const long long* nodes, const double* amps,
                           int consistent, R ih3, typename Cx<R>::T* b, cudaStream_t s) {
  const size_t smem = (size_t)p.n_g * TAB_STRIDE * sizeof(R);
  cudaFuncSetAttribute(sources_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int nt = nsrc * 27;
  sources_kernel<R><<<(nt + 255) / 256, 256, smem, s>>>(p, nsrc, nodes, amps, consistent, ih3, b);
  return cudaGetLastError();
}
template cudaError_t launch_sources<float>(const ApplyParams<float>&, int, const long long*, const double*, int, float,
                                           float2*, cudaStream_t);
template cudaError_t launch_sources<double>(const ApplyParams<double>&, int, const long long*, const double*, int,
                                            double, double2*, cudaStream_t);

template <typename R>
cudaError_t launch_vstats(const R* v, long long n, int nx, int ldx, R inv_fh, R g_min, R g_max, unsigned long long* out,
                          cudaStream_t s) {
  vstats_kernel<R><<<592, 256, 0, s>>>(v, n, nx, ldx, inv_fh, g_min, g_max, out);
  return cudaGetLastError();
}
template cudaError_t launch_vstats<float>(const float*, long long, int, int, float, float, float, unsigned long long*,
                                          cudaStream_t);
template cudaError_t launch_vstats<double>(const double*, long long, int, int, double, double, double, unsigned long long*,
                                           cudaStream_t);

// =============================================================================================
// loopback communicator (P slabs in one process on one device): out[i] = op over the P ranks' buffers
// in rank order (sum or max) — the device half of its allreduce
// =============================================================================================
__global__ void loop_reduce_kernel(LoopPtrs ptrs, int np, double* __restrict__ out, long long n, int op) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double a = ptrs.p[0][i];
    for (int q = 1; q < np; q++) a = op == 0 ? a + ptrs.p[q][i] : fmax(a, ptrs.p[q][i]);
    out[i] = a;
  }
}
cudaError_t launch_loop_reduce(const LoopPtrs& ptrs, int np, double* out, long long n, int op, cudaStream_t s) {
  const int nb = (int)std::min<long long>(148, (n + 255) / 256);
  loop_reduce_kernel<<<nb > 0 ? nb : 1, 256, 0, s>>>(ptrs, np, out, n, op);
  return cudaGetLastError();
}

constexpr int VEC_NT = 256;

template <typename R>
cudaError_t launch_bicg(int which, const VecParams<R>& q, int nrhs, cudaStream_t s) {
  dim3 grid((unsigned)q.nblocks, (unsigned)nrhs);
  switch (which) {
    case BICG_INIT: bicg_init_kernel<R><<<grid, VEC_NT, 0, s>>>(q); break;
    case BICG_S: bicg_s_kernel<R><<<grid, VEC_NT, 0, s>>>(q); break;
    case BICG_UPDATE: bicg_update_kernel<R, VEC_NT><<<grid, VEC_NT, 0, s>>>(q); break;
    case BICG_RHO_RESET: bicg_rho_reset_kernel<<<(nrhs + 127) / 128, 128, 0, s>>>(q.dotR, q.state, q.active, nrhs); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}
template cudaError_t launch_bicg<float>(int, const VecParams<float>&, int, cudaStream_t);
template cudaError_t launch_bicg<double>(int, const VecParams<double>&, int, cudaStream_t);

template <typename R>
cudaError_t launch_bicgl(int which, const VecParams<R>& q, int nrhs, cudaStream_t s) {
  dim3 grid((unsigned)q.nblocks, (unsigned)nrhs);
  switch (which) {
    case BCL_INIT: bicgl_kernel<R, VEC_NT, BCL_INIT><<<grid, VEC_NT, 0, s>>>(q); break;
    case BCL_A: bicgl_kernel<R, VEC_NT, BCL_A><<<grid, VEC_NT, 0, s>>>(q); break;
    case BCL_B: bicgl_kernel<R, VEC_NT, BCL_B><<<grid, VEC_NT, 0, s>>>(q); break;
    case BCL_C: bicgl_kernel<R, VEC_NT, BCL_C><<<grid, VEC_NT, 0, s>>>(q); break;
    case BCL_D: bicgl_kernel<R, VEC_NT, BCL_D><<<grid, VEC_NT, 0, s>>>(q); break;
    case BCL_E: bicgl_kernel<R, VEC_NT, BCL_E><<<grid, VEC_NT, 0, s>>>(q); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}
template cudaError_t launch_bicgl<float>(int, const VecParams<float>&, int, cudaStream_t);
template cudaError_t launch_bicgl<double>(int, const VecParams<double>&, int, cudaStream_t);

template <typename R>
cudaError_t launch_norm2(const typename Cx<R>::T* f, long long fstride, long long plane, long long n, int nx, int ldx,
                         int nrhs, int nblocks, double* partials, double* out, unsigned int* tickets, cudaStream_t s) {
  dim3 grid((unsigned)nblocks, (unsigned)nrhs);
  norm2_kernel<R, VEC_NT><<<grid, VEC_NT, 0, s>>>(f, fstride, plane, n, nx, ldx, partials, out, tickets);
  return cudaGetLastError();
}
template cudaError_t launch_norm2<float>(const float2*, long long, long long, long long, int, int, int, int, double*,
                                         double*, unsigned int*, cudaStream_t);
template cudaError_t launch_norm2<double>(const double2*, long long, long long, long long, int, int, int, int, double*,
                                          double*, unsigned int*, cudaStream_t);

}  // namespace hz
