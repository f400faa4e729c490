// NEXT-3: the convergent Born series (CBS) reference wavefield on the GPU (the paper's
// heterogeneous-model references, "highly-accurate Convergent Born Series (CBS) method", stopped at
// a backward error of 1e-12; the construction of the cited method restated in oracle/cbs.py and
// DESIGN.md reading A26).  complex128 throughout.
//
//   box:   the model padded by `pad` cells per side; k² = (ω/v_nearest)² + i·a·k0²·Σ_axes (d_a/pad)²
//   k0² = ½(min + max) Re k²,  ε = 1.05·max|k² − k0²| (≥ 1e-3 k0²),  V = k² − k0² − iε,  γ = (i/ε) V
//   G:     Fourier symbol 1/(|p|² − k0² − iε), p = 2π·fftfreq(n, h) per axis (cuFFT Z2Z, 3-D)
//   iteration (u₀ = 0):  t = V u − s;  t ← G t;  u ← u − γ (u − t)
//   backward error every check_every iterations: ‖IFFT(−|p|² FFT u) + k² u − s‖ / ‖s‖
//
// Kernels (HBM-bound pointwise passes between the FFTs): cbs_step (update u from t and form the next
// t = V u in one pass: 80 B/pt), cbs_green (t *= G/N on the spectrum: 32 B/pt), cbs_lap (r *= −|p|²/N),
// cbs_resid (r += k² u, 48 B/pt), point-source scatter, deterministic fp64 norm (block partials, one
// final block in fixed order), the box k² build and its min / max reductions.
#include <cuda_runtime.h>
#include <cufft.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "hz_internal.h"

namespace hz {
namespace {

struct Box {
  int nx, ny, nz, pad;
  int Nx, Ny, Nz;
  long long N;
};

__device__ __forceinline__ double2 cmul2(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__device__ __forceinline__ void box_index(const Box& d, long long i, int& X, int& Y, int& Z) {
  X = (int)(i % d.Nx);
  const long long t = i / d.Nx;
  Y = (int)(t % d.Ny);
  Z = (int)(t / d.Ny);
}

// cells into the padding along one axis
__device__ __forceinline__ double pad_dist(int I, int n, int pad) {
  return (double)max(0, max(pad - I, I - (pad + n - 1)));
}

// |p|² at spectral index (X, Y, Z): p = 2π·fftfreq(N, h)
__device__ __forceinline__ double p2_of(const Box& d, int X, int Y, int Z, double twopi_h) {
  const int fx = X < (d.Nx + 1) / 2 ? X : X - d.Nx;
  const int fy = Y < (d.Ny + 1) / 2 ? Y : Y - d.Ny;
  const int fz = Z < (d.Nz + 1) / 2 ? Z : Z - d.Nz;
  const double px = twopi_h * fx / d.Nx, py = twopi_h * fy / d.Ny, pz = twopi_h * fz / d.Nz;
  return px * px + py * py + pz * pz;
}

__global__ void cbs_k2_kernel(const double* __restrict__ v, Box d, double omega, double ak0, double2* __restrict__ k2) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.N) return;
  int X, Y, Z;
  box_index(d, i, X, Y, Z);
  const int x = min(max(X - d.pad, 0), d.nx - 1), y = min(max(Y - d.pad, 0), d.ny - 1), z = min(max(Z - d.pad, 0), d.nz - 1);
  const double vv = v[((long long)z * d.ny + y) * d.nx + x];
  const double kr = omega / vv;
  double a = 0.0;
  if (d.pad > 0) {
    const double ex = pad_dist(X, d.nx, d.pad) / d.pad, ey = pad_dist(Y, d.ny, d.pad) / d.pad, ez = pad_dist(Z, d.nz, d.pad) / d.pad;
    a = ak0 * (ex * ex + ey * ey + ez * ez);
  }
  k2[i] = make_double2(kr * kr, a);
}

// max of non-negative doubles through their bit patterns (monotone for x ≥ 0)
__device__ __forceinline__ void atomic_max_pos(unsigned long long* m, double x) {
  atomicMax(m, (unsigned long long)__double_as_longlong(x));
}

// per-block reduction of (min v, max v) of the model, or max |k² − k0²| over the box
__global__ void cbs_vrange_kernel(const double* __restrict__ v, long long n, unsigned long long* out) {
  __shared__ double smin[256], smax[256];
  double lo = HUGE_VAL, hi = 0.0;
  unsigned long long bad = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double x = v[i];
    if (!(x > 0.0) || !isfinite(x)) {
      bad++;
      continue;
    }
    lo = fmin(lo, x);
    hi = fmax(hi, x);
  }
  if (bad) atomicAdd(out + 3, bad);
  smin[threadIdx.x] = lo;
  smax[threadIdx.x] = hi;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      smin[threadIdx.x] = fmin(smin[threadIdx.x], smin[threadIdx.x + o]);
      smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    atomicMin(out, (unsigned long long)__double_as_longlong(smin[0]));
    atomic_max_pos(out + 1, smax[0]);
  }
}
__global__ void cbs_epsmax_kernel(const double2* __restrict__ k2, long long n, double k0sq, unsigned long long* out) {
  __shared__ double s[256];
  double hi = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double2 a = k2[i];
    hi = fmax(hi, hypot(a.x - k0sq, a.y));
  }
  s[threadIdx.x] = hi;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] = fmax(s[threadIdx.x], s[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) atomic_max_pos(out, s[0]);
}

// t = V u with V = k² − k0² − iε (the first iteration's t from u₀ = 0 is just −s)
// fused update: u ← u − γ (u − t), then t = V u (the sources are subtracted by cbs_src)
__global__ void cbs_step_kernel(double2* __restrict__ u, double2* __restrict__ t, const double2* __restrict__ k2, long long n,
                                double k0sq, double eps, int first) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 kk = k2[i];
  const double2 V = make_double2(kk.x - k0sq, kk.y - eps);
  double2 uu = u[i];
  if (!first) {
    const double2 g = make_double2(-V.y / eps, V.x / eps);   // γ = (i/ε) V
    const double2 tt = t[i];
    const double2 d = make_double2(uu.x - tt.x, uu.y - tt.y);
    const double2 gd = cmul2(g, d);
    uu = make_double2(uu.x - gd.x, uu.y - gd.y);
    u[i] = uu;
  }
  t[i] = cmul2(V, uu);
}
// last update only (no next t)
__global__ void cbs_update_kernel(double2* __restrict__ u, const double2* __restrict__ t, const double2* __restrict__ k2, long long n,
                                  double k0sq, double eps) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 kk = k2[i];
  const double2 g = make_double2(-(kk.y - eps) / eps, (kk.x - k0sq) / eps);
  const double2 uu = u[i], tt = t[i];
  const double2 gd = cmul2(g, make_double2(uu.x - tt.x, uu.y - tt.y));
  u[i] = make_double2(uu.x - gd.x, uu.y - gd.y);
}
// f[src] −= s (point sources: box index and value amp/h³)
__global__ void cbs_src_kernel(double2* __restrict__ f, const long long* __restrict__ idx, const double2* __restrict__ val, int ns) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= ns) return;
  double2* p = f + idx[k];
  p->x -= val[k].x;
  p->y -= val[k].y;
}
// t ← t·G/N on the spectrum
__global__ void cbs_green_kernel(double2* __restrict__ t, Box d, double twopi_h, double k0sq, double eps) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.N) return;
  int X, Y, Z;
  box_index(d, i, X, Y, Z);
  const double a = p2_of(d, X, Y, Z, twopi_h) - k0sq;   // 1/(a − iε) = (a + iε)/(a² + ε²)
  const double den = (a * a + eps * eps) * (double)d.N;
  const double2 g = make_double2(a / den, eps / den);
  t[i] = cmul2(g, t[i]);
}
// r ← r·(−|p|²)/N on the spectrum
__global__ void cbs_lap_kernel(double2* __restrict__ r, Box d, double twopi_h) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.N) return;
  int X, Y, Z;
  box_index(d, i, X, Y, Z);
  const double s = -p2_of(d, X, Y, Z, twopi_h) / (double)d.N;
  const double2 a = r[i];
  r[i] = make_double2(s * a.x, s * a.y);
}
// r ← r + k² u
__global__ void cbs_resid_kernel(double2* __restrict__ r, const double2* __restrict__ u, const double2* __restrict__ k2, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 a = r[i], ku = cmul2(k2[i], u[i]);
  r[i] = make_double2(a.x + ku.x, a.y + ku.y);
}
// ‖r‖²: fixed-order block partials, then one block sums them in order
__global__ void cbs_norm_partial_kernel(const double2* __restrict__ r, long long n, double* __restrict__ part) {
  __shared__ double s[256];
  double acc = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double2 a = r[i];
    acc = fma(a.x, a.x, fma(a.y, a.y, acc));
  }
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = s[0];
}
__global__ void cbs_norm_final_kernel(const double* __restrict__ part, int nb, double* __restrict__ out) {
  __shared__ double s[256];
  double acc = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) acc += part[i];
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0];
}
// model region of the box field → dense [nz][ny][nx]
__global__ void cbs_extract_kernel(const double2* __restrict__ u, Box d, double2* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long n = (long long)d.nx * d.ny * d.nz;
  if (i >= n) return;
  const int x = (int)(i % d.nx);
  const long long t = i / d.nx;
  const int y = (int)(t % d.ny), z = (int)(t / d.ny);
  out[i] = u[((long long)(z + d.pad) * d.Ny + (y + d.pad)) * d.Nx + (x + d.pad)];
}

struct DevMem {
  std::vector<void*> ptrs;
  ~DevMem() {
    for (void* p : ptrs) cudaFree(p);
  }
  template <typename T> cudaError_t get(T** p, size_t n) {
    void* q = nullptr;
    cudaError_t e = cudaMalloc(&q, n * sizeof(T));
    if (e == cudaSuccess) ptrs.push_back(q);
    *p = reinterpret_cast<T*>(q);
    return e;
  }
};
struct Plan {
  cufftHandle h = 0;
  bool ok = false;
  ~Plan() {
    if (ok) cufftDestroy(h);
  }
};

}  // namespace
}  // namespace hz

using namespace hz;

#define CBS_CUDA(x)                                                                      \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess) {                                                             \
      set_error(std::string("hz_cbs_solve: ") + cudaGetErrorString(e_));                 \
      return e_ == cudaErrorMemoryAllocation ? HZ_ERR_OOM : HZ_ERR_CUDA;                  \
    }                                                                                    \
  } while (0)
#define CBS_FFT(x)                                                                       \
  do {                                                                                   \
    cufftResult r_ = (x);                                                                \
    if (r_ != CUFFT_SUCCESS) {                                                           \
      set_error("hz_cbs_solve: cuFFT error " + std::to_string((int)r_));                 \
      return HZ_ERR_CUDA;                                                                \
    }                                                                                    \
  } while (0)

extern "C" hz_cbs_opts hz_cbs_opts_default(void) {
  hz_cbs_opts o;
  o.pad = -1;          // two of the longest wavelengths
  o.absorb = 1.0;
  o.tol = 1e-12;
  o.max_iter = 200000;
  o.check_every = 20;
  return o;
}

extern "C" hz_status hz_cbs_solve(hz_ctx* ctx, int nx, int ny, int nz, double h, const double* v, double freq, int nsrc,
                                  const long long* src_xyz, const double* amps, const hz_cbs_opts* opts, double* u_out,
                                  hz_cbs_stats* stats, void* stream) {
  if (!ctx || !v || !u_out || !src_xyz || nsrc < 1 || nx < 1 || ny < 1 || nz < 1) {
    set_error("hz_cbs_solve: bad arguments");
    return HZ_ERR_INVALID_ARG;
  }
  if (!(h > 0) || !(freq > 0)) {
    set_error("hz_cbs_solve: h and freq must be positive");
    return HZ_ERR_DOMAIN;
  }
  const hz_cbs_opts o = opts ? *opts : hz_cbs_opts_default();
  if (!(o.tol > 0) || o.max_iter < 1 || o.check_every < 1 || o.absorb < 0) {
    set_error("hz_cbs_solve: bad options");
    return HZ_ERR_INVALID_ARG;
  }
  CBS_CUDA(cudaSetDevice(ctx_device(ctx)));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const auto t0 = std::chrono::steady_clock::now();
  const long long nm = (long long)nx * ny * nz;
  DevMem mem;
  // the model on the device
  const double* vd = v;
  if (!device_pointer(v)) {
    double* tmp = nullptr;
    CBS_CUDA(mem.get(&tmp, (size_t)nm));
    CBS_CUDA(cudaMemcpyAsync(tmp, v, sizeof(double) * nm, cudaMemcpyHostToDevice, s));
    vd = tmp;
  }
  unsigned long long* red = nullptr;
  CBS_CUDA(mem.get(&red, 4));
  auto bits = [](double x) {
    unsigned long long b;
    std::memcpy(&b, &x, sizeof(b));
    return b;
  };
  auto dbl = [](unsigned long long b) {
    double x;
    std::memcpy(&x, &b, sizeof(x));
    return x;
  };
  const unsigned long long init[4] = {bits(HUGE_VAL), 0ull, 0ull, 0ull};   // min v, max v, max|k²−k0²|, invalid v
  CBS_CUDA(cudaMemcpyAsync(red, init, sizeof(init), cudaMemcpyHostToDevice, s));
  cbs_vrange_kernel<<<296, 256, 0, s>>>(vd, nm, red);
  CBS_CUDA(cudaGetLastError());
  unsigned long long hr[4];
  CBS_CUDA(cudaMemcpyAsync(hr, red, sizeof(hr), cudaMemcpyDeviceToHost, s));
  CBS_CUDA(cudaStreamSynchronize(s));
  const double vmin = dbl(hr[0]), vmax = dbl(hr[1]);
  if (hr[3] != 0 || !(vmin > 0) || !std::isfinite(vmax)) {
    set_error("hz_cbs_solve: velocities must be positive and finite");
    return HZ_ERR_DOMAIN;
  }
  const double omega = 2.0 * M_PI * freq;
  const int pad = o.pad >= 0 ? o.pad : (int)std::ceil(2.0 * vmax / (freq * h));
  Box d{nx, ny, nz, pad, nx + 2 * pad, ny + 2 * pad, nz + 2 * pad, 0};
  d.N = (long long)d.Nx * d.Ny * d.Nz;
  for (int k = 0; k < nsrc; k++) {
    const long long* q = src_xyz + 3 * k;
    if (q[0] < 0 || q[0] >= nx || q[1] < 0 || q[1] >= ny || q[2] < 0 || q[2] >= nz) {
      set_error("hz_cbs_solve: source outside the model");
      return HZ_ERR_INVALID_ARG;
    }
  }
  const double k0sq = 0.5 * ((omega / vmax) * (omega / vmax) + (omega / vmin) * (omega / vmin));
  double2 *k2 = nullptr, *u = nullptr, *t = nullptr, *r = nullptr, *sv = nullptr;
  long long* si = nullptr;
  CBS_CUDA(mem.get(&k2, (size_t)d.N));
  CBS_CUDA(mem.get(&u, (size_t)d.N));
  CBS_CUDA(mem.get(&t, (size_t)d.N));
  CBS_CUDA(mem.get(&r, (size_t)d.N));
  CBS_CUDA(mem.get(&sv, (size_t)nsrc));
  CBS_CUDA(mem.get(&si, (size_t)nsrc));
  const int TB = 256;
  const unsigned nbN = (unsigned)((d.N + TB - 1) / TB);
  long long launches = 1;
  cbs_k2_kernel<<<nbN, TB, 0, s>>>(vd, d, omega, o.absorb * k0sq, k2);
  cbs_epsmax_kernel<<<296, 256, 0, s>>>(k2, d.N, k0sq, red + 2);
  launches += 2;
  CBS_CUDA(cudaGetLastError());
  CBS_CUDA(cudaMemcpyAsync(hr, red, sizeof(hr), cudaMemcpyDeviceToHost, s));
  CBS_CUDA(cudaStreamSynchronize(s));
  const double eps = std::max(1.05 * dbl(hr[2]), 1e-3 * k0sq);
  // sources: s = amp/h³ at the box node; ‖s‖ from the merged sources
  std::vector<long long> hidx(nsrc);
  std::vector<double2> hval(nsrc);
  std::vector<std::pair<long long, double2>> merged;
  const double ih3 = 1.0 / (h * h * h);
  for (int k = 0; k < nsrc; k++) {
    const long long* q = src_xyz + 3 * k;
    hidx[k] = ((q[2] + pad) * d.Ny + (q[1] + pad)) * (long long)d.Nx + (q[0] + pad);
    hval[k] = make_double2((amps ? amps[2 * k] : 1.0) * ih3, (amps ? amps[2 * k + 1] : 0.0) * ih3);
    bool found = false;
    for (auto& m : merged)
      if (m.first == hidx[k]) { m.second.x += hval[k].x; m.second.y += hval[k].y; found = true; }
    if (!found) merged.push_back({hidx[k], hval[k]});
  }
  double s2 = 0.0;
  for (auto& m : merged) s2 += m.second.x * m.second.x + m.second.y * m.second.y;
  if (!(s2 > 0)) {
    set_error("hz_cbs_solve: zero source");
    return HZ_ERR_INVALID_ARG;
  }
  CBS_CUDA(cudaMemcpyAsync(si, hidx.data(), sizeof(long long) * nsrc, cudaMemcpyHostToDevice, s));
  CBS_CUDA(cudaMemcpyAsync(sv, hval.data(), sizeof(double2) * nsrc, cudaMemcpyHostToDevice, s));
  CBS_CUDA(cudaMemsetAsync(u, 0, sizeof(double2) * d.N, s));
  // cuFFT plan of the box (C order: Nz slowest)
  Plan plan;
  CBS_FFT(cufftPlan3d(&plan.h, d.Nz, d.Ny, d.Nx, CUFFT_Z2Z));
  plan.ok = true;
  CBS_FFT(cufftSetStream(plan.h, s));
  const int NB = 592;
  double *part = nullptr, *nrm = nullptr;
  CBS_CUDA(mem.get(&part, NB));
  CBS_CUDA(mem.get(&nrm, 1));
  const double twopi_h = 2.0 * M_PI / h;
  const unsigned nbs = (unsigned)((nsrc + 127) / 128);
  // t = V·0 − s
  cbs_step_kernel<<<nbN, TB, 0, s>>>(u, t, k2, d.N, k0sq, eps, 1);
  cbs_src_kernel<<<nbs, 128, 0, s>>>(t, si, sv, nsrc);
  launches += 2;
  int it = 0;
  double be = HUGE_VAL;
  hz_status status = HZ_NOT_CONVERGED;
  while (it < o.max_iter) {
    CBS_FFT(cufftExecZ2Z(plan.h, reinterpret_cast<cufftDoubleComplex*>(t), reinterpret_cast<cufftDoubleComplex*>(t), CUFFT_FORWARD));
    cbs_green_kernel<<<nbN, TB, 0, s>>>(t, d, twopi_h, k0sq, eps);
    CBS_FFT(cufftExecZ2Z(plan.h, reinterpret_cast<cufftDoubleComplex*>(t), reinterpret_cast<cufftDoubleComplex*>(t), CUFFT_INVERSE));
    it++;
    launches += 1;
    const bool check = it % o.check_every == 0 || it == o.max_iter;
    if (!check) {   // u ← u − γ(u − t) and the next t = V u − s in one pass
      cbs_step_kernel<<<nbN, TB, 0, s>>>(u, t, k2, d.N, k0sq, eps, 0);
      cbs_src_kernel<<<nbs, 128, 0, s>>>(t, si, sv, nsrc);
      launches += 2;
      continue;
    }
    cbs_update_kernel<<<nbN, TB, 0, s>>>(u, t, k2, d.N, k0sq, eps);
    // backward error: r = ∇²u + k²u − s
    CBS_CUDA(cudaMemcpyAsync(r, u, sizeof(double2) * d.N, cudaMemcpyDeviceToDevice, s));
    CBS_FFT(cufftExecZ2Z(plan.h, reinterpret_cast<cufftDoubleComplex*>(r), reinterpret_cast<cufftDoubleComplex*>(r), CUFFT_FORWARD));
    cbs_lap_kernel<<<nbN, TB, 0, s>>>(r, d, twopi_h);
    CBS_FFT(cufftExecZ2Z(plan.h, reinterpret_cast<cufftDoubleComplex*>(r), reinterpret_cast<cufftDoubleComplex*>(r), CUFFT_INVERSE));
    cbs_resid_kernel<<<nbN, TB, 0, s>>>(r, u, k2, d.N);
    cbs_src_kernel<<<nbs, 128, 0, s>>>(r, si, sv, nsrc);
    cbs_norm_partial_kernel<<<NB, 256, 0, s>>>(r, d.N, part);
    cbs_norm_final_kernel<<<1, 256, 0, s>>>(part, NB, nrm);
    launches += 7;
    CBS_CUDA(cudaGetLastError());
    double r2 = 0.0;
    CBS_CUDA(cudaMemcpyAsync(&r2, nrm, sizeof(double), cudaMemcpyDeviceToHost, s));
    CBS_CUDA(cudaStreamSynchronize(s));
    be = std::sqrt(r2 / s2);
    if (!std::isfinite(be)) {
      set_error("hz_cbs_solve: iteration diverged");
      return HZ_ERR_CUDA;
    }
    if (be <= o.tol) {
      status = HZ_OK;
      break;
    }
    if (it < o.max_iter) {   // the next t from the updated u
      cbs_step_kernel<<<nbN, TB, 0, s>>>(u, t, k2, d.N, k0sq, eps, 1);
      cbs_src_kernel<<<nbs, 128, 0, s>>>(t, si, sv, nsrc);
      launches += 2;
    }
  }
  // the model region out
  double2* ud = nullptr;
  const bool dev_out = device_pointer(u_out);
  if (dev_out) {
    ud = reinterpret_cast<double2*>(u_out);
  } else {
    CBS_CUDA(mem.get(&ud, (size_t)nm));
  }
  cbs_extract_kernel<<<(unsigned)((nm + TB - 1) / TB), TB, 0, s>>>(u, d, ud);
  launches++;
  CBS_CUDA(cudaGetLastError());
  if (!dev_out) CBS_CUDA(cudaMemcpyAsync(u_out, ud, sizeof(double2) * nm, cudaMemcpyDeviceToHost, s));
  CBS_CUDA(cudaStreamSynchronize(s));
  add_launches(launches);
  if (stats) {
    stats->iterations = it;
    stats->backward_error = be;
    stats->k0sq = k0sq;
    stats->eps = eps;
    stats->box[0] = d.Nx;
    stats->box[1] = d.Ny;
    stats->box[2] = d.Nz;
    stats->pad = pad;
    stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  return status;
}
