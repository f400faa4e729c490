// NEXT-4 (preconditioned solve): a complex shifted-Laplacian multigrid preconditioner for the
// complex64 BiCGSTAB (hz_solve_opts.precond = 1; reading A27 in DESIGN.md).
//
//   M = ∇²_h,PML + (1 + iβ) ω² / v²,  β = 0.5
// on each level with the per-axis stretched second differences of reading A8 (a± = 1/(H² ξ(i) ξ(i ± ½)),
// ξ evaluated at the fine-grid positions of the coarse nodes), approximately inverted by one V-cycle:
// damped Jacobi (ω_J = 0.8, one pre- and one post-sweep), full-weighting restriction, trilinear
// prolongation, vertex-centred coarsening n_c = ⌊n/2⌋ + 1 down to a few points per dimension, and
// 16 Jacobi sweeps on the coarsest level (where k²H² ≫ 1 makes Jacobi converge).  The damping β keeps M invertible
// and the coarse problems smoothable (the CSL preconditioner of the Helmholtz literature, the
// "iterative route" the paper contrasts with its direct solver).
//
// Layout: level 0 reads / writes the solver's fields ([nrhs][nz+2][ny][ldx], one halo plane: single
// slab only); coarse levels are dense [nrhs][nz][ny][nx].  complex64.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <vector>

#include "hz_internal.h"
#include "kernels.h"

namespace hz {
namespace {

struct Lvl {
  int nx, ny, nz;
  long long ldx, plane, off, fstride;
  const float* w;                  // 1/v² at the level's nodes (same layout, first field)
  const float2* am[3];
  const float2* ap[3];
  float2 shift;                    // (1 + iβ) ω²
};

__device__ __forceinline__ float2 c_mul(float2 a, float2 b) { return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ float2 c_add(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 c_sub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 c_div(float2 a, float2 b) {
  const float d = b.x * b.x + b.y * b.y;
  return make_float2((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}

__device__ __forceinline__ long long lidx(const Lvl& L, int x, int y, int z) { return L.off + z * L.plane + y * L.ldx + x; }

// the diagonal D of M at one node: (1 + iβ) ω² w − Σ_axes (a⁻ + a⁺)
__device__ __forceinline__ float2 diag_m(const Lvl& L, int x, int y, int z) {
  const float wk = L.w[lidx(L, x, y, z)];
  const float2 k2 = make_float2(L.shift.x * wk, L.shift.y * wk);
  const float2 sa = c_add(c_add(c_add(L.am[0][x], L.ap[0][x]), c_add(L.am[1][y], L.ap[1][y])), c_add(L.am[2][z], L.ap[2][z]));
  return c_sub(k2, sa);
}
// (M e)(x,y,z) (e: this RHS's field; out-of-grid neighbours are 0) and the diagonal D
__device__ __forceinline__ void apply_m(const Lvl& L, const float2* __restrict__ e, int x, int y, int z, float2& Me, float2& D) {
  const long long i = lidx(L, x, y, z);
  const float2 c = e[i];
  const float2 z2 = make_float2(0.f, 0.f);
  const float2 xm = x > 0 ? e[i - 1] : z2, xp = x + 1 < L.nx ? e[i + 1] : z2;
  const float2 ym = y > 0 ? e[i - L.ldx] : z2, yp = y + 1 < L.ny ? e[i + L.ldx] : z2;
  const float2 zm = z > 0 ? e[i - L.plane] : z2, zp = z + 1 < L.nz ? e[i + L.plane] : z2;
  const float wk = L.w[i];
  const float2 k2 = make_float2(L.shift.x * wk, L.shift.y * wk);
  Me = c_mul(k2, c);
  Me = c_add(Me, c_mul(L.am[0][x], c_sub(xm, c)));
  Me = c_add(Me, c_mul(L.ap[0][x], c_sub(xp, c)));
  Me = c_add(Me, c_mul(L.am[1][y], c_sub(ym, c)));
  Me = c_add(Me, c_mul(L.ap[1][y], c_sub(yp, c)));
  Me = c_add(Me, c_mul(L.am[2][z], c_sub(zm, c)));
  Me = c_add(Me, c_mul(L.ap[2][z], c_sub(zp, c)));
  D = diag_m(L, x, y, z);
}

__device__ __forceinline__ bool node_of(const Lvl& L, long long t, int& x, int& y, int& z) {
  const long long n = (long long)L.nx * L.ny * L.nz;
  if (t >= n) return false;
  x = (int)(t % L.nx);
  const long long q = t / L.nx;
  y = (int)(q % L.ny);
  z = (int)(q / L.ny);
  return true;
}

// e_out = e_in + ω_J (f − M e_in)/D; first: e_in = 0
__global__ void mg_jacobi_kernel(Lvl L, const float2* __restrict__ ein, const float2* __restrict__ f, float2* __restrict__ eout,
                                 float wj, int first, const int* __restrict__ active) {
  const int r = blockIdx.y;
  if (active && active[r] == 0) return;
  int x, y, z;
  if (!node_of(L, (long long)blockIdx.x * blockDim.x + threadIdx.x, x, y, z)) return;
  const long long ro = (long long)r * L.fstride, i = lidx(L, x, y, z);
  float2 Me, D;
  if (first) {   // from e = 0: ω_J f / D
    const float2 q = c_div(f[ro + i], diag_m(L, x, y, z));
    eout[ro + i] = make_float2(wj * q.x, wj * q.y);
    return;
  }
  apply_m(L, ein + ro, x, y, z, Me, D);
  const float2 q = c_div(c_sub(f[ro + i], Me), D);
  const float2 c = ein[ro + i];
  eout[ro + i] = make_float2(c.x + wj * q.x, c.y + wj * q.y);
}
// r = f − M e
__global__ void mg_resid_kernel(Lvl L, const float2* __restrict__ e, const float2* __restrict__ f, float2* __restrict__ res,
                                const int* __restrict__ active) {
  const int r = blockIdx.y;
  if (active && active[r] == 0) return;
  int x, y, z;
  if (!node_of(L, (long long)blockIdx.x * blockDim.x + threadIdx.x, x, y, z)) return;
  const long long ro = (long long)r * L.fstride, i = lidx(L, x, y, z);
  float2 Me, D;
  apply_m(L, e + ro, x, y, z, Me, D);
  res[ro + i] = c_sub(f[ro + i], Me);
}
// coarse f = full weighting of the fine residual (1-D weights ¼ ½ ¼ per axis; out-of-grid = 0)
__global__ void mg_restrict_kernel(Lvl F, const float2* __restrict__ rf, Lvl C, float2* __restrict__ fc, const int* __restrict__ active) {
  const int r = blockIdx.y;
  if (active && active[r] == 0) return;
  int X, Y, Z;
  if (!node_of(C, (long long)blockIdx.x * blockDim.x + threadIdx.x, X, Y, Z)) return;
  const long long rof = (long long)r * F.fstride;
  float2 acc = make_float2(0.f, 0.f);
  for (int dz = -1; dz <= 1; dz++) {
    const int z = 2 * Z + dz;
    if (z < 0 || z >= F.nz) continue;
    const float wz = dz == 0 ? 0.5f : 0.25f;
    for (int dy = -1; dy <= 1; dy++) {
      const int y = 2 * Y + dy;
      if (y < 0 || y >= F.ny) continue;
      const float wy = wz * (dy == 0 ? 0.5f : 0.25f);
      for (int dx = -1; dx <= 1; dx++) {
        const int x = 2 * X + dx;
        if (x < 0 || x >= F.nx) continue;
        const float ww = wy * (dx == 0 ? 0.5f : 0.25f);
        const float2 v = rf[rof + lidx(F, x, y, z)];
        acc.x += ww * v.x;
        acc.y += ww * v.y;
      }
    }
  }
  fc[(long long)r * C.fstride + lidx(C, X, Y, Z)] = acc;
}
// fine e += trilinear interpolation of the coarse correction
__global__ void mg_prolong_kernel(Lvl C, const float2* __restrict__ ec, Lvl F, float2* __restrict__ ef, const int* __restrict__ active) {
  const int r = blockIdx.y;
  if (active && active[r] == 0) return;
  int x, y, z;
  if (!node_of(F, (long long)blockIdx.x * blockDim.x + threadIdx.x, x, y, z)) return;
  const long long roc = (long long)r * C.fstride;
  const int X0 = x >> 1, Y0 = y >> 1, Z0 = z >> 1;
  const int nX = (x & 1) ? 2 : 1, nY = (y & 1) ? 2 : 1, nZ = (z & 1) ? 2 : 1;
  const float fx = (x & 1) ? 0.5f : 1.f, fy = (y & 1) ? 0.5f : 1.f, fz = (z & 1) ? 0.5f : 1.f;
  float2 acc = make_float2(0.f, 0.f);
  for (int a = 0; a < nZ; a++) {
    const int Z = Z0 + a;
    if (Z >= C.nz) continue;
    for (int b = 0; b < nY; b++) {
      const int Y = Y0 + b;
      if (Y >= C.ny) continue;
      for (int c = 0; c < nX; c++) {
        const int X = X0 + c;
        if (X >= C.nx) continue;
        const float2 v = ec[roc + lidx(C, X, Y, Z)];
        const float ww = fx * fy * fz;
        acc.x += ww * v.x;
        acc.y += ww * v.y;
      }
    }
  }
  const long long i = (long long)r * F.fstride + lidx(F, x, y, z);
  const float2 o = ef[i];
  ef[i] = make_float2(o.x + acc.x, o.y + acc.y);
}
// coarse w by injection
__global__ void mg_inject_w_kernel(Lvl F, Lvl C, float* __restrict__ wc) {
  int X, Y, Z;
  if (!node_of(C, (long long)blockIdx.x * blockDim.x + threadIdx.x, X, Y, Z)) return;
  const int x = min(2 * X, F.nx - 1), y = min(2 * Y, F.ny - 1), z = min(2 * Z, F.nz - 1);
  wc[lidx(C, X, Y, Z)] = F.w[lidx(F, x, y, z)];
}

}  // namespace

// smoothing policy per level from κ = k²H² (the damped-Jacobi error factor of a Fourier mode is
// 1 − ω(1 + s/D), s ∈ [−6, 6], D = (1 + iβ)κ − 6: ω_J = 0.8 smooths while κ is small; for κ ≥ 12,
// |6/D| < 1 and ω_J = 1 converges on every mode; in between Jacobi amplifies the smooth modes, so
// those levels only pass the coarse-grid correction through)
enum { MG_FINE = 0, MG_SKIP = 1, MG_MASS = 2 };

struct MgHierarchy {
  std::vector<Lvl> L;
  std::vector<int> mode;
  std::vector<void*> bufs;
  std::vector<float2*> e, t, f, r;   // per level: correction, Jacobi ping-pong, right-hand side, residual
  int nrhs = 0;
  ~MgHierarchy() {
    for (void* p : bufs) cudaFree(p);
  }
};

namespace {
// per-axis stretched coefficients of a level with stride m (reading A8 at the coarse spacing m·h)
void level_axis(int n_fine, int n_c, int m, int npml, double h, double omega, double v_pml, double R, std::vector<float2>& am,
                std::vector<float2>& ap) {
  auto gamma = [&](double s) {
    if (npml <= 0) return 0.0;
    const double Lp = npml * h;
    const double d = h * std::fmax(0.0, std::fmax(npml - s, s - (n_fine - 1 - npml)));
    return 1.5 * v_pml / Lp * std::log(1.0 / R) * (d / Lp) * (d / Lp);
  };
  auto xi = [&](double s) { return std::complex<double>(1.0, gamma(s) / omega); };
  const double H = m * h;
  am.resize(n_c);
  ap.resize(n_c);
  for (int I = 0; I < n_c; I++) {
    const double s = (double)I * m;
    const std::complex<double> a = 1.0 / (H * H * xi(s) * xi(s - 0.5 * m)), b = 1.0 / (H * H * xi(s) * xi(s + 0.5 * m));
    am[I] = make_float2((float)a.real(), (float)a.imag());
    ap[I] = make_float2((float)b.real(), (float)b.imag());
  }
}
}  // namespace

void mg_destroy(MgHierarchy* m) { delete m; }

cudaError_t mg_create(const MgSpec& sp, MgHierarchy** out) {
  *out = nullptr;
  MgHierarchy* m = new MgHierarchy;
  m->nrhs = sp.nrhs;
  auto alloc = [&](size_t bytes, void** p) {
    cudaError_t e = cudaMalloc(p, bytes);
    if (e == cudaSuccess) {
      m->bufs.push_back(*p);
      cudaMemset(*p, 0, bytes);
    }
    return e;
  };
  const float2 shift = make_float2((float)(sp.omega * sp.omega), (float)(sp.beta * sp.omega * sp.omega));
  int nx = sp.nx, ny = sp.ny, nz = sp.nz, stride = 1;
  cudaError_t err = cudaSuccess;
  for (int lev = 0;; lev++) {
    Lvl L;
    L.nx = nx;
    L.ny = ny;
    L.nz = nz;
    if (lev == 0) {
      L.ldx = sp.ldx;
      L.plane = sp.plane;
      L.off = sp.plane;   // one halo plane
      L.fstride = sp.fstride;
      L.w = sp.w;
    } else {
      L.ldx = nx;
      L.plane = (long long)nx * ny;
      L.off = 0;
      L.fstride = (long long)nx * ny * nz;
      void* wp = nullptr;
      if ((err = alloc(sizeof(float) * L.fstride, &wp)) != cudaSuccess) break;
      L.w = reinterpret_cast<float*>(wp);
      const Lvl& F = m->L.back();
      mg_inject_w_kernel<<<(unsigned)((L.fstride + 255) / 256), 256>>>(F, L, reinterpret_cast<float*>(wp));
    }
    std::vector<float2> am, ap;
    const int ns[3] = {nx, ny, nz}, nf[3] = {sp.nx, sp.ny, sp.nz};
    for (int a = 0; a < 3; a++) {
      level_axis(nf[a], ns[a], stride, sp.npml, sp.h, sp.omega, sp.v_pml, sp.r_coeff, am, ap);
      void *pm = nullptr, *pp = nullptr;
      if ((err = alloc(sizeof(float2) * ns[a], &pm)) != cudaSuccess) break;
      if ((err = alloc(sizeof(float2) * ns[a], &pp)) != cudaSuccess) break;
      cudaMemcpy(pm, am.data(), sizeof(float2) * ns[a], cudaMemcpyHostToDevice);
      cudaMemcpy(pp, ap.data(), sizeof(float2) * ns[a], cudaMemcpyHostToDevice);
      L.am[a] = reinterpret_cast<float2*>(pm);
      L.ap[a] = reinterpret_cast<float2*>(pp);
    }
    if (err != cudaSuccess) break;
    L.shift = shift;
    m->L.push_back(L);
    {
      const double H = stride * sp.h;
      const double kmax = sp.omega * H / sp.vmin, kmin = sp.omega * H / sp.vmax;
      const double kap_max = kmax * kmax, kap_min = kmin * kmin;
      // |6/D| < 1 on every mode ⟺ |(1 + iβ)κ − 6| > 6 ⟺ κ > 12/(1 + β²)
      const double kap_mass = 1.1 * 12.0 / (1.0 + sp.beta * sp.beta);
      m->mode.push_back(kap_max <= 2.0 ? MG_FINE : (kap_min >= kap_mass ? MG_MASS : MG_SKIP));
    }
    // buffers: level 0's f / e are the caller's; t and r always; coarse levels all four
    const size_t fb = sizeof(float2) * (size_t)L.fstride * sp.nrhs;
    void *pe = nullptr, *pt = nullptr, *pf = nullptr, *pr = nullptr;
    if (lev > 0) {
      if ((err = alloc(fb, &pe)) != cudaSuccess) break;
      if ((err = alloc(fb, &pf)) != cudaSuccess) break;
    }
    if ((err = alloc(fb, &pt)) != cudaSuccess) break;
    if ((err = alloc(fb, &pr)) != cudaSuccess) break;
    m->e.push_back(reinterpret_cast<float2*>(pe));
    m->t.push_back(reinterpret_cast<float2*>(pt));
    m->f.push_back(reinterpret_cast<float2*>(pf));
    m->r.push_back(reinterpret_cast<float2*>(pr));
    // next level?
    const int cx = nx / 2 + 1, cy = ny / 2 + 1, cz = nz / 2 + 1;
    // coarsen down to a few points per dimension: on the coarsest grids k²H² ≫ 1 and the shifted
    // operator is dominated by (1 + iβ)k², where Jacobi converges; the intermediate levels (k²H² ~ 1-6,
    // where Jacobi amplifies the smooth modes) rely on the coarse-grid correction below them
    if (cx < 4 || cy < 4 || cz < 4 || lev + 1 >= sp.max_levels) break;
    nx = cx;
    ny = cy;
    nz = cz;
    stride *= 2;
  }
  if (err != cudaSuccess) {
    delete m;
    return err;
  }
  err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    delete m;
    return err;
  }
  *out = m;
  return cudaSuccess;
}

int mg_levels(const MgHierarchy* m) { return (int)m->L.size(); }

// e ≈ M⁻¹ f by one V-cycle (level 0 buffers: the caller's f and e)
cudaError_t mg_vcycle(MgHierarchy* m, const float2* f0, float2* e0, int nrhs, const int* active, cudaStream_t s,
                      long long* launches) {
  const int nl = (int)m->L.size();
  auto grid = [&](const Lvl& L) { return dim3((unsigned)(((long long)L.nx * L.ny * L.nz + 255) / 256), (unsigned)nrhs); };
  long long nlaunch = 0;
  auto fb = [&](const Lvl& L) { return sizeof(float2) * (size_t)L.fstride * nrhs; };
  // k Jacobi sweeps with relaxation wj from e = 0 (ping-pong through t; the result ends in e)
  auto sweeps = [&](int l, const float2* f, float2* e, int k, float wj) {
    const Lvl& L = m->L[l];
    float2* a = (k % 2 == 1) ? e : m->t[l];
    float2* b = (k % 2 == 1) ? m->t[l] : e;
    mg_jacobi_kernel<<<grid(L), 256, 0, s>>>(L, b, f, a, wj, 1, active);
    nlaunch++;
    for (int j = 1; j < k; j++) {
      mg_jacobi_kernel<<<grid(L), 256, 0, s>>>(L, a, f, b, wj, 0, active);
      std::swap(a, b);
      nlaunch++;
    }
  };
  // descend
  for (int l = 0; l < nl; l++) {
    const Lvl& L = m->L[l];
    const float2* f = l == 0 ? f0 : m->f[l];
    float2* e = l == 0 ? e0 : m->e[l];
    const int md = m->mode[l];
    if (l == nl - 1) {   // coarsest
      if (md == MG_MASS) sweeps(l, f, e, 8, 1.0f);
      else sweeps(l, f, e, 2, 0.8f);
      break;
    }
    const Lvl& C = m->L[l + 1];
    if (md == MG_SKIP) {   // no smoothing: the coarse problem gets f itself, e starts at 0
      cudaMemsetAsync(e, 0, fb(L), s);
      mg_restrict_kernel<<<grid(C), 256, 0, s>>>(L, f, C, m->f[l + 1], active);
      nlaunch++;
      continue;
    }
    sweeps(l, f, e, md == MG_MASS ? 2 : 1, md == MG_MASS ? 1.0f : 0.8f);
    mg_resid_kernel<<<grid(L), 256, 0, s>>>(L, e, f, m->r[l], active);
    mg_restrict_kernel<<<grid(C), 256, 0, s>>>(L, m->r[l], C, m->f[l + 1], active);
    nlaunch += 2;
  }
  // ascend
  for (int l = nl - 2; l >= 0; l--) {
    const Lvl& L = m->L[l];
    const Lvl& C = m->L[l + 1];
    const float2* f = l == 0 ? f0 : m->f[l];
    float2* e = l == 0 ? e0 : m->e[l];
    const int md = m->mode[l];
    mg_prolong_kernel<<<grid(L), 256, 0, s>>>(C, m->e[l + 1], L, e, active);
    nlaunch++;
    if (md == MG_SKIP) continue;
    const int k = md == MG_MASS ? 2 : 1;
    const float wj = md == MG_MASS ? 1.0f : 0.8f;
    for (int j = 0; j < k; j++) {   // post-smoothing from the corrected e
      mg_jacobi_kernel<<<grid(L), 256, 0, s>>>(L, e, f, m->t[l], wj, 0, active);
      cudaMemcpyAsync(e, m->t[l], fb(L), cudaMemcpyDeviceToDevice, s);
      nlaunch++;
    }
  }
  if (launches) *launches += nlaunch;
  return cudaGetLastError();
}

}  // namespace hz
