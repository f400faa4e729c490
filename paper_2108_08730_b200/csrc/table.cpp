// Host weight-table builder — north-star step (1) build_weight_table(G range, dG, lambda).
//
// Paper: P:145-160 (linearised ṽ = 1 rows H_l, g; H2 corrected per reading A1),
// P:178-187 (per-G blocks H^(i), g^(i), phi outer / theta inner), P:213-237 (block-diagonal H with
// a Tikhonov term lambda ||L w||^2, L = D P).  Readings A2 (unknowns ws1, ws2, mu0, mu1, mu2 in
// per-point mass units), A10 (angles), A11 (first differences without boundary rows), A12.
//
// B200-side design: this is a one-time host computation (361 blocks of 25 x 5).  Instead of a dense
// QR of the 10825 x 1805 stacked matrix we form the block-TRIDIAGONAL normal equations
//   (H_i^T H_i + lambda d_i I) w_i - lambda w_{i-1} - lambda w_{i+1} = H_i^T g_i,
// d_i = number of difference rows touching block i (1 at the ends, 2 inside), and solve them by
// block Gaussian elimination (block Thomas) in 80-bit long double, followed by two steps of
// iterative refinement.  cond(normal) ~ 1.5e10 at lambda = 1e-2, so long double keeps the weights
// accurate to ~1e-9 relative (the oracle uses numpy lstsq on the stacked matrix).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "hz_internal.h"

namespace hz {

typedef long double ld;

namespace {
// One row from the direction cosines' factors (cos φ, sin φ, cos θ, sin θ), evaluated in the same
// order as h_row so that both give bit-identical rows.
void h_row_cs(ld G, ld cphi, ld sphi, ld cth, ld sth, ld H[5], ld* g) {
  const ld pi = 3.141592653589793238462643383279502884L;
  ld a = 2 * pi * cphi * cth / G;
  ld b = 2 * pi * cphi * sth / G;
  ld c = 2 * pi * sphi / G;
  ld ca = cosl(a), cb = cosl(b), cc = cosl(c);
  ld A = ca * cb * cc;
  ld B = ca * cb + ca * cc + cb * cc;
  ld C = ca + cb + cc;
  ld k = 2 * pi * pi / (G * G);
  H[0] = 0.5L * (3 + 3 * A - B - C);                      // H1
  H[1] = 0.5L * (1 + 3 * A - 5 * B / 3 + C / 3);          // H2 with "+1" (reading A1)
  H[2] = k * (A - 1);                                     // H3
  H[3] = k * (6 * A - 2 * C);                             // H4
  H[4] = k * (12 * A - 4 * B);                            // H5
  *g = 0.5L * ((4 * pi * pi / (G * G) + 3) * A - B + C - 3);  // g
}
}  // namespace

void h_row(ld G, ld theta, ld phi, ld H[5], ld* g) { h_row_cs(G, cosl(phi), sinl(phi), cosl(theta), sinl(theta), H, g); }

namespace {

// In-place inverse of a 5x5 matrix (Gauss-Jordan with partial pivoting).  Returns false if singular.
bool inv5(ld M[5][5], ld Inv[5][5]) {
  ld a[5][10];
  for (int i = 0; i < 5; i++)
    for (int j = 0; j < 10; j++) a[i][j] = (j < 5) ? M[i][j] : (j - 5 == i ? 1.0L : 0.0L);
  ld scale = 0;
  for (int i = 0; i < 5; i++)
    for (int j = 0; j < 5; j++) scale = fmaxl(scale, fabsl(M[i][j]));
  for (int col = 0; col < 5; col++) {
    int piv = col;
    for (int r = col + 1; r < 5; r++)
      if (fabsl(a[r][col]) > fabsl(a[piv][col])) piv = r;
    if (fabsl(a[piv][col]) <= 1e-16L * scale) return false;   // rank-deficient (A14)
    if (piv != col)
      for (int j = 0; j < 10; j++) { ld t = a[col][j]; a[col][j] = a[piv][j]; a[piv][j] = t; }
    ld d = a[col][col];
    for (int j = 0; j < 10; j++) a[col][j] /= d;
    for (int r = 0; r < 5; r++)
      if (r != col) {
        ld f = a[r][col];
        if (f != 0)
          for (int j = 0; j < 10; j++) a[r][j] -= f * a[col][j];
      }
  }
  for (int i = 0; i < 5; i++)
    for (int j = 0; j < 5; j++) Inv[i][j] = a[i][j + 5];
  return true;
}

struct BlockSystem {
  int n;
  std::vector<ld> D;   // [n][5][5] diagonal blocks
  ld off;              // off-diagonal blocks are off * I (= -lambda)
  std::vector<ld> rhs; // [n][5]
};

// Block Thomas for D_i w_i + off (w_{i-1} + w_{i+1}) = r_i.  factor(): the inverses of the eliminated
// diagonal blocks D'_0 = D_0, D'_i = D_i - off^2 D'_{i-1}^{-1} (they do not depend on r, so the
// iterative-refinement solves reuse them); solve(): r'_i = r_i - off D'_{i-1}^{-1} r'_{i-1}, then
// back substitution.
bool factor_block_tridiag(const BlockSystem& S, std::vector<ld>& invs) {
  const int n = S.n;
  invs.assign(25 * (size_t)n, 0.0L);
  for (int i = 0; i < n; i++) {
    ld Di[5][5];
    for (int a = 0; a < 5; a++)
      for (int b = 0; b < 5; b++) Di[a][b] = S.D[25 * i + 5 * a + b];
    if (i > 0) {
      const ld* Ip = &invs[25 * (i - 1)];
      for (int a = 0; a < 5; a++)
        for (int b = 0; b < 5; b++) Di[a][b] -= S.off * S.off * Ip[5 * a + b];
    }
    ld Inv[5][5];
    if (!inv5(Di, Inv)) return false;
    for (int a = 0; a < 5; a++)
      for (int b = 0; b < 5; b++) invs[25 * i + 5 * a + b] = Inv[a][b];
  }
  return true;
}

void solve_block_tridiag(const BlockSystem& S, const std::vector<ld>& invs, const std::vector<ld>& r,
                         std::vector<ld>& w) {
  const int n = S.n;
  std::vector<ld> rp(5 * (size_t)n);
  for (int i = 0; i < n; i++) {
    for (int a = 0; a < 5; a++) {
      ld ri = r[5 * i + a];
      if (i > 0) {
        const ld* Ip = &invs[25 * (i - 1)];
        ld s = 0;
        for (int b = 0; b < 5; b++) s += Ip[5 * a + b] * rp[5 * (i - 1) + b];
        ri -= S.off * s;
      }
      rp[5 * i + a] = ri;
    }
  }
  w.assign(5 * (size_t)n, 0.0L);
  for (int i = n - 1; i >= 0; i--) {
    ld t[5];
    for (int a = 0; a < 5; a++) t[a] = rp[5 * i + a] - (i + 1 < n ? S.off * w[5 * (i + 1) + a] : 0.0L);
    for (int a = 0; a < 5; a++) {
      ld s = 0;
      for (int b = 0; b < 5; b++) s += invs[25 * i + 5 * a + b] * t[b];
      w[5 * i + a] = s;
    }
  }
}

}  // namespace

hz_status build_table(double g_min, double g_max, double dg, double lambda,
                      const std::vector<double>& theta, const std::vector<double>& phi, Table* out) {
  if (!(dg > 0) || !(g_max > g_min) || !(g_min > 2.0) || !(lambda >= 0) || theta.empty() || phi.empty()) {
    set_error("hz_build_weight_table: need g_min > 2, g_max > g_min, dg > 0, lambda >= 0, angles");
    return HZ_ERR_INVALID_ARG;
  }
  const int n = (int)llround((g_max - g_min) / dg) + 1;
  if (n < 2) {
    set_error("hz_build_weight_table: fewer than 2 tabulated G values");
    return HZ_ERR_INVALID_ARG;
  }
  BlockSystem S;
  S.n = n;
  S.D.assign(25 * (size_t)n, 0.0L);
  S.rhs.assign(5 * (size_t)n, 0.0L);
  S.off = -(ld)lambda;
  // the angles' sines and cosines once (the G loop only needs cos of the scaled direction cosines)
  std::vector<ld> cph(phi.size()), sph(phi.size()), cth(theta.size()), sth(theta.size());
  for (size_t k = 0; k < phi.size(); k++) { cph[k] = cosl((ld)phi[k]); sph[k] = sinl((ld)phi[k]); }
  for (size_t k = 0; k < theta.size(); k++) { cth[k] = cosl((ld)theta[k]); sth[k] = sinl((ld)theta[k]); }
  // the per-G blocks are independent: threads own contiguous ranges of G, each block is summed in
  // the same (phi outer, theta inner) order as a serial loop, so the table is bitwise thread-count
  // independent
  auto assemble = [&](int i0, int i1) {
    for (int i = i0; i < i1; i++) {
      ld G = (ld)g_min + (ld)dg * i;
      for (size_t kp = 0; kp < phi.size(); kp++)        // phi outer
        for (size_t jt = 0; jt < theta.size(); jt++) {  // theta inner
          ld H[5], g;
          h_row_cs(G, cph[kp], sph[kp], cth[jt], sth[jt], H, &g);
          for (int a = 0; a < 5; a++) {
            for (int b = 0; b < 5; b++) S.D[25 * i + 5 * a + b] += H[a] * H[b];
            S.rhs[5 * i + a] += H[a] * g;
          }
        }
      ld d = (i == 0 || i == n - 1) ? 1.0L : 2.0L;  // D^T D of first differences (no boundary rows)
      for (int a = 0; a < 5; a++) S.D[25 * i + 5 * a + a] += (ld)lambda * d;
    }
  };
  const long long rows = (long long)n * (long long)(phi.size() * theta.size());
  const int nthr = rows < 4000 ? 1 : (int)std::min<unsigned>(8u, std::max(1u, std::thread::hardware_concurrency()));
  if (nthr == 1) {
    assemble(0, n);
  } else {
    std::vector<std::thread> pool;
    for (int k = 0; k < nthr; k++) pool.emplace_back(assemble, (int)((long long)n * k / nthr), (int)((long long)n * (k + 1) / nthr));
    for (auto& t : pool) t.join();
  }
  std::vector<ld> w, invs;
  if (!factor_block_tridiag(S, invs)) {
    set_error("hz_build_weight_table: singular normal equations (lambda = 0 with rank-3 blocks? A14)");
    return HZ_ERR_RANK;
  }
  solve_block_tridiag(S, invs, S.rhs, w);
  // iterative refinement on the normal equations
  for (int it = 0; it < 2; it++) {
    std::vector<ld> r(5 * (size_t)n);
    for (int i = 0; i < n; i++)
      for (int a = 0; a < 5; a++) {
        ld s = S.rhs[5 * i + a];
        for (int b = 0; b < 5; b++) s -= S.D[25 * i + 5 * a + b] * w[5 * i + b];
        if (i > 0) s -= S.off * w[5 * (i - 1) + a];
        if (i + 1 < n) s -= S.off * w[5 * (i + 1) + a];
        r[5 * i + a] = s;
      }
    std::vector<ld> dw;
    solve_block_tridiag(S, invs, r, dw);
    for (size_t k = 0; k < w.size(); k++) w[k] += dw[k];
  }
  out->g_min = g_min;
  out->dg = dg;
  out->n_g = n;
  out->lambda = lambda;
  out->rows5.resize(5 * (size_t)n);
  for (size_t k = 0; k < w.size(); k++) out->rows5[k] = (double)w[k];
  return HZ_OK;
}

}  // namespace hz
