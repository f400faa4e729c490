/*
 * hz.h — C ABI of libhz, the B200 (sm_100a) wavelength-adaptive 27-point Helmholtz hot path.
 *
 * Method: Aghamiry, Gholami, Combe & Operto, "Accurate 3D frequency-domain seismic wave modeling
 * with the wavelength-adaptive 27-point finite-difference stencil" (arXiv 2108.08730).
 * Citations "P:n" are lines of that paper's text; readings "An" are listed in
 * DESIGN.md §2 (same numbering as SURVEY.md §8(c)).
 *
 * The four calls of the north star:
 *   build_weight_table(G range, dG, lambda)  -> hz_build_weight_table
 *   assemble_coeffs(v, f, h, pml)             -> hz_assemble_coeffs
 *   apply_impedance(u -> Au)                  -> hz_apply_impedance
 *   solve(b[nrhs] -> u)                       -> hz_solve
 *
 * Conventions
 *   - Grids are C-ordered [z][y][x] (x fastest).  A rank owns the z-slab [z0, z0+nz_local) of a
 *     global nx*ny*nz_global grid whose dimensions INCLUDE the PML pad (A18).
 *   - Complex fields are interleaved (re, im): complex64 = 2 x float, complex128 = 2 x double.
 *     Field buffers have one halo plane at each end and a padded row pitch:
 *     [nrhs][nz_local+2][ny][ldx] with ldx = hz_field_ldx(nx) = nx rounded up to a multiple of 4
 *     (32-byte rows for complex64: the apply moves its plane tiles with tensor-map TMA copies, which
 *     need 16-byte row strides, and every row starts on a DRAM sector).  Local plane k lives at index
 *     k+1; column x < nx of row y at [y][x].  The halo planes are owned by the library during a call
 *     (see each function); the caller allocates them.  Pad columns [nx, ldx) are never read as
 *     field values; outputs of the apply (au) get zeros there, the solver leaves x's pads as given.
 *   - Real model arrays (velocity) are float for HZ_C64 and double for HZ_C128, [nz_local][ny][nx].
 *   - Pointers may be device or host memory: the library inspects each pointer
 *     (cudaPointerGetAttributes) and stages host buffers through device memory itself.  The
 *     caller owns every buffer it passes; the library owns hz_ctx / hz_table / hz_coeffs objects
 *     and all solver workspace.
 *   - `stream` is a cudaStream_t passed as void* (NULL = the legacy default stream).
 *   - Errors: a negative hz_status means nothing was written and hz_last_error() (thread-local)
 *     explains; a positive status means the call completed and its outputs are valid, with a
 *     warning (read the stats).  There is no CPU fallback: without a CUDA device every compute
 *     call returns HZ_ERR_CUDA.
 */
#ifndef HZ_H_
#define HZ_H_

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HZ_OK = 0,
  HZ_NOT_CONVERGED = 1,    /* solve: max_iter reached; x holds the best (last) iterate   */
  HZ_BREAKDOWN = 2,        /* solve: BiCGSTAB breakdown persisted after restarts                 */
  HZ_WARN_CLAMPED = 3,     /* assemble: some points had G outside the table range (clamped)      */
  HZ_ERR_INVALID_ARG = -1, /* bad sizes / NULL pointers / inconsistent grid                          */
  HZ_ERR_DOMAIN = -2,      /* v <= 0 or non-finite, f <= 0, h <= 0       */
  HZ_ERR_RANK = -3,        /* weight LS singular (e.g. lambda = 0 with rank-3 blocks, A14)          */
  HZ_ERR_OOM = -4,
  HZ_ERR_CUDA = -5,
  HZ_ERR_NCCL = -6,
  HZ_ERR_SOURCE_IN_PML = -7 /* point source inside the PML                              */
} hz_status;

typedef enum { HZ_C64 = 0, HZ_C128 = 1 } hz_dtype;

/* Mass formulation: Eq. 8 (per-neighbour kappa, default A5) or the collocation-kappa
 * variant "Eq. 10". */
typedef enum { HZ_MASS_EQ8 = 0, HZ_MASS_COLLOC = 1 } hz_mass;
/* Weight rule of a row: GA = the weights tabulated at the row's own local G; GAm = the mean of
 * the weights tabulated at the row's 27 stencil nodes (in-grid nodes only; reading A19).
 * GA_RECORD = GA in "record mode": the per-point weights are stored once at assemble
 * and read by every apply instead of being recomputed from v (same values; +20 / 40 B per point). */
typedef enum { HZ_RULE_GA = 0, HZ_RULE_GAM = 1, HZ_RULE_GA_RECORD = 2 } hz_rule;

typedef struct hz_ctx hz_ctx;
typedef struct hz_table hz_table;
typedef struct hz_coeffs hz_coeffs;

const char* hz_last_error(void);
const char* hz_version(void);
/* Row pitch (elements) of every field buffer for a grid nx wide: nx rounded up to a multiple of 4. */
int hz_field_ldx(int nx);

/* ---------------------------------------------------------------------------------------------
 * Context: one per rank (process).  nranks > 1 creates an NCCL communicator from `id` (obtained
 * on rank 0 with hz_get_unique_id and broadcast by the caller, e.g. through torch.distributed);
 * the library owns the communicator and its streams.  nranks == 1 needs no id (may be NULL).
 * ------------------------------------------------------------------------------------------- */
hz_status hz_get_unique_id(unsigned char id[128]);
hz_status hz_ctx_create(int cuda_device, int nranks, int rank, const unsigned char* id, hz_ctx** out);
/* Loopback group: nranks (1..16) contexts of ONE process on ONE device, out[0..nranks-1], one per z-slab
 * rank.  Each rank's calls must come from its own host thread (the ranks meet in host barriers inside
 * every collective call); halo planes move with one cudaMemcpyAsync per plane and dot products are
 * summed over the ranks by a device kernel in rank order — the same call sites as the NCCL path.  For
 * testing the multi-slab data path without several GPUs.  Destroy every context with hz_ctx_destroy. */
hz_status hz_ctx_create_loopback(int cuda_device, int nranks, hz_ctx** out);
void hz_ctx_destroy(hz_ctx* ctx);

/* ---------------------------------------------------------------------------------------------
 * (1) build_weight_table — host, fp64 inputs, long-double arithmetic, deterministic.
 * Tabulates G_i = g_min + i*dg, i = 0..n_g-1 (n_g = round((g_max-g_min)/dg)+1) and solves
 *   min_w ||H w - g||^2 + lambda ||D P w||^2
 * with per-G blocks of rows H_l(G_i, theta_j, phi_k), g (Eq. linear_basic; H2 with the
 * "+1" of reading A1), phi outer / theta inner, D = first differences along G with no
 * boundary rows (A11).  Unknowns per G: (ws1, ws2, mu0, mu1, mu2) (A2).
 * angles == NULL: theta, phi in {0,10,20,30,40} degrees (A10).
 * Errors: HZ_ERR_INVALID_ARG (n_g < 2, dg <= 0, g_min <= 2), HZ_ERR_RANK (singular system).
 * ------------------------------------------------------------------------------------------- */
typedef struct {
  int n_theta, n_phi;
  const double* theta_rad; /* [n_theta] */
  const double* phi_rad;   /* [n_phi]   */
} hz_angles;

hz_status hz_build_weight_table(double g_min, double g_max, double dg, double lambda,
                                const hz_angles* angles, hz_table** out);

/* Import a table from rows (ws1, ws2, mu0, mu1, mu2) [n_g][5] at G_i = g_min + i*dg (shared-table
 * parity; n_g == 1 gives the non-adaptive G4 / Gm stencils of P:273 as one-row tables). */
hz_status hz_table_import(double g_min, double dg, int n_g, const double* rows5, hz_table** out);

/* Export: n_g, and optionally rows5 [n_g][5] and class weights rows7 [n_g][7] =
 * (ws1, ws2, ws3, wm0, wm1, wm2, wm3) with ws3 = 1-ws1-ws2, wm_k = (mu0, 6 mu1, 12 mu2),
 * wm3 = 1 - wm0 - wm1 - wm2.  Either array may be NULL. */
hz_status hz_table_rows(const hz_table* t, int* n_g, double* rows5, double* rows7);
void hz_table_destroy(hz_table* t);

/* ---------------------------------------------------------------------------------------------
 * (2) assemble_coeffs — device.  Copies v (with one halo plane per side, exchanged with the
 * neighbouring ranks) into library memory, validates it, counts clamped points, builds the 1-D
 * PML arrays (profile A7, per-axis stretching A8) and uploads the table.  The per-point
 * coefficients (G = v/(f h), lookup + interpolation, t0..t2, mu0..mu3) are
 * NOT stored: every apply recomputes them from v (fused mode, 4 bytes/point).  rule = HZ_RULE_GAM
 * (HZ_RULE_GA_RECORD) instead stores the 27-node mean (the row's own) weights once
 * ([5][nz_local+2][ny][nx] in the dtype's precision) and the apply reads them (+20 / 40 bytes per
 * point and apply).
 * grid: this rank's slab of the global grid.  pml->v_pml <= 0 selects max(v) over all ranks.
 * With nranks > 1 the table rows of rank 0 are broadcast so every rank uses identical weights.
 * Returns HZ_WARN_CLAMPED (outputs valid) when *n_clamped > 0.
 * ------------------------------------------------------------------------------------------- */
typedef struct {
  int nx, ny, nz_global; /* global grid including the PML pad                  */
  int z0, nz_local;      /* this rank's planes [z0, z0 + nz_local)               */
  double h;              /* grid interval (m)                                    */
  int v_halo;            /* 0: v is [nz_local][ny][nx] and its halo planes come from the neighbour
                            ranks (NCCL); 1: v is [nz_local+2][ny][nx] and already holds planes
                            z0-1 and z0+nz_local (ignored where they fall outside the grid) — lets
                            one process emulate a z-slab decomposition                          */
} hz_grid;

typedef struct {
  int npml;        /* PML width in nodes on every face (0 = no PML)                         */
  double r_coeff;  /* target reflection coefficient R (A7); 1 => gamma = 0 (transparent)   */
  double v_pml;    /* velocity in the gamma profile; <= 0 => max(v)                         */
} hz_pml;

hz_status hz_assemble_coeffs(hz_ctx* ctx, const hz_grid* grid, hz_dtype dtype, const void* v,
                             double freq_hz, const hz_pml* pml, const hz_table* table, hz_mass mass,
                             hz_rule rule, hz_coeffs** out, long long* n_clamped);

/* Parity export (not on the hot path).  record: [8][nz_local][ny][nx] real (float for C64, double
 * for C128) = (k^2 = (2 pi f / v)^2, t0, t1, t2, mu0, mu1, mu2, mu3) per point (may be NULL).
 * pml: complex128 host array [3 axes x,y,z][2 (a-, a+)][nmax] with a-(i) = 1/(h^2 xi(i) xi(i-1/2)),
 * a+(i) = 1/(h^2 xi(i) xi(i+1/2)); nmax >= max(nx, ny, nz_global) (may be NULL). */
hz_status hz_coeffs_export(const hz_coeffs* c, void* record, void* pml_host, int nmax);
void hz_coeffs_destroy(hz_coeffs* c);

/* Visco-acoustic, variable-density medium (NEXT-2; Eqs. 1.1-1.4 and 2; DESIGN.md readings
 * A24, A25).  Attaches buoyancy b = 1/rho and the quality factor Q to an assembled operator, which
 * then reads
 *   (Au)_n = omega^2 sum_d mu_{|d|}(w_n) u_{n+d} / kappa_{n+d}        kappa = v_c^2 / b,
 *                                                                    v_c = v (1 - i/(2Q))   (A24)
 *          + sum_a sum_{p,q} T(p,q; w_n) [beta+ a+_a (u_+ - u_0) + beta- a-_a (u_- - u_0)]_{line p,q}
 *   beta+- = (b+-(n) + b+-(n + d_perp))/2,  b+-(m) = (b_m + b_{m +- e_a})/2              (A25)
 * (the weights w_n still come from G = v/(f h)).  b, q: real arrays of the coeffs' real type
 * (float for HZ_C64, double for HZ_C128) in v's layout ([nz_local][ny][nx], or [nz_local+2][ny][nx]
 * when grid.v_halo), host or device, copied (the caller keeps ownership); NULL b means b = 1, NULL q
 * means Q = infinity; both NULL restores the rho = 1 elastic operator.  Halo planes come from the
 * neighbour ranks as for v.  Every later apply / solve / residual of c uses the medium; the kernel
 * is apply_medium.cu (a gather kernel: correctness first).  Errors:
 * HZ_ERR_DOMAIN if a b is not positive and finite or a Q not > 0 (each rank checks its slab),
 * HZ_ERR_CUDA on allocation / copy failures.  Synchronous on `stream`. */
hz_status hz_coeffs_set_medium(hz_coeffs* c, const void* b, const void* q, void* stream);

/* ---------------------------------------------------------------------------------------------
 * (3) apply_impedance — Au = [M + S] u for nrhs fields, matrix-free, asynchronous on
 * `stream`.  u and au: [nrhs][nz_local+2][ny][ldx] complex of the coeffs' dtype.  u's halo planes
 * are overwritten with the neighbouring ranks' boundary planes (nranks > 1); planes outside the
 * global grid are treated as zero (Dirichlet, A9) and never read.  au's halo planes are not written;
 * its pad columns are written as zeros (complex64) or left untouched (complex128).
 * Row n of the operator (interior class-sum form; PML rows add the stretched per-axis terms):
 *   (Au)_n = omega^2 sum_d mu_{|d|}(w_n) u_{n+d} / v_{n+d}^2                 (Eq. 8)
 *          + sum_a sum_e D_a(n_a, e) sum_{p,q} T(p,q; w_n) u_{n + e e_a + p e_b + q e_c}   (A6, A8)
 * ------------------------------------------------------------------------------------------- */
hz_status hz_apply_impedance(const hz_coeffs* c, void* u, void* au, int nrhs, void* stream);

/* ---------------------------------------------------------------------------------------------
 * (4) solve — batched BiCGSTAB (or BiCGStab(2), opts.ell) for A x_r = b_r, r = 0..nrhs-1 (north
 * star (3)); blocking.  opts == NULL or hz_solve_opts_default(): the defaults below; in a caller's
 * struct every field left 0 selects its default (a zero-initialised struct is the default setting).
 * b, x: [nrhs][nz_local+2][ny][ldx]; x holds the initial guess on entry (zeros OK) and the final
 * iterate on exit.  Each RHS iterates independently (per-RHS scalars on the device, fp64 dot
 * accumulation, residual replacement every replace_every iterations) and stops when its
 * recomputed TRUE residual ||b - A x|| / ||b|| <= rtol (A21).  relres_out[nrhs] receives the true
 * relative residual and iters_out[nrhs] the iteration count (either may be NULL).
 * complex64 coefficients: vectors are stored and applied in complex64, but the replaced residual
 * b - A(x + x_lo) is applied in fp64 and the iterate carries a compensation term x_lo (TwoSum of
 * the x update, device-resident, folded into x on exit), so the true residual can reach 1e-6 and
 * below (a plain complex64 iteration floors near 1e-6 on the configs of BASELINE.json); the
 * iteration itself runs to rtol/2 so the fp64-recomputed residual lands below rtol.  A RHS whose
 * true residual stagnates (stats.stagnated) is retired with HZ_NOT_CONVERGED and its last iterate.
 * Host pointers for b / x are accepted: the call stages them (pinned) through device buffers.
 * Returns HZ_OK, HZ_NOT_CONVERGED or HZ_BREAKDOWN (outputs valid), or an error.
 * ------------------------------------------------------------------------------------------- */
typedef struct {
  double rtol;       /* default 1e-6 (0 = default)                                 */
  int max_iter;      /* default 20000 (0 = default)                                */
  int replace_every; /* residual replacement period, default 50 (0 = default, < 0 = never) */
  int check_every;   /* host convergence poll period, default 10 (0 = default)     */
  int timing;        /* 1 = time every operator-apply launch with CUDA events      */
  int ell;           /* Krylov method: 1 (or 0) = BiCGSTAB (default); 2 = BiCGStab(2)
                        (Sleijpen & Fokkema 1993: two BiCG steps then a 2-term minimal-
                        residual polynomial; four applies per outer step, counted as two
                        iterations; robust where BiCGSTAB's omega -> 0 stalls it — DESIGN.md
                        reading A23; max_iter is tested per outer step, so the count can
                        end at max_iter + 1).  Any other value: HZ_ERR_INVALID_ARG.     */
  int stall_window;  /* a RHS whose true residual has not dropped 10% within this many
                        iterations is retired (HZ_NOT_CONVERGED, stats.stagnated = 1);
                        0 = default max(20*replace_every, 1000); < 0 = never            */
  int precond;       /* 0: none.  1: right preconditioning by one V-cycle of the complex
                        shifted-Laplacian multigrid (∇² + (1 + 0.5i)ω²/v², damped Jacobi,
                        DESIGN.md reading A27; NEXT-4, the iterative route of P:35).
                        complex64, ell = 1, one rank, GA / Eq. 8 / Eq. "10" coefficients
                        (not the visco-acoustic medium); otherwise HZ_ERR_INVALID_ARG. */
} hz_solve_opts;

typedef struct {
  double apply_ms_total;    /* sum of operator-apply kernel durations (timing = 1)               */
  long long apply_launches; /* number of operator applies (one kernel launch each for complex64,
                               two for the register-path kernels: complex128, fp64 residual)      */
  long long kernel_launches;/* all libhz kernel launches during the call                         */
  double apply_bytes_total; /* algorithmic HBM bytes of all applies: per apply
                               n_points * (sizeof(real) + n_active_rhs * k * sizeof(complex)),
                               k = fields read/written per RHS by the launch's epilogue          */
  double apply_points_total;/* grid points x active RHS processed by all applies                  */
  int replacements;         /* residual replacements performed                                   */
  int restarts;             /* breakdown restarts                                                */
  int iterations;           /* BiCGSTAB(-equivalent) iterations of the batch (max over RHS)       */
  int stagnated;            /* 1 if some RHS was retired because its true residual stagnated
                               (no 10% reduction in stall_window iterations)      */
} hz_solve_stats;

/* The default options: rtol 1e-6, max_iter 20000, replace_every 50, check_every 10, ell 1. */
hz_solve_opts hz_solve_opts_default(void);
/* A RHS whose BiCGSTAB breaks down (rho, omega or (r0^, v) ~ 0) is restarted from its recomputed true
 * residual; one that breaks down more than max(50, stall_window/check_every + 1) times is retired on
 * its own and the call returns HZ_BREAKDOWN (the other RHS continue). */
hz_status hz_solve(const hz_coeffs* c, const void* b, void* x, int nrhs, const hz_solve_opts* opts,
                   double* relres_out, int* iters_out, hz_solve_stats* stats, void* stream);

/* Point-source RHS (reading A15).  node_xyz: GLOBAL node indices [nsrc][3] (x, y, z);
 * amp_re_im: [nsrc][2] (NULL = unit amplitudes).  consistent = 1: b_n = amp mu_{|n-s|}(w_n)/h^3 on
 * the 27 nodes around s (row n's own weights); 0: nodal amp/h^3.  b: [nsrc][nz_local+2][ny][ldx],
 * zero-filled by the call, entries outside this rank's slab skipped.  HZ_ERR_SOURCE_IN_PML if a
 * source lies inside the PML. */
hz_status hz_point_sources(const hz_coeffs* c, int nsrc, const long long* node_xyz,
                           const double* amp_re_im, int consistent, void* b, void* stream);

/* ---------------------------------------------------------------------------------------------
 * Evaluation (not on the hot path)
 * hz_eqerror: the paper's accuracy metric (Eq. eqerror; reading A20) between two
 * wavefields of this rank's slab, [nz_local+2][ny][ldx] complex of the coeffs' dtype (host or device;
 * the owned planes are read):
 *   err = sum W |Re(u_ref - u)| / sum W |Re u_ref|  +  sum W |Im(u_ref - u)| / sum W |Im u_ref|
 * with W = h * distance to the source node src_xyz (global x, y, z), over the nodes at least
 * npml_mask nodes away from every face and more than ball_cells nodes from the source.  Sums in fp64
 * (fixed-order block reduction), summed over the ranks.  HZ_ERR_DOMAIN if a reference sum is 0.
 * hz_table_dispersion: normalised numerical phase velocity of the table's stencil (P:129-160,
 * Eq. vtilde) at G[i] (clamped linear interpolation of the table, A13) for the propagation angles
 * (theta[j], phi[j]) in radians, evaluated on the device in fp64: vtilde[i*nang + j] (host or device
 * memory; G, theta, phi are host arrays).  HZ_ERR_DOMAIN for G <= 0.
 * ------------------------------------------------------------------------------------------- */
/* hz_export_matrix: the explicit impedance matrix rows of this rank's slab (the paper's
 * sparse direct-solver setting): for every owned node n (C order [nz_local][ny][nx]) its 27 entries
 * A[n, n+d] (d in C order dz, dy, dx in {-1,0,1}) in the per-axis form (A6, A8; the coeffs' mass form
 * and weight rule), cols[n][27] = global node index (z*ny + y)*nx + x, or -1 with value 0 outside the
 * grid (Dirichlet, A9); vals[n][27] complex of the dtype.  Host or device arrays (caller-owned). */
hz_status hz_export_matrix(const hz_coeffs* c, long long* cols, void* vals, void* stream);
hz_status hz_eqerror(const hz_coeffs* c, const void* u_ref, const void* u, const long long src_xyz[3],
                     int npml_mask, double ball_cells, double* err_out, void* stream);
hz_status hz_table_dispersion(const hz_table* t, int nG, const double* G, int nang, const double* theta,
                              const double* phi, double* vtilde, void* stream);

/* Number of libhz kernels launched since process start (evidence for the bench's gpu_launches). */
long long hz_kernel_launch_count(void);

/* libhz keeps device buffers released by destroyed coeffs / solver workspaces in a cache for reuse
 * (re-assembling and re-solving every step then allocates nothing); this returns the cache to CUDA. */
void hz_trim_memory(void);


/* ---- NEXT-3: convergent Born series (CBS) reference wavefield ------------------------------------
 * hz_cbs_solve: the paper's heterogeneous-model reference ("highly-accurate Convergent Born
 * Series (CBS) method", iteration stopped at a backward error of 1e-12), restated in DESIGN.md reading A26
 * and oracle/cbs.py.  Solves (∇² + k²) u = s, k = 2πf/v, with the spectral Laplacian on the model
 * embedded in a periodic box padded by opts.pad cells per side (velocity of the nearest model node plus
 * an absorbing term i·absorb·k0²·Σ_axes (d/pad)²), by the preconditioned Born iteration
 *   u ← u − γ[u − G(V u − s)],  V = k² − k0² − iε,  γ = (i/ε)V,  G = 1/(|p|² − k0² − iε) (cuFFT Z2Z),
 * k0² = mid-range Re k², ε = 1.05·max|k² − k0²|, until ‖(∇² + k²)u − s‖/‖s‖ ≤ opts.tol (checked every
 * opts.check_every iterations).  complex128 throughout, one GPU (the context's device).
 *   v        [nz][ny][nx] float64 velocities (m/s), dense (no pitch, no halo), host or device
 *   src_xyz  nsrc × (x, y, z) node indices (host); s = amp/h³ at each node
 *   amps     nsrc × (re, im) (host) or NULL (unit amplitudes)
 *   u        [nz][ny][nx] interleaved complex128 (host or device, caller-owned): the model region
 *   stats    may be NULL: iterations, final backward error, k0², ε, box dims, pad, seconds
 * opts == NULL: hz_cbs_opts_default() (pad = -1: two of the longest wavelengths; absorb 1; tol 1e-12;
 * max_iter 200000; check_every 20).  Returns HZ_OK, HZ_NOT_CONVERGED (max_iter reached; u = last
 * iterate), HZ_ERR_INVALID_ARG (sizes, sources outside the model, options), HZ_ERR_DOMAIN (v ≤ 0 or
 * non-finite, h or f ≤ 0), HZ_ERR_OOM / HZ_ERR_CUDA.  Synchronous on `stream`. */
typedef struct {
  int pad;            /* padding cells per side (< 0: two of the longest wavelengths)     */
  double absorb;      /* absorbing strength a (α = a·k0²·Σ (d/pad)²)                      */
  double tol;         /* backward-error tolerance (1e-12)                           */
  int max_iter;
  int check_every;    /* iterations between backward-error evaluations                    */
} hz_cbs_opts;
typedef struct {
  int iterations;
  double backward_error;
  double k0sq, eps;
  int box[3];         /* Nx, Ny, Nz of the FFT box */
  int pad;
  double seconds;
} hz_cbs_stats;
hz_cbs_opts hz_cbs_opts_default(void);
hz_status hz_cbs_solve(hz_ctx* ctx, int nx, int ny, int nz, double h, const double* v, double freq, int nsrc,
                       const long long* src_xyz, const double* amps, const hz_cbs_opts* opts, double* u,
                       hz_cbs_stats* stats, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HZ_H_ */
