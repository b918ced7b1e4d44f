/*
 * uno_cg.h — C ABI of libunocg.so, the B200 (sm_100a) hot path of UNO-CG
 * (Herb & Fritzen, arXiv 2508.02681; PAPER.md in the reference tree).
 *
 * What the library computes
 * -------------------------
 * The UNO-CG hybrid solver, Alg 2: preconditioned CG on the
 * Q1 voxel finite-element system A u = f of a two-phase periodic RVE
 * (§3.1 Eq 20-22; thermal §5.1 Eq 74-77, elastic §5.2 Eq 78-84),
 * preconditioned by the Unitary-Neural-Operator apply s = T^H Q T r (Eq 46-49,
 * P:458-490) with T the orthonormal DFT (Table 1 row "Periodic") and Q
 * the per-frequency c x c symbol G_hat(k).  Because no trained weights exist,
 * G_hat is the FANS reference-medium Green's operator (§3.3.4 Eq 33-37)
 * times (c = 1) / plus (c = 3) a seeded SPD perturbation.
 *
 * Conventions (all calls)
 * -----------------------
 *  - fp64 everywhere; phase fields are uint8 (0 = matrix, 1 = inclusion, §5).
 *  - Grid: N1 (x, fastest) x N2 (y) x N3 (z) voxels, N3 = 1 in 2D; cubic voxels of
 *    edge h.  Boundary conditions: periodic on every axis, or (3D) the mixed case of
 *    Eq 82 / §6.4 with periodic x, y and Dirichlet faces on z (bc = {0,0,1}; U = DFT_x (x)
 *    DFT_y (x) DST-I_z, Table 1 "Mixed" P:452; node planes z = 1..N3-1 are the unknowns,
 *    N1 >= 32, N3 <= 512), or (3D) Dirichlet faces on every axis (bc = {1,1,1}; U = DST-I on
 *    every axis, Table 1 row "Dirichlet" P:451; N1 >= 32 thermal / 16 elastic, N2 >= 16,
 *    8 <= N3, all <= 512); in 2D also Dirichlet on both axes (bc = {1,1,0}) and the mixed
 *    case periodic x / Dirichlet y (bc = {0,1,0}; U = F_x (x) DST-I_y, Table 1 row "Mixed"),
 *    16 <= N1, N2 <= 512.  Other combinations return UNO_ERR_UNSUPPORTED.
 *    N1, N2 in {8..1024}, N3 in {1} U {4..1024}, all powers of two.
 *  - Field layout (device): component-planar C order [nrhs][c][P3][N2][N1] with P3 = N3
 *    (periodic, and the all-Dirichlet / 2D cases: the nodes with index 0 on a Dirichlet axis
 *    are the fixed boundary nodes, held at 0 on input and output) or N3 - 1 (3D mixed
 *    Dirichlet z: stored planes are nodes
 *    z = 1..N3-1); node
 *    (i,j,k) at h*(i,j,k); voxel (i,j,k) has corners (i+a1, j+a2, k+a3) mod N.
 *    The paper's interleaved vec() (§1.6 Eq 1) is a fixed permutation of this.
 *  - c = 1 (thermal) or c = dim (elastic).  nrhs load cases are iterated together,
 *    each with its own CG scalars (a converged load is frozen, so its iterates equal
 *    an unbatched solve).
 *  - Loads (host): thermal macroscopic gradient g_bar in R^dim; elastic macroscopic
 *    strain eps_bar as a Mandel vector (App. A Eq A2-A4), length 3 (2D)
 *    or 6 (3D), order (11,22,[33],sqrt2*12,[sqrt2*13,sqrt2*23]).
 *  - Streams: every call is stream-ordered on desc.stream (a cudaStream_t owned by
 *    the caller, e.g. torch.cuda.current_stream().cuda_stream); calls that return
 *    host scalars synchronise that stream.
 *  - Ownership: all field buffers (phase, u, f, r, z, ...) are caller-owned device
 *    memory.  The handle's workspace (CG vectors r, d, p, u, a second direction buffer for the
 *    paired u updates of 3D grids, one spectrum buffer, the
 *    tabulated symbol, twiddle tables, reduction scratch; uno_cg_workspace_size bytes) is
 *    either caller-provided (borrowed, never freed by the library) or allocated by
 *    uno_cg_create and freed in uno_cg_destroy.  Outside it the library allocates only
 *    on demand: the per-solve coefficient record (3 x 8 x (cap+1) doubles, grown on the
 *    first solve with a larger cap), the Jacobi diagonal (uno_cg_set_preconditioner) and
 *    the training spectrum (uno_cg_train_features).
 *  - Errors: every call returns uno_status; on error nothing is written to the
 *    outputs unless stated, and uno_cg_last_error() returns a thread-local message.
 *    No C++ exception crosses the ABI.  Calls on one handle are not thread-safe.
 */
#ifndef UNO_CG_H
#define UNO_CG_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define UNO_API __attribute__((visibility("default")))
#else
#define UNO_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct uno_cg_handle uno_cg_handle; /* opaque */

typedef enum {
  UNO_OK = 0,
  UNO_ERR_ARG = 1,         /* NULL pointer or invalid scalar argument                    */
  UNO_ERR_SHAPE = 2,       /* grid size not supported (see Conventions)                   */
  UNO_ERR_CUDA = 3,        /* a CUDA runtime call failed (message in uno_cg_last_error)   */
  UNO_ERR_UNSUPPORTED = 4, /* valid per the paper but not built (boundary-condition pattern,
                              see Conventions; slab-mode restrictions in uno_cg_slab.h)   */
  UNO_ERR_NOT_SPD = 5,     /* Eq 55 safety check failed at create            */
  UNO_ERR_BREAKDOWN = 6,   /* d.p <= 0 or gamma_1 <= 0 during solve           */
  UNO_ERR_NONFINITE = 7,   /* NaN/Inf residual during solve                               */
  UNO_ERR_NCCL = 8         /* slab mode (uno_cg_slab.h): a peer/communicator exchange could
                              not be set up (peer buffer table, peer access)               */
} uno_status;

enum { UNO_THERMAL = 0, UNO_ELASTIC = 1 };

typedef struct {
  int32_t dim;        /* 2 or 3                                                          */
  int32_t n[3];       /* voxel counts N1, N2, N3 (N3 = 1 when dim == 2)                  */
  double h;           /* voxel edge; <= 0 means 1/N1 (unit cell)              */
  int32_t physics;    /* UNO_THERMAL (c = 1) or UNO_ELASTIC (c = dim)                    */
  int32_t bc[3];      /* per axis: 0 periodic, 1 Dirichlet; accepted patterns in Conventions */
  double mat[2][2];   /* phase 0 / phase 1: thermal {kappa, unused}; elastic {lambda, mu} */
  double ref[2];      /* reference medium (kappa_r | lambda_r, mu_r); ref[0] <= 0 means the
                         arithmetic mean of the phases          */
  uint64_t seed;      /* perturbation seed; 0 = unperturbed FANS symbol                  */
  double amp;         /* perturbation amplitude: c=1 rho in [1-amp, 1+amp];
                         c=3 G = Phi + amp*tr(Phi)/3*psi(theta) (Eq B5)                  */
  int32_t nrhs;       /* load cases iterated together, 1..8                              */
  void* stream;       /* cudaStream_t (NULL = legacy default stream)                     */
} uno_cg_desc;

typedef struct {
  int32_t iterations;  /* Alg 2 iterations performed (K applications)                      */
  int32_t converged;   /* 1 if ||r||_inf <= rel_tol * ||r0||_inf was reached               */
  int32_t status;      /* uno_status of this load case (BREAKDOWN / NONFINITE per load)   */
  int32_t pad_;
  double r0_inf;       /* ||r0||_inf = ||f||_inf                                           */
  double rel_res;      /* final recursive ||r||_inf / ||r0||_inf                           */
  double gamma_last;   /* last gamma_1 = r.s (Alg 2 l.7)                                   */
} uno_cg_report;

/* Device workspace a handle for `desc` needs (bytes): every buffer of Alg 2's state (r, d, p,
 * u), the spectrum, the G_hat table (Eq 51), twiddles and reduction scratch.  Validates desc
 * exactly as uno_cg_create does (same status codes); desc.stream is not used.            */
UNO_API uno_status uno_cg_workspace_size(const uno_cg_desc* desc, size_t* bytes);

/* Create a solver for one microstructure (the problem of Eq 22 / §5 on this grid).  Computes the
 * reference medium, tabulates G_hat(k)/n on the R2C half spectrum (Eq 46/49/51: the unique
 * entries v, C = c(c+1)/2 planes) and runs the Eq 55 check (every block with k != 0 SPD with
 * lambda_min > 1e-14; G_hat(0) = 0 shares the periodic null space).
 *   d_phase: device uint8 [N3][N2][N1], caller-owned, must outlive the handle.
 *   d_workspace: device memory of uno_cg_workspace_size(desc) bytes, 256-byte aligned,
 *     caller-owned and not touched by anyone else while the handle lives; NULL = the library
 *     allocates it (stream-ordered pool on desc.stream) and frees it in uno_cg_destroy.
 * Returns UNO_ERR_NOT_SPD (and no handle) if Eq 55 fails; UNO_ERR_ARG for a misaligned
 * workspace; UNO_ERR_CUDA if an allocation fails.                                        */
UNO_API uno_status uno_cg_create(const uno_cg_desc* desc, const uint8_t* d_phase, void* d_workspace,
                                 uno_cg_handle** out);

UNO_API uno_status uno_cg_destroy(uno_cg_handle* h);

/* Re-target a handle to another problem of the SAME grid, physics, h and nrhs: new phase
 * field, materials, reference medium, seed/amp.  Re-runs the a0 setup of uno_cg_create
 * (reference medium, G_hat table, Eq 55) on the handle's workspace without reallocating.
 * desc.stream is ignored (the handle keeps its stream).  On UNO_ERR_NOT_SPD the handle
 * keeps the new (rejected) problem and must be updated again before solving.            */
UNO_API uno_status uno_cg_update(uno_cg_handle* h, const uno_cg_desc* desc, const uint8_t* d_phase);

/* Galerkin right-hand side f = l(phi_i) of the decomposition Eq 76 / Eq 81:
 *   thermal f_i = -sum_{e ni i} kappa_e (s(a).g_bar) h^(d-1)/2^(d-1)
 *   elastic f_(i,alpha) = -sum_e sum_j s(a)_j sigma_bar^e_(alpha j) h^(d-1)/2^(d-1),
 *           sigma_bar^e = lambda_e tr(eps_bar) I + 2 mu_e eps_bar
 *   h_loads: host [nrhs][dim] (thermal) or [nrhs][D] (elastic, Mandel).
 *   d_f: device [nrhs][c][N3][N2][N1].                                                  */
UNO_API uno_status uno_cg_rhs(uno_cg_handle* h, const double* h_loads, double* d_f);

/* p = A u (Alg 2 l.9) for all nrhs vectors; optional u.Au per vector.
 *   d_u, d_Au: device [nrhs][c][N3][N2][N1] (must not alias).  h_uAu: host [nrhs] or NULL. */
UNO_API uno_status uno_cg_apply_K(uno_cg_handle* h, const double* d_u, double* d_Au, double* h_uAu);

/* z = T^H Q T r (Alg 2 l.4-6) for all nrhs vectors; optional r.z per vector (Alg 2 l.7,
 * evaluated in the transformed space by Parseval).
 *   d_r, d_z: device [nrhs][c][N3][N2][N1] (may alias).  h_rz: host [nrhs] or NULL.     */
UNO_API uno_status uno_cg_apply_precond(uno_cg_handle* h, const double* d_r, double* d_z, double* h_rz);

/* Alg 2 from u0 = 0 for the nrhs loads: r = f; d = 0; gamma_1 = 1; iterate while
 * ||r||_inf > rel_tol * ||r0||_inf (relative stop on the recursive residual)
 * and iterations < max_iter.  fixed_iters > 0 runs exactly that many iterations instead
 * (parity protocol).  An RHS with ||f||_inf <= 1e-13 * max modulus *
 * h^(d-1) * ||load||_inf is a zero RHS: 0 iterations, u = 0.  On return u holds the
 * per-component mean-free solution.
 *   h_loads: as uno_cg_rhs.  d_u: device [nrhs][c][N3][N2][N1] (output).
 *   rep: host [nrhs] reports (may be NULL).  h_hist: host [nrhs][cap+1] residual history
 *   ||r_m||_inf/||r0||_inf, m = 0..cap with cap = fixed_iters > 0 ? fixed_iters : max_iter
 *   (entries past a load's last iteration are unspecified), or NULL.
 * Returns UNO_ERR_BREAKDOWN / UNO_ERR_NONFINITE if any load broke down (rep says which). */
UNO_API uno_status uno_cg_solve(uno_cg_handle* h, const double* h_loads, double rel_tol, int32_t max_iter,
                        int32_t fixed_iters, double* d_u, uno_cg_report* rep, double* h_hist);

/* Effective property from the nrhs solutions:
 *   out_ij = <C>_ij - f^(i) . u^(j) / |Omega|,  |Omega| = N1 N2 N3 h^dim,
 * thermal <C>_ij = <kappa> delta_ij (g_bar loads), elastic <C>_ij = B^(i):<D>:B^(j)
 * evaluated for the given loads (Mandel).  f^(i) is recomputed from the phase field.
 *   d_u: device [nrhs][c][N3][N2][N1]; h_loads as uno_cg_rhs; h_out: host [nrhs][nrhs]. */
UNO_API uno_status uno_cg_effective_property(uno_cg_handle* h, const double* d_u, const double* h_loads, double* h_out);

/* Preconditioner of the PCG loop (uno_cg_solve) and of uno_cg_apply_precond:
 *   UNO_PRECOND_UNO      P = T^H Q T, the UNO / FANS symbol (default; Eq 48)
 *   UNO_PRECOND_IDENTITY P = I, unpreconditioned CG
 *   UNO_PRECOND_JACOBI   P = diag(A)^-1 (Eq 25), diag(A) from the phase field
 * — the paper's baselines of §6 / Table 4.  The choice stays with the handle
 * (uno_cg_update recomputes the Jacobi diagonal for the new problem).                     */
enum { UNO_PRECOND_UNO = 0, UNO_PRECOND_IDENTITY = 1, UNO_PRECOND_JACOBI = 2 };
UNO_API uno_status uno_cg_set_preconditioner(uno_cg_handle* h, int32_t kind);

/* Second-order UNO preconditioner training (§4.4 Alg 4, Eq 59-72, App. B; 3D
 * periodic grids, c = 1 or 3).  Training pairs (Eq 58, 60): r = f, s = A^-1 f (e.g. from
 * uno_cg_rhs / uno_cg_solve on the training microstructures).
 *   uno_cg_train_features: transforms the nrhs pairs once with the library's forward passes and
 *     accumulates d_feat += scale * (alpha_1..alpha_C, beta_1..beta_C) per half-spectrum bin
 *     (Eq 67 / B.2 with the unitary T).  d_r, d_s: device [nrhs][c][N3][N2][N1];
 *     d_feat: device [2C][H1][N3][N2] (C = c(c+1)/2), caller-zeroed, layout [kx][kz][ky].
 *   uno_cg_train_pairs: the mode set K = {|k_i| <= M} as conjugate pairs {k, -k}, ordered by
 *     min(flat(k), flat(-k)) with flat = (kz N2 + ky) N1 + kx; h_bins [npair][2] receives the
 *     half-spectrum bins of each pair (-1: none).
 *   uno_cg_train_newton: `epochs` Newton-Raphson steps (Alg 4 l.3-7; step halved while the
 *     loss increases) on theta_0 (bypass, Eq 43; host [C] in/out) and theta_p (device [npair][C]
 *     in/out), v(k) = psi(theta_0) + [k in K] psi(theta_p(k)) with psi of Eq 45 (c=1: t^2) / B5.
 *     h_loss [epochs+1] (or NULL) receives the loss without the constant delta.
 *   uno_cg_train_install: uses the trained symbol (G(0) = 0) as this handle's preconditioner
 *     and runs the Eq 55 check (UNO_ERR_NOT_SPD if it fails).                               */
UNO_API uno_status uno_cg_train_features(uno_cg_handle* h, const double* d_r, const double* d_s, double scale,
                                         double* d_feat);
UNO_API uno_status uno_cg_train_pairs(uno_cg_handle* h, int32_t M, int64_t* npair, int32_t* h_bins);
UNO_API uno_status uno_cg_train_newton(uno_cg_handle* h, const double* d_feat, int32_t M, int32_t epochs,
                                       double* h_theta0, double* d_thetas, double* h_loss);
UNO_API uno_status uno_cg_train_install(uno_cg_handle* h, int32_t M, const double* h_theta0, const double* d_thetas);

/* Timing of the most recent uno_cg_solve (CUDA events on desc.stream, ms), and the number
 * of library kernels it launched.                                                       */
UNO_API uno_status uno_cg_last_solve_stats(uno_cg_handle* h, double* ms, int64_t* kernel_launches);

/* PCG coefficients of the most recent uno_cg_solve for load case `load`: gamma_1 (= r.s,
 * Alg 2 l.7) and alpha (= gamma_1 / d.p, l.10) of iterations 1..m, recorded on the device by
 * the scalar kernels.  *m_out = m (iterations run); min(m, cap) entries are written to each
 * host array [cap].  UNO_ERR_ARG: null handle / m_out, load outside [0, nrhs), cap < 0, or
 * cap > 0 with a null array.                                                               */
UNO_API uno_status uno_cg_last_coefficients(uno_cg_handle* h, int32_t load, int32_t cap, double* h_gamma,
                                            double* h_alpha, int32_t* m_out);

/* Spectral estimate of the preconditioned operator P A from the most recent solve (PAPER.md
 * Tab 4 columns): the PCG coefficients define the Lanczos tridiagonal T_m of P A,
 *   T[0][0] = 1/alpha_0,  T[j][j] = 1/alpha_j + beta_{j-1}/alpha_{j-1},
 *   T[j][j+1] = T[j+1][j] = sqrt(beta_j)/alpha_j,  beta_j = gamma_{j+1}/gamma_j,
 * whose extreme eigenvalues (host Sturm-sequence bisection) estimate lambda_min / lambda_max
 * of P A from inside (Ritz values).  h_out[5] = {lambda_min, lambda_max, cond_2 = lambda_max /
 * lambda_min, C_CG = (sqrt(cond) - 1)/(sqrt(cond) + 1) (Eq 27), N_iter_est =
 * ln(tol/2)/ln(C_CG) (the Eq 27 bound 2 C^m <= tol, un-rounded; 1 if C_CG <= 0)}; *m_out = m.
 * UNO_ERR_ARG: null pointers, load outside [0, nrhs), tol outside (0, 1), or no iteration
 * recorded (m = 0).                                                                        */
UNO_API uno_status uno_cg_spectrum(uno_cg_handle* h, int32_t load, double tol, double* h_out, int32_t* m_out);

/* Kernel-level timing hook for bench.py: per-kernel-class accumulated device time (ms)
 * and launch counts since create or the last reset, measured with CUDA events on
 * desc.stream when enabled (adds an event pair per launch; off by default).
 *   which: 0 = K apply, 1 = x-pass forward, 2 = y-pass, 3 = G pass, 4 = x-pass inverse,
 *   5 = other.                                                                          */
UNO_API uno_status uno_cg_kernel_timing(uno_cg_handle* h, int32_t enable, int32_t reset, double* ms6, int64_t* count6);

UNO_API const char* uno_cg_last_error(void);
UNO_API const char* uno_cg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* UNO_CG_H */
