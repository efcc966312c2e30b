/*
 * rte_b200.h -- drop-in C-ABI for the batched parametric source-iteration hot
 * path of arxiv 2402.10488 (ROM-enhanced SI with synthetic acceleration),
 * implemented with hand-written sm_100a CUDA kernels (librte_b200.so).
 *
 * The reference exposes this path as a C++ class API (namespace rte, see
 * SURVEY.md s8(b)); every entry point below replaces one reference call for a
 * whole BATCH of parameter samples mu_0..mu_{S-1} at once.  The replaced
 * reference interface is cited per function (paths relative to
 * /root/reference/proj/core/).
 *
 * Conventions
 *   - Plain pointers and sizes only; no exceptions cross the ABI.  Every
 *     function returns RTE_OK (0) or an error code; rte_last_error() gives the
 *     message.  RTE_ERR_INVALID maps to the reference's std::invalid_argument,
 *     RTE_ERR_RUNTIME to std::runtime_error (e.g. singular reduced operator in
 *     romig, strategies.cpp:11-16).  Non-convergence is NOT an error: it is
 *     reported per sample (rte_si_report.converged = 0), as in sisa.cpp:30-47.
 *   - "_dev" pointers are device memory on the context's device, fp64, one
 *     contiguous block per sample: x[s * n_dof + cell * n_local + local]
 *     (the reference's per-sample DOF layout, dg_space.hpp:24).  Kinetic
 *     vectors are direction-major per sample: f[(s * n_dirs + j) * n_dof + i]
 *     (transport_system.hpp:73-89).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *     stream).  Calls are stream-ordered; only rte_si_solve and the rte_*_host
 *     convenience calls synchronize.
 *   - One context per host thread at a time; contexts are independent.
 */
#ifndef RTE_B200_H_
#define RTE_B200_H_

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rte_ctx rte_ctx; /* opaque: one problem batch on one device */

enum rte_status {
  RTE_OK = 0,
  RTE_ERR_INVALID = 1,     /* bad argument (reference: std::invalid_argument) */
  RTE_ERR_RUNTIME = 2,     /* numerical/runtime failure (std::runtime_error) */
  RTE_ERR_CUDA = 3,        /* CUDA error */
  RTE_ERR_UNSUPPORTED = 4  /* valid request outside what this build implements */
};

enum rte_geometry { RTE_SLAB1D = 0, RTE_XY2D = 1 };

/* Problem batch.  Replaces TransportSystem(problem, mesh, space, quad, mu)
 * (transport_system.hpp:32-34, ctor transport_system.cpp:82-109) for S
 * parameter values.  The coefficient closures of ProblemDefinition are given
 * already integrated into per-cell mass blocks (the reference's
 * build_masses, transport_system.cpp:111-140; see rte_weighted_mass below).
 * All pointers are host memory and are copied. */
typedef struct rte_problem {
  int geometry;          /* RTE_SLAB1D or RTE_XY2D */
  int nx, ny;            /* cells (ny ignored for slab) */
  const double* bounds;  /* slab: nx+1 strictly increasing boundaries (Mesh::slab) */
  double x0, x1, y0, y1; /* xy: uniform grid extents (Mesh::rect_uniform) */
  int n_dirs;
  const double* dirs;    /* [n_dirs][3] unit vectors (vx, vy, vz) */
  const double* weights; /* [n_dirs], normalised (sum 1) */
  double inflow[4];      /* isotropic inflow: left, right, bottom, top */
  int n_samples;         /* S >= 1 */
  int block;             /* 1: per-cell scalar sigma (block = sigma * I);
                            n_local^2: full per-cell blocks (slab only) */
  const double* mt;      /* [S][cells][block] total-collision mass blocks */
  const double* ms;      /* [S][cells][block] scattering mass blocks */
  const double* source;  /* [S or 1][n_dof] volumetric source load vector G */
  int source_shared;     /* 1: one G for all samples */
} rte_problem;

/* Affine decomposition sigma(x; mu) = sum_k psi_k(mu) w_k(x) (problem.hpp:
 * 24-29) used by the kinetic term operators (apply_term_kinetic,
 * transport_system.cpp:560-596) and the reduced models
 * (ReducedModel::assemble, reduced_model.cpp:32-39). */
typedef struct rte_affine {
  int k_terms;
  const double* term_mt; /* [K][cells][block] per-term total mass blocks */
  const double* term_ms; /* [K][cells][block] per-term scattering blocks */
  const double* psi;     /* [S][K], psi[s][0] must be 1 */
} rte_affine;

/* Online reduced model (ReducedModel, reduced_model.hpp:19-44). Host memory,
 * column-major like the reference's Eigen storage. */
typedef struct rte_rom {
  int rank;              /* r */
  int k_affine;          /* K */
  const double* u_rho;   /* [r][n_dof] column-major n_dof x r */
  const double* u_iso;   /* [r][n_dof] column-major n_dof x r */
  const double* a_r;     /* [K][r][r] column-major r x r */
  const double* b_r;     /* [r] */
  double eps_pod;
  double eps_train;
} rte_rom;

enum rte_method {
  RTE_SI = 0,     /* plain source iteration (strategy == nullptr) */
  RTE_DSA = 1,    /* DsaStrategy (solvers.hpp:54-65) */
  RTE_ROMSA = 2,  /* RomsaStrategy (strategies.hpp:25-46) on the correction model */
  RTE_ROMSAD = 3, /* RomsadStrategy (strategies.hpp:48-67) */
  RTE_ROMIG = 4,  /* romig initial guess (strategies.cpp:8-28) + DSA */
  RTE_CUSTOM = 5  /* caller-supplied CorrectionStrategy (solvers.hpp:38-51) via rte_si_config.correct */
};

/* The CorrectionStrategy plugin point (solvers.hpp:38-51) for RTE_CUSTOM:
 * called once per SI iteration l (1-based) after the stop test, on the
 * solve's stream, with active_host[s] = 1 for every sample that needs a
 * correction this iteration.  delta_dev = rho* - rho [S][n_dof] (device);
 * the callback writes corr_dev[s] for active samples (device, stream-ordered
 * before it returns) and kind_host[s] = the strategy's last_kind() letter
 * ('D', 'R', 'S', ...) or 0 for "no correction" (rho = rho*).  The next
 * iterate is rho = rho* + corr (sisa.cpp:128-130).  Nonzero return aborts the
 * solve with RTE_ERR_RUNTIME.  strategy.setup(system) is the caller's job
 * before rte_si_solve. */
typedef int (*rte_correction_fn)(void* user, int l, int n_samples, long n_dof, const int* active_host,
                                 const double* delta_dev, double* corr_dev, char* kind_host, void* stream);

enum rte_norm { RTE_NORM_ABS = 0, RTE_NORM_REL = 1 };

typedef struct rte_si_config {
  int method;          /* rte_method */
  double eps;          /* stop tolerance (SolveConfig::eps_sisa) */
  int norm;            /* RTE_NORM_ABS: ||rho*-rho||_inf < eps (sisa.cpp:123);
                          RTE_NORM_REL: ||rho*-rho||_inf / ||rho*||_inf < eps */
  int max_iters;       /* SolveConfig::max_iters */
  int fixed_iters;     /* > 0: run exactly this many iterations, no stop test */
  int theta;           /* ROMSAD switch iteration budget */
  double eps_romsad;   /* ROMSAD switching tolerance (romsad_tolerance) */
  int use_guess;       /* 1: rho_dev holds the initial guess on entry */
  int compute_residual;/* 1: final ||rho - L rho - bbar||_inf (one extra sweep) */
  int check_every;     /* host polls the active count every k iterations (0 = 4) */
  rte_correction_fn correct; /* RTE_CUSTOM only */
  void* correct_user;        /* passed through to correct */
  double dsa_inner;    /* xy DSA only; 0: every correction solved to the DSA tolerance
                          (rte_dsa_set_tolerance, default 1e-12 relative); c in (0,1):
                          iteration l solves to relative residual max(tol, c * eps / change_l)
                          ("inner tolerance 1e-2 eps_SISA"; ignored with fixed_iters) */
  double dsa_floor;    /* xy DSA only; c > 0: iteration l also accepts relative residual
                          min(0.1, c * 2^-53 * ||rho*||_inf / ||rho* - rho||_inf): the accuracy
                          below which the correction cannot move the iterate by more than about
                          c ulps of rho* times the correction's gain (round-off floor of the
                          outer iteration; applies with fixed_iters too).  0: off */
} rte_si_config;

/* Per-sample outcome of the iterative XY DSA solves (the reference's direct
 * SparseLU cannot under-solve; its failures throw, dsa.cpp:253-256, 269-271). */
enum rte_dsa_status {
  RTE_DSA_OK = 0,
  RTE_DSA_MAXIT = 1,      /* stopped at the iteration cap above the tolerance */
  RTE_DSA_BREAKDOWN = 2,  /* BiCGStab breakdown (omega = 0) above the tolerance */
  RTE_DSA_NAN = 3         /* non-finite residual */
};

typedef struct rte_si_report {
  int converged;
  int iterations;
  long n_sweep;        /* reference accounting: 1 (bbar) + iterations */
  int switch_iter;     /* ROMSAD: first iteration corrected by DSA (-1: none) */
  int singular;        /* reduced operator singular at this mu */
  double final_residual;
  double last_change;
  int dsa_status;      /* worst rte_dsa_status over this sample's DSA corrections */
} rte_si_report;

/* ---- lifecycle ---------------------------------------------------------- */
int rte_create(const rte_problem* p, int device, rte_ctx** out);
void rte_destroy(rte_ctx* ctx);
const char* rte_last_error(const rte_ctx* ctx); /* ctx may be NULL (create failures) */
long rte_n_dof(const rte_ctx* ctx);
int rte_n_samples(const rte_ctx* ctx);
int rte_n_slots(const rte_ctx* ctx); /* unique (vx,vy) sweep slots (transport_system.cpp:194-202) */
/* XY sweep work decomposition the context's full sweeps use: directions per
 * lane (8, 4, 2 or 1) and direction groups per quadrant (slab: 0, 0).
 * Diagnostic; RTE_SWEEP_DPL (environment, read per call) forces the first. */
int rte_sweep_plan(rte_ctx* ctx, int* dirs_per_lane, int* groups);

/* ---- transport operator (batched over samples) -------------------------- */
/* Device vectors are [n_samples][n_dof] doubles, contiguous, 16-byte aligned
 * (the XY sweep stages them with 16-byte bulk copies; a misaligned pointer is
 * RTE_ERR_INVALID). */
/* TransportSystem::apply_L (transport_system.cpp:393-404): out = L rho. */
int rte_apply_L(rte_ctx* ctx, const double* rho_dev, double* out_dev, void* stream);
/* TransportSystem::assemble_rhs (transport_system.cpp:406-418): bbar. */
int rte_assemble_rhs(rte_ctx* ctx, double* bbar_dev, void* stream);
/* Fused fixed-point map rho* = L rho + bbar in ONE sweep (identical in exact
 * arithmetic to apply_L + assemble_rhs, sisa.cpp:118). */
int rte_fixed_point(rte_ctx* ctx, const double* rho_dev, double* out_dev, void* stream);
/* TransportSystem::sweep_direction (transport_system.cpp:366-371) for
 * direction j of every sample: f = (D_j + Sigma_t)^{-1} rhs. */
int rte_sweep_direction(rte_ctx* ctx, int j, const double* rhs_dev, double* f_dev, void* stream);
/* TransportSystem::kinetic_sweep (transport_system.cpp:420-431). */
int rte_kinetic_sweep(rte_ctx* ctx, const double* rho_dev, double* f_dev, void* stream);
/* TransportSystem::density_of (transport_system.cpp:433-441). */
int rte_density_of(rte_ctx* ctx, const double* f_dev, double* rho_dev, void* stream);
/* TransportSystem::apply_Ms / apply_Mt (transport_system.cpp:373-391). */
int rte_apply_Ms(rte_ctx* ctx, const double* x_dev, double* out_dev, void* stream);
int rte_apply_Mt(rte_ctx* ctx, const double* x_dev, double* out_dev, void* stream);

/* ---- affine terms / kinetic operators ---------------------------------- */
int rte_set_affine(rte_ctx* ctx, const rte_affine* aff);
/* TransportSystem::apply_term_kinetic (transport_system.cpp:560-596) for
 * sample 0's discretization (term operators are parameter independent);
 * u/out: [n_cols][n_dirs * n_dof]. */
int rte_apply_term_kinetic(rte_ctx* ctx, int k, int n_cols, const double* u_dev, double* out_dev,
                           void* stream);
/* apply_kinetic (transport_system.cpp:598-613): out = A_mu u = sum_k psi_k(mu)
 * A_k u for every sample; u/out [S][n_dirs * n_dof] (distinct buffers).
 * Requires rte_set_affine. */
int rte_apply_kinetic(rte_ctx* ctx, const double* u_dev, double* out_dev, void* stream);
/* apply_streaming_collision (transport_system.cpp:482-558): out = (D_j +
 * Sigma_t) f for direction j with zero inflow; f/out [S][n_dof] (distinct). */
int rte_apply_streaming_collision(rte_ctx* ctx, int j, const double* f_dev, double* out_dev, void* stream);
/* kinetic_rhs (transport_system.cpp:615-624): block j = G + g_j^bc per sample;
 * out [S][n_dirs * n_dof]. */
int rte_kinetic_rhs(rte_ctx* ctx, double* out_dev, void* stream);

/* collect_snapshots (snapshots.cpp:118-194) for every sample: training
 * SI-DSA in kinetic form, stopping on ||drho||_inf < eps_train.  Stores
 * f^(l) for l <= window in f_iter_dev [S][window][n_dirs*n_dof], drho^(l) in
 * drho_dev [S][window][n_dof] and the last (converged) f in f_conv_dev
 * [S][n_dirs*n_dof].  converged_host[S], n_iter_host[S] (w_mu =
 * min(n_iter, window)). */
int rte_collect_snapshots(rte_ctx* ctx, int window, double eps_train, int max_iters, double* f_iter_dev,
                          double* f_conv_dev, double* drho_dev, int* converged_host, int* n_iter_host);

/* Training matrices from rte_collect_snapshots output (PrimarySource /
 * CorrectionSource, snapshots.cpp:316-376): kind 0 = converged solutions,
 * kind 1 = correction columns f - f^(l), l <= min(n_iter, window,
 * window_limit); converged samples only.  out_dev (may be NULL to count)
 * [n_cols][n_dirs*n_dof]; *n_cols receives the column count. */
int rte_snapshot_columns(rte_ctx* ctx, int window, const double* f_iter_dev, const double* f_conv_dev,
                         const int* n_iter_host, const int* converged_host, int kind, int window_limit,
                         double* out_dev, int* n_cols);

/* ---- POD and Galerkin projections (pod.cpp, reduced_model.cpp) ----------- */
/* POD of F (m x n column-major, device; m >= n, n <= 128): all n singular
 * values to sigma_host (descending) and the first rank_max left singular
 * vectors to U_dev (m x rank_max, column-major).  Shifted CholeskyQR3 on the
 * device + one-sided Jacobi SVD of the n x n factor (replaces dgesdd / TSQR,
 * pod.cpp:81-94, 173-276). */
int rte_pod(int device, long m, int n, const double* F_dev, int rank_max, double* U_dev, double* sigma_host,
            void* stream);
/* truncation_rank (pod.cpp:117-139). */
int rte_truncation_rank(const double* sigma, int n, double eps_pod);
/* build_reduced_model (reduced_model.cpp:106-199) on the device from a basis
 * U_dev (n_dirs*n_dof x r, column-major) with the context's (sample-
 * independent) term operators; outputs in the rte_rom layout to host arrays.
 * RTE_ERR_RUNTIME if ||U^T U - I||_max > 1e-10 (reduced_model.cpp:189-194). */
int rte_build_rom(rte_ctx* ctx, int r, const double* U_dev, double* u_rho_host, double* u_iso_host,
                  double* a_r_host, double* b_r_host);

/* ---- DSA (dsa.cpp) ----------------------------------------------------- */
/* DsaOperator ctor (dsa.cpp:154-258): assemble + factor per sample. */
int rte_dsa_setup(rte_ctx* ctx, void* stream);
/* DsaOperator::solve_density (dsa.cpp:264-273). */
int rte_dsa_solve_density(rte_ctx* ctx, const double* rhs_dev, double* out_dev, void* stream);
/* DsaOperator::correct (dsa.cpp:275-277): C * Ms * delta. */
int rte_dsa_correct(rte_ctx* ctx, const double* delta_dev, double* out_dev, void* stream);
/* XY geometry: the coupled system is solved iteratively (BiCGStab with a
 * multigrid V-cycle preconditioner) to relative residual `tol` (default
 * 1e-12) within `max_iters` (default 1000); <= 0 keeps the current value.
 * The reference uses a direct SparseLU (dsa.cpp:253). */
int rte_dsa_set_tolerance(rte_ctx* ctx, double tol, int max_iters);
/* Krylov iterations of the last XY DSA solve (0 for slab: direct). */
int rte_dsa_last_iterations(const rte_ctx* ctx);
/* Krylov iteration counts (max over the samples) of the XY DSA solves since
 * the start of the last rte_si_solve / rte_gmres_solve (or since the last
 * direct DSA call): returns the number of solves logged (0 for slabs, < 0 on
 * a device error) and writes the first min(that, cap) counts to out.  Inside
 * rte_si_solve there is one entry per trip of the device loop; trips after
 * the last sample stopped (the host polls the active count every check_every
 * iterations) are masked and log 0. */
int rte_dsa_iteration_log(const rte_ctx* ctx, int* out, int cap);
/* The XY solve starts from the minimal-residual combination of the sample's
 * last solutions (a warm start; the history holds up to 8 solution vectors and
 * their operator images, up to half of the free device memory, for the
 * context's lifetime).  Direct rte_dsa_solve_density / rte_dsa_correct calls
 * warm-start from the earlier calls' solutions (results agree within the
 * solver tolerance, not bitwise); rte_si_solve and rte_gmres_solve clear the
 * history when they start, so a solve does not depend on earlier calls.  This
 * clears it explicitly.  Direct solves that end above the tolerance return
 * RTE_ERR_RUNTIME (the reference throws, dsa.cpp:269-271). */
int rte_dsa_reset_history(rte_ctx* ctx, void* stream);
/* DsaOperator::apply_eliminated (dsa.cpp:279-293, dsa.hpp:43-46): the
 * current-eliminated density operator S x = A_rr x - A_rJ T^{-1} A_Jr x for
 * every sample.  The current block T is factored lazily on first use (slab:
 * block cyclic reduction; XY: solved by CG to relative residual 1e-13).
 * x and out are [S][ndof] device buffers and must not alias. */
int rte_dsa_apply_eliminated(rte_ctx* ctx, const double* x_dev, double* out_dev, void* stream);
/* DsaOperator::coupled_dim (dsa.hpp:48). */
long rte_dsa_coupled_dim(const rte_ctx* ctx);

/* ---- reduced models (reduced_model.cpp, strategies.cpp) ----------------- */
/* which: 0 = primary model (ROMIG), 1 = correction model (ROMSA/ROMSAD).
 * Requires rte_set_affine (psi per sample). */
int rte_rom_load(rte_ctx* ctx, int which, const rte_rom* rom);
/* romig (strategies.cpp:8-28) for every sample: rho0 = U_rho A_r(mu)^{-1} b_r.
 * status_host[s] = 0 ok, 1 singular, 2 Galerkin residual check failed. */
int rte_romig(rte_ctx* ctx, double* rho0_dev, int* status_host, void* stream);

/* ---- source iteration (sisa.cpp:14-54) ----------------------------------- */
/* Batched sisa_solve: all samples iterate on the device; converged samples
 * are masked.  rho_dev [S][n_dof] holds the guess on entry (use_guess) and
 * the solution on exit.  reports_host[S]; history_host [S][max_iters] (change
 * per iteration, may be NULL); log_host [S][max_iters] correction kinds
 * 'D','R','S' or 0 (may be NULL).  Of each row only the first W entries are
 * written (W = the largest iteration count of the batch; entries past a
 * sample's own count are 0); the rest is left untouched.  fixed_iters > max_iters is RTE_ERR_INVALID.
 * A DSA correction that ends above its tolerance (rte_dsa_status) fills the
 * reports and returns RTE_ERR_RUNTIME (dsa.cpp:269-271 throws). */
int rte_si_solve(rte_ctx* ctx, const rte_si_config* cfg, double* rho_dev, rte_si_report* reports_host,
                 double* history_host, char* log_host);

/* ---- (P)GMRES (gmres.cpp:15-124) ------------------------------------------ */
enum rte_gmres_guess { RTE_GUESS_ZERO = 0, RTE_GUESS_SUPPLIED = 1, RTE_GUESS_ROMIG = 2 };

typedef struct rte_gmres_config {
  int preconditioned;  /* 1: P = I + C Ms with the consistent DSA operator (PGMRES); 0: GMRES */
  int restart;         /* SolveConfig::gmres_restart (reference default 25) */
  double rel_tol;      /* SolveConfig::gmres_rel_tol: preconditioned relative residual (1e-11) */
  int max_iters;       /* SolveConfig::max_iters: cap on inner iterations */
  int guess;           /* rte_gmres_guess; RTE_GUESS_ROMIG = PGMRES-ROMIG (runner.cpp:202-205),
                          needs the primary model (rte_rom_load which = 0) */
} rte_gmres_config;

typedef struct rte_gmres_report {
  int converged;
  int iterations;      /* inner iterations (SolveReport::iterations) */
  long n_sweep;        /* reference accounting: 1 (bbar) + 1 per cycle start + 1 per inner step */
  int cycles;          /* restart cycles started */
  double final_residual; /* converged: ||A rho - bbar||_inf of the verifying cycle start;
                            else ||rho - L rho - bbar||_inf */
  int history_len;     /* SolveReport::change_history size (entries beyond history_cap dropped) */
  int dsa_status;      /* worst rte_dsa_status over this sample's preconditioner solves */
} rte_gmres_report;

/* Batched gmres_solve for every sample: rho_dev [S][n_dof] holds the guess on
 * entry (RTE_GUESS_SUPPLIED) and the solution on exit; reports_host[S];
 * history_host [S][history_cap] (may be NULL).  Synchronizes once per step
 * (one transport sweep + one DSA solve for every unfinished sample). */
int rte_gmres_solve(rte_ctx* ctx, const rte_gmres_config* cfg, double* rho_dev, rte_gmres_report* reports_host,
                    double* history_host, int history_cap);

/* ---- measurement ---------------------------------------------------------- */
/* Per-context kernel timing with CUDA events recorded on the launching stream
 * around every kernel the context issues, by category.  Off by default. */
enum rte_prof_kind { RTE_PROF_SWEEP = 0, RTE_PROF_REDUCE = 1, RTE_PROF_DSA = 2, RTE_PROF_ROM = 3,
                     RTE_PROF_OTHER = 4, RTE_PROF_DSA_SMOOTH0 = 5, RTE_PROF_KINDS = 6 };
/* RTE_PROF_DSA_SMOOTH0 times the finest-level XY DSA smoother half-sweeps
 * individually (they are also included in RTE_PROF_DSA). */
int rte_profile_enable(rte_ctx* ctx, int on);
/* Synchronizes, returns summed milliseconds and launch counts per kind since
 * the last read, and clears them. */
int rte_profile_read(rte_ctx* ctx, double* ms_by_kind, long* launches_by_kind);
/* FP64 FMA throughput probe (independent DFMA chains on every SM): the
 * denominator for fp64_fraction.  Returns TFLOP/s (2 flops per FMA). */
int rte_probe_dfma(int device, double* tflops);

/* ---- host-side discretization helpers (problem setup) ------------------- */
/* quadrature.cpp:8-39: n-point Gauss-Legendre nodes/weights on [-1,1]. */
int rte_gauss_legendre_nodes(int n, double* x, double* w);
/* weighted_mass (transport_system.cpp:17-55) for every cell: wvals holds the
 * coefficient values at the cell points returned by rte_cell_points;
 * out [cells][n_local^2]. */
int rte_cell_points(int geometry, int nx, int ny, const double* bounds, double x0, double x1, double y0,
                    double y1, int nq, double* px, double* py);
int rte_weighted_mass(int geometry, int nx, int ny, const double* bounds, double x0, double x1, double y0,
                      double y1, int nq, const double* wvals, double* out);
/* project (dg_space.cpp:31-71) from values at the cell points. */
int rte_project(int geometry, int nx, int ny, const double* bounds, double x0, double x1, double y0,
                double y1, int nq, const double* fvals, double* out);
/* The same for a weight / function that is one constant at every point
 * (identical arithmetic; no per-point value array). */
int rte_weighted_mass_const(int geometry, int nx, int ny, const double* bounds, double x0, double x1, double y0,
                            double y1, int nq, double w, double* out);
int rte_project_const(int geometry, int nx, int ny, const double* bounds, double x0, double x1, double y0,
                      double y1, int nq, double f, double* out);
/* Batch assembly helpers (the TransportSystem constructor's build_masses,
 * transport_system.cpp:111-140, for S samples): rte_scalar_blocks reduces
 * per-cell blocks [n][nl*nl] to scalars when every block is d0 I to 1e-12
 * (else RTE_ERR_UNSUPPORTED); rte_combine_terms forms out[s][e] =
 * sum_k psi[s][k] terms[k][e] in ascending k, products rounded before adds. */
int rte_scalar_blocks(long n, int nl, const double* m, double* out);
int rte_combine_terms(int S, int K, long n, const double* psi, const double* terms, double* out);
/* cases.cpp:11-13: n unit draws (gen() >> 11) * 2^-53 of std::mt19937_64(seed). */
int rte_unit_draws(unsigned long long seed, long n, double* out);

/* Bounds checking without compute-sanitizer (not available on the GPU pool).
 * With RTE_GUARD=1 in the environment every library device allocation is
 * padded by 4 KB guard zones of 0xFF bytes (its user region starts filled
 * with the same pattern: NaN as fp64/fp32), so out-of-bounds writes are
 * counted here and out-of-bounds / uninitialised reads surface as NaN.
 * rte_guard_check: violations found so far (freed and live buffers) and the
 * number of guard checks made; RTE_ERR_UNSUPPORTED without RTE_GUARD.
 * rte_guard_selftest: writes one element past a 10-double allocation (the
 * check must then report it). */
int rte_guard_check(long* violations, long* checked);
int rte_guard_selftest(int device);

#ifdef __cplusplus
}
#endif
#endif /* RTE_B200_H_ */
