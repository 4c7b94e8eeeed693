/*
 * st.h — C ABI of the B200-native all-at-once space-time solver (libst.so).
 *
 * Method: arxiv 2508.09589 (Alexandersen & Appel). The library solves the stabilised
 * continuous-Galerkin space-time finite-element system of transient heat conduction
 *     K(rho) T = f            (sec. 3.1.2; weak form PAPER.md:338-353)
 * its adjoint (transposed) system
 *     K(rho)^T lambda = dphi/dT   (sec. 3.3.3)
 * and the element sensitivities
 *     dphi/drho_e = -lambda^T (dK/drho_e) T
 * with FGMRES right-preconditioned by one space-time geometric multigrid
 * V-cycle per iteration on the semi-coarsened hierarchy of Algorithm 1,
 * Galerkin coarse operators J_{l+1} = P_l^T J_l P_l.
 *
 * Conventions:
 *  - All floating point is IEEE fp64.
 *  - Coordinates are the rescaled ones: x in [0,1]^sdim, t in [0,1];
 *    k~ = k tau / L^2, Q~ = Q tau (Delta T = 1).
 *  - Node layout: index = i1 + (n+1)*(i2 + (n+1)*([i3 + (n+1)*] it)), x1 fastest, t slowest.
 *    N_n = (n+1)^sdim (nt+1) doubles per nodal vector (T, lambda, dJdT, f).
 *  - Element layout of rho and dJ: space-time design (ST_SPACE_TIME): [nt][n]..[n] (x1
 *    fastest), n^sdim nt doubles; time-constant design (ST_TIME_CONSTANT, the extruded design
 *    of PAPER.md:262, 604-608): [n]..[n], n^sdim doubles, and dJ is summed through time.
 *  - Pointers may be DEVICE pointers (current device of the context) or HOST pointers;
 *    the library detects host memory (cudaPointerGetAttributes) and stages it through
 *    device buffers inside the call. Caller owns every vector; the context owns workspaces.
 *  - Every call enqueues on the context's stream and returns after completion. Without a
 *    caller stream the context creates a blocking stream (ordered with the legacy default
 *    stream, e.g. PyTorch's default stream).
 *  - Dirichlet data (R-1..R-4): T = T0 on the t = 0 node plane (initial
 *    condition); T = 0 on the sink patch of the face x1 = 0 (all t, including t = 0) whose
 *    transverse coordinates lie within halfwidth of center. Symmetric elimination with
 *    unit diagonal.
 *  - Return value: ST_OK or a negative ST_E_* code; st_strerror() gives text.
 *    No C++ exception crosses this boundary.
 */
#ifndef ST_H_
#define ST_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ST_ABI_VERSION 3

enum {
  ST_OK = 0,
  ST_E_INVALID_ARG = -1,   /* bad size, null pointer, non-square grid, n < 2      */
  ST_E_DIVISIBILITY = -2,  /* a level cannot be halved in the direction Algorithm 1 picks      */
  ST_E_NOT_CONVERGED = -3, /* maxit reached; best iterate written and stats filled             */
  ST_E_BREAKDOWN = -4,     /* Krylov breakdown (zero norm / non-finite value)                   */
  ST_E_OOM = -5,           /* device allocation failed                                          */
  ST_E_CUDA = -6,          /* CUDA runtime error (text via st_strerror / st_last_error)         */
  ST_E_NCCL = -7,          /* communicator error                                                */
  ST_E_UNSUPPORTED = -8    /* option combination not implemented                                */
};

enum { ST_TIME_CONSTANT = 0, ST_SPACE_TIME = 1 };
/* Sources (rescaled units, R-7): UNIFORM Q~ = Q0 tau; SIN Q~ = Q0 tau (1 + a sin(w tau t));
 * the paper's examples, Q0 given already rescaled (no tau factor): EX1 Q~ = 1/2 Q0 (1 - t)(1 + cos 50 t)
 * (Example 1, Q0 = 100); EX2 Q~ = Q0 exp(-|x - x0(t)|^2 / (2 sigma^2)) with
 * x0(t) = (1/2 + R cos(w tau t + pi/2), 1/2 + R sin(w tau t + pi/2)) (Example 2: Q0 = 1,
 * sigma = 0.05, R = 0.25, w = pi, tau = 6; (2+1)D only). */
enum { ST_SRC_UNIFORM = 0, ST_SRC_SIN = 1, ST_SRC_EX1 = 2, ST_SRC_EX2 = 3 };
/* Smoothers: damped Jacobi (default); the paper's GMRES(k)-Jacobi smoother
 * (k = nu_pre / nu_post fixed steps, <= 24; one GPU). ST_SMOOTH_CHEBYSHEV is reserved
 * (ST_E_UNSUPPORTED). */
enum { ST_SMOOTH_JACOBI = 0, ST_SMOOTH_CHEBYSHEV = 1, ST_SMOOTH_GMRES = 2 };
/* Outer Krylov method: FGMRES(m) keeps the m preconditioned vectors
 * Z_j = M V_j; right-preconditioned GMRES(m) keeps only the basis V and forms x += M (V y) with one more
 * V-cycle per restart (valid because the Jacobi V-cycle is a fixed linear map; m fewer full-length
 * vectors — the memory plan of config 3 on one GPU). The GMRES smoother is not a
 * fixed linear map: ST_KRYLOV_GMRES requires ST_SMOOTH_JACOBI. */
enum { ST_KRYLOV_FGMRES = 0, ST_KRYLOV_GMRES = 1 };
/* Coarsest-level solver: exact dense inverse (default, <= 4096 stored nodes) or the paper's GMRES(<= coarse_maxit)
 * with Jacobi preconditioning to coarse_rtol (200 iterations, rtol 1e-6). */
enum { ST_COARSE_DENSE = 0, ST_COARSE_GMRES = 1 };
/* Stencil-kernel family (test / experiment hook; every family computes the same operator): the TMA
 * kernels where they apply (default), the cp.async-ring kernels, or the generic kernels only. */
enum { ST_KERNELS_TMA = 0, ST_KERNELS_CPASYNC = 1, ST_KERNELS_GENERIC = 2, ST_KERNELS_TMA2D = 3 };

/* Regular space-time mesh of n^sdim x nt elements. L, tau only rescale. */
typedef struct {
  int32_t sdim;   /* 2 ((2+1)D, 8-node trilinear hex) or 3 ((3+1)D, 16-node element)   */
  int64_t n;      /* elements per spatial direction (square/cubic elements)            */
  int64_t nt;     /* time elements                                                     */
  double L, tau;  /* characteristic length and final time           */
} st_grid_t;

/* Modified SIMP: C = C_ins + (C_con-C_ins) rho^p_c,
 * k = k_ins + (k_con-k_ins) rho^p_k; k~ = k tau / L^2. */
typedef struct { double C_ins, C_con, p_c, k_ins, k_con, p_k; } st_materials_t;

/* Dirichlet data. face: 0 = x1 = 0 (only face implemented). */
typedef struct {
  double T0;          /* value on the t = 0 node plane                                   */
  int32_t has_patch;  /* 0 => insulated everywhere except the IC                         */
  int32_t face;
  double center, halfwidth; /* fractions of L; BASELINE default 0.5, 0.05               */
  int32_t all_walls;  /* 1: T = 0 on every spatial boundary node at all t (Example 2's cold
                         walls) instead of the patch                         */
} st_bcs_t;

/* Source (kinds above): UNIFORM Q0;  SIN: Q0 (1 + a sin(w t_phys)), t_phys = tau t; EX1; EX2 (sigma, R). */
typedef struct { int32_t kind; double Q0, a, w, sigma, R; } st_source_t;

typedef struct {
  int32_t design_mode;      /* ST_TIME_CONSTANT | ST_SPACE_TIME                          */
  double rtol;              /* FGMRES stop: true ||b - K T|| / ||b|| <= rtol              */
  int32_t maxit;            /* max outer iterations (total over restarts)                */
  int32_t restart;          /* FGMRES restart length m                                   */
  int32_t smoother;         /* ST_SMOOTH_JACOBI | ST_SMOOTH_GMRES                        */
  int32_t nu_pre, nu_post;  /* Jacobi sweeps / GMRES smoother steps (pre, post)          */
  double omega;             /* Jacobi damping                                            */
  double lambda_crit;       /* Algorithm 1 threshold (0.5)                 */
  int64_t coarse_max_nodes; /* stop coarsening at <= this many nodes (R-19)     */
  int32_t max_levels;       /* 0 = unlimited                                             */
  int32_t full_coarsening;  /* 1 = coarsen space and time together    */
  int32_t use_graphs;       /* 1 (default): every replicated coarse level of the V-cycle runs as
                               one CUDA graph launch per cycle                              */
  int32_t verbose;
  int64_t agg_nodes;        /* time slabs: agglomerate a level once it has fewer than this
                               many nodes per rank (default 262144)                         */
  int32_t nu_coarse;        /* Jacobi sweeps (pre = post) on the coarse levels; 0 = nu_pre /
                               nu_post there too (default 5; nu_pre = nu_post = 2 on the fine
                               level: DESIGN.md sec. 9)                                     */
  /* ---- ABI 3: every former environment knob is an option, read per call ---------------- */
  int32_t krylov;           /* ST_KRYLOV_FGMRES (default) | ST_KRYLOV_GMRES                     */
  int32_t coarse_solver;    /* ST_COARSE_DENSE (default) | ST_COARSE_GMRES                      */
  double coarse_rtol;       /* ST_COARSE_GMRES: relative residual target (default 1e-6)          */
  int32_t coarse_maxit;     /* ST_COARSE_GMRES: iteration cap (default 200)                      */
  int32_t kernel_family;    /* ST_KERNELS_* (default ST_KERNELS_TMA)                             */
  int32_t chunk_planes;     /* persistent stencil kernels: planes per time chunk of the work list;
                               0 = automatic, > 0 forced, < 0 no chunking   */
  int32_t max_ctas;         /* persistent stencil kernels: cap on the grid (0 = one full wave);
                               a small cap makes every CTA walk long multi-tile plane runs; < 0:
                               tv2d trims the wave so the tiles form equal full groups (exp.)   */
  int32_t fuse_prolong;     /* 1 (default): prolongation + correction fused into the first
                               post-sweep where a kernel supports it; 0: separate kernels      */
  double omega_factor;      /* per-level Jacobi weight omega_l = min(omega, omega_factor / R_l)
                               (default 1.9)                                 */
  double dgks_eta;          /* FGMRES re-orthogonalisation when ||w'|| < dgks_eta ||w|| (0.1)   */
  int64_t graph_max_nodes;  /* replicated levels below this many nodes run in the V-cycle's
                               CUDA graph (0 = every replicated coarse level)                  */
  double smoother_rtol;     /* ST_SMOOTH_GMRES: stop the inner GMRES once ||r|| <= smoother_rtol
                               ||r0|| (1e-6); 0 = fixed nu steps (graph-capturable) */
  int64_t nu_fine_nodes;    /* coarse levels with at least this many nodes use the fine-level sweep
                               counts nu_pre / nu_post instead of nu_coarse (their sweeps cost HBM
                               passes, not launch latency); 0 = level 0 only  */
  int32_t pitch_align;      /* row pitch of the internal vectors rounded up to a multiple of this many
                               doubles (even; 2 = 16-byte rows, the TMA minimum; default 4 = one
                               DRAM sector)                                                     */
} st_options_t;

/* Distribution over time slabs. NULL or size == 1 => one GPU.
 * Rank r owns element layers [r nt/G, (r+1) nt/G) and node planes (r nt/G, (r+1) nt/G]
 * (rank 0 also plane 0); nt must be divisible by G. Every level of the multigrid hierarchy whose
 * time extent still divides into G slabs stays distributed; the coarser levels are gathered
 * onto every rank and solved redundantly (agglomeration).
 * Transports: ST_COMM_NCCL — nccl_comm is an ncclComm_t of `size` ranks (one GPU each; see
 * st_nccl_unique_id / st_nccl_comm_init); halo planes with grouped ncclSend/ncclRecv, Krylov
 * sums with ncclAllReduce, agglomeration with ncclAllGather, all on cuda_stream.
 * ST_COMM_HOST — the caller's host callbacks (below) move pinned host buffers; any number of
 * ranks may share one GPU (used by the tests). Callbacks return 0 on success. */
enum { ST_COMM_NONE = 0, ST_COMM_NCCL = 1, ST_COMM_HOST = 2 };
#define ST_NCCL_ID_BYTES 128
typedef struct {
  void* user;
  /* exchange `count` doubles with `peer`: send `send`, receive into `recv` (host memory) */
  int (*sendrecv)(void* user, int32_t peer, const double* send, double* recv, int64_t count);
  /* in-place elementwise sum over all ranks of `count` doubles (host memory) */
  int (*allreduce_sum)(void* user, double* buf, int64_t count);
  /* recv[size * count] = concatenation over ranks (in rank order) of send[count] */
  int (*allgather)(void* user, const double* send, double* recv, int64_t count);
} st_host_comm_t;
typedef struct {
  void* nccl_comm;
  int32_t rank, size;
  void* cuda_stream;
  int32_t device;
  int32_t transport;          /* ST_COMM_* (size > 1)                                        */
  st_host_comm_t host;        /* ST_COMM_HOST                                                 */
} st_dist_t;

/* Local slab of this rank (caller vector layout). T, lambda, dJdT: the owned node planes
 * [plane0, plane0 + n_planes), dense, x1 fastest. rho (space-time design): element layers
 * [layer0, layer0 + rho_layers) = the owned layers plus, except on the last rank, the first
 * layer of the next slab (its ghost); dJ: the owned layers [layer0, layer0 + n_layers).
 * Time-constant design: rho and dJ are the full spatial field on every rank (dJ summed over
 * all ranks' layers). */
typedef struct {
  int32_t rank, size;
  int64_t plane0, n_planes;
  int64_t layer0, n_layers, rho_layers;
  int64_t nodes_local;        /* n_planes (n+1)^sdim                                         */
  int64_t design_local;       /* entries of rho this rank passes                             */
  int32_t n_levels, n_dist_levels;
} st_layout_t;

typedef struct st_ctx st_ctx_t;

typedef struct {
  int32_t iterations;        /* outer FGMRES iterations of the last solve                 */
  int32_t restarts;
  double rel_residual;       /* final TRUE relative residual ||b - K x|| / ||b||          */
  double setup_ms, solve_ms; /* last rho-dependent setup and last solve, device ms         */
  int32_t n_levels;
  int32_t converged;
  int32_t vcycles;           /* V-cycles of the last solve (GMRES: iterations + restarts)  */
  int64_t setups;            /* rho-dependent rebuilds since st_setup (design changes seen) */
} st_stats_t;

typedef struct {
  int32_t n_levels;
  int64_t n[32], nt[32];     /* elements per level                                        */
  int32_t kind[32];          /* 0 fine, 1 space, 2 time, 3 full                            */
  int32_t form[32];          /* operator storage: 0 matrix-free (rho), 1 MK, 2 block-4, 3 dense */
  int64_t nodes[32];
  double omega[32];          /* damped-Jacobi weight of the level (last design)                */
  double lam_max[32];        /* Gershgorin bound on |lambda|_max(D^-1 A)     */
} st_hierarchy_t;

/* Fill `o` with the library defaults (rtol 1e-8, restart 16, FGMRES, Jacobi nu 2/2 on the fine level and
 * 5/5 on the coarse levels, weight cap 0.75, omega_factor 1.9, lambda_crit 0.5, coarse_max_nodes 400, dense
 * coarsest solve, agg_nodes 262144, TMA kernels, automatic chunking, both transfer fusions on). */
void st_default_options(st_options_t* o);

/* Validate, run Algorithm 1, allocate all workspaces, assemble f on the device.
 * Errors: ST_E_INVALID_ARG, ST_E_DIVISIBILITY, ST_E_OOM, ST_E_CUDA. */
int st_setup(const st_grid_t* grid, const st_materials_t* mats, const st_bcs_t* bcs,
             const st_source_t* src, const st_options_t* opts, const st_dist_t* dist,
             st_ctx_t** out);

void st_destroy(st_ctx_t* ctx);

/* Forward solve K_bc(rho) T = b. T: in = initial guess (warm start,
 * PAPER.md:385), out = solution with prescribed values at constrained nodes.
 * rho: element densities (layout above). Returns ST_OK or ST_E_NOT_CONVERGED (best
 * iterate written). */
int st_solve(st_ctx_t* ctx, const double* rho, double* T);

/* Adjoint solve K_bc(rho)^T lambda = m_f .* dJdT. lambda: in = initial
 * guess, out = solution (0 at constrained nodes). dJdT at constrained nodes is ignored.
 * dJdT = NULL selects the time-integrated thermal compliance phi = f^T T, dphi/dT = f (BASELINE
 * config 1, R-8) without a caller vector for f. */
int st_adjoint(st_ctx_t* ctx, const double* rho, const double* dJdT, double* lambda);

/* Sensitivities dJ_e = -lambda_e^T (dC/drho G + dk~/drho Kx) T_e,
 * summed through time for a time-constant design. */
int st_sensitivity(st_ctx_t* ctx, const double* rho, const double* T, const double* lambda,
                   double* dJ);

/* One design iteration's state work in one call (the per-iteration work of the
 * optimisation loop of PAPER.md sec. 4): st_solve(rho, T), then st_adjoint(rho, dJdT, lambda), then
 * st_sensitivity(rho, T, lambda, dJ), with identical arguments, layouts and results. rho is bound (and
 * a host design copied to the device) once; T and lambda are in = initial guesses, out = solutions;
 * dJdT = NULL selects the compliance. With HOST vectors the result copies overlap the next phase: T
 * goes back to the host on a side stream during the adjoint solve, lambda during the sensitivities,
 * and the sensitivities read T from its device copy (no second upload) — host traffic per call:
 * rho, T, lambda (+ dJdT) in, T, lambda, dJ out. fwd_stats (nullable) receives the forward solve's
 * statistics; st_get_stats afterwards reports the adjoint solve's. Returns ST_OK, or the first
 * solve's ST_E_NOT_CONVERGED (both solves run, all outputs written), or an error. */
int st_design_step(st_ctx_t* ctx, const double* rho, const double* dJdT, double* T, double* lambda,
                   double* dJ, st_stats_t* fwd_stats);

/* Test hook: y = K x (transpose = 0) or K^T x (1); bc = 1 applies the eliminated
 * operator m_f K m_f + m_c, bc = 0 the unconstrained K. */
int st_apply(st_ctx_t* ctx, const double* rho, const double* x, double* y, int transpose, int bc);

/* Test hook: z = M b, one multigrid V-cycle (the FGMRES preconditioner) of the
 * forward (transpose = 0) or adjoint (1) operator; b, z: this rank's owned planes. */
int st_vcycle(st_ctx_t* ctx, const double* rho, const double* b, double* z, int transpose);

/* Source vector f and the eliminated right-hand side b. */
int st_rhs(st_ctx_t* ctx, const double* rho, double* f, double* b);

/* Multigrid test hooks on level l (0 = finest): y = A_l x (masked, Galerkin operator). */
int st_level_apply(st_ctx_t* ctx, const double* rho, int level, const double* x, double* y,
                   int transpose);

/* Multigrid test hook: the transfer between level l and level l + 1 (linear
 * interpolation P along the coarsened directions, restriction P^T). restrict_ = 1: out (level l + 1
 * nodes) = P^T in (level l nodes), zero at the constrained coarse nodes; restrict_ = 0: out (level l
 * nodes) = P in (level l + 1 nodes), zero at the constrained fine nodes. Vectors in the dense node
 * order of their level (host or device). Single-rank contexts; ST_E_INVALID_ARG for the coarsest level. */
int st_level_transfer(st_ctx_t* ctx, const double* rho, int level, const double* in, double* out,
                      int restrict_);

/* Benchmark hook: enqueue `reps` back-to-back launches of the level-l operator kernel in
 * mode (0 apply, 1 residual y = b - A x, 2 damped-Jacobi sweep, 3 first sweep from zero)
 * on the context's internal work vectors and return WITHOUT synchronising (the caller
 * brackets them with events on the context stream). rho: device pointer. Level 0 rebuilds its
 * per-design tables (the k~ table of a (2+1)D space-time design) only when rho is a different
 * pointer from the previous binding, so the launches are the only work enqueued when the same
 * unchanged rho is passed again (the caller must not modify rho in place between such calls). */
int st_bench_op(st_ctx_t* ctx, const double* rho, int level, int mode, int transpose, int reps);

/* ---- Config-5 design loop (driver level: BASELINE config 5, R-13; NOT the paper's
 * method, which uses a PDE filter, projection and MMA) ---------------------- */
/* Density filter with hat weights max(0, radius - |index distance|) over the element grid
 * (x1, x2[, x3], t); a time-constant design is filtered in space. transpose = 0: out = F in,
 * in = this rank's owned element layers, out = the layers st_solve takes (owned + the next slab's
 * first layer, filtered); transpose = 1 (chain rule): out = F^T in on the owned layers. */
int st_filter(st_ctx_t* ctx, const double* in, double* out, int transpose, double radius);
/* Optimality-criteria update rho_new = clip(rho sqrt(max(0, -dJ) / Lambda), [max(rho_min, rho - move),
 * min(1, rho + move)]) with Lambda by bisection so that the mean over all elements (all ranks) is
 * volfrac. rho, dJ, rho_new: owned element layers. Lambda is written to *lambda_out if non-null. */
int st_oc_update(st_ctx_t* ctx, const double* rho, const double* dJ, double volfrac, double move, double rho_min,
                 double* rho_new, double* lambda_out);
/* ---- The paper's design regularisation --------------------
 * PDE filter (K_f + M_f) g~ = T_f g on the space-time Q1 mesh with natural boundaries and
 * d = diag(rx^2/12, ..., rt^2/12) in rescaled coordinates (the paper: rx = 2.4 dx, rt = 2.4 dt), the
 * element value g~_e = mean of its nodal values (R-25), and the Heaviside projection
 * g_bar = (tanh(beta eta) + tanh(beta (g~_e - eta))) / (tanh(beta eta) + tanh(beta (1 - eta)))
 * (beta = 32, eta = 0.5 in the paper). gamma, gamma_e, gamma_bar: [nt][n]..[n] element fields of a
 * space-time design (one GPU). gamma_e may be NULL. The filter system is solved by Jacobi-preconditioned
 * CG to 1e-12 (st_get_stats iterations). */
int st_pde_filter(st_ctx_t* ctx, const double* gamma, double rx, double rt, double beta, double eta,
                  double* gamma_e, double* gamma_bar);
/* Chain rule: dphi/dgamma = T_f^T (K_f + M_f)^-1 A^T (dg_bar/dg~ .* dphi/dg_bar), from the
 * filtered element field gamma_e of st_pde_filter. */
int st_pde_filter_grad(st_ctx_t* ctx, const double* gamma_e, const double* dphi_dgbar, double rx, double rt,
                       double beta, double eta, double* dphi_dgamma);
/* The paper's objective: phi = (sum_e Tavg_e^P)^(1/P) over all elements (all ranks),
 * Tavg_e the mean of the element's nodal temperatures (P = 20 in the paper), and, if dphidT is
 * non-null, its gradient on this rank's owned planes — the adjoint RHS. */
int st_pnorm(st_ctx_t* ctx, const double* T, double P, double* phi, double* dphidT);
/* out = x . y over the owned nodes of all ranks (e.g. the compliance f^T T). */
int st_dot(st_ctx_t* ctx, const double* x, const double* y, double* out);

/* ---- GPU time-stepping baseline (the comparison method of PAPER.md:620, 704-712) ----
 * First-order backward difference (M_C / dt + K_k) T^{m+1} = (M_C / dt) T^m + F(t_{m+1}), dt = 1 / nsteps
 * (rescaled), T^0 = T0 (0 on the sink / walls), on the context's spatial mesh with its materials, source
 * (spatially uniform kinds UNIFORM / SIN / EX1) and spatial Dirichlet data; each step solved to the
 * context's rtol by CG preconditioned with a spatial geometric-multigrid V-cycle (full spatial
 * coarsening, Galerkin, damped Jacobi 2 + 2, dense coarsest), one CUDA graph launch per CG iteration.
 * rho: the time-constant design (n^sdim, ST_TIME_CONSTANT contexts, one GPU). T: (nsteps + 1) planes
 * of (n+1)^sdim nodes in the caller layout (nsteps = nt gives the space-time vector layout), device or
 * host. Errors: ST_E_UNSUPPORTED (space-time design, slabs, EX2 source), ST_E_INVALID_ARG. */
typedef struct {
  int32_t steps;
  int32_t max_step_iterations;   /* most CG iterations of one step                               */
  int64_t cg_iterations;         /* total over the steps                                          */
  double ms;                     /* device time of setup + all steps                             */
  int64_t launches;              /* kernels launched (graph nodes counted)                       */
} st_ts_stats_t;
int st_timestep(st_ctx_t* ctx, const double* rho, int32_t nsteps, double* T, st_ts_stats_t* stats);

int st_get_stats(const st_ctx_t* ctx, st_stats_t* s);
int st_local_layout(const st_ctx_t* ctx, st_layout_t* layout);

/* Host-only planning (no device call): the Algorithm-1 hierarchy and this rank's slab of every
 * level for a given rank / size, exactly as st_setup would build them. */
typedef struct {
  int32_t n_levels, n_dist_levels;
  int64_t n[32], nt[32];            /* global elements per level                              */
  int32_t kind[32];                 /* 0 fine, 1 space, 2 time                                */
  int32_t dist[32];                 /* 1: time slab, 0: replicated on every rank              */
  int64_t layer0[32], n_layers[32]; /* owned element layers of a slab level (replicated: all) */
  int64_t local_layers[32];         /* layers held locally (owned + ghost layer)              */
  int64_t plane0, n_planes;         /* owned fine node planes (the caller's vector layout)    */
} st_plan_t;
int st_plan(const st_grid_t* grid, const st_materials_t* mats, const st_bcs_t* bcs, const st_options_t* opts,
            int32_t rank, int32_t size, st_plan_t* plan);
/* sizeof of the ABI structs (binding self-check): grid, materials, bcs, source, options, dist,
 * stats, hierarchy, layout, plan, ts_stats */
int st_struct_sizes(int64_t out[11]);
/* NCCL helpers (libnccl.so.2 is opened at run time): a unique id on one rank, broadcast by
 * the caller, then one communicator per rank. Return ST_OK or ST_E_NCCL. */
int st_nccl_unique_id(char id[ST_NCCL_ID_BYTES]);
int st_nccl_comm_init(const char id[ST_NCCL_ID_BYTES], int32_t rank, int32_t size, void** comm);
int st_nccl_comm_destroy(void* comm);
/* Checks a communicator against (rank, size) (ncclCommCount / ncclCommUserRank; *nranks receives the
 * count) and runs every NCCL call the slab path uses on it — ncclAllReduce, ncclAllGather and grouped
 * ncclSend / ncclRecv with the ring neighbours (the rank itself when size = 1) — comparing the results.
 * ST_OK or ST_E_NCCL (text in st_last_error). st_setup with ST_COMM_NCCL performs the count check and
 * logs one line on rank 0. */
int st_nccl_selftest(void* comm, int32_t rank, int32_t size, int32_t* nranks);
int st_get_hierarchy(const st_ctx_t* ctx, st_hierarchy_t* h);
int64_t st_num_nodes(const st_ctx_t* ctx);
int64_t st_num_design(const st_ctx_t* ctx);
/* Number of kernels this library launched since setup (bench evidence). */
int64_t st_kernel_launches(const st_ctx_t* ctx);
const char* st_strerror(int code);
const char* st_last_error(void);
int st_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ST_H_ */
