// api.cu — the C ABI of libst (include/st.h): context, Algorithm-1 hierarchy, rho-dependent
// Galerkin setup, V-cycle, FGMRES, adjoint, sensitivities. Host orchestration in C++;
// every arithmetic step of the path runs in the CUDA kernels of ops/transfer/krylov/misc.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "st.h"
#include "comm.h"
#include "common.cuh"
#include "kernels.h"

using namespace st;

// csrc/pdefilter.cu
int st_run_pde_filter(int sd, int n, int nt, double rx, double rt, double beta, double eta, const double* gamma,
                      double* ge, double* gb, double* const* vec, double* dd, double* hh, RedWs ws, cudaStream_t s);
int st_run_pde_filter_grad(int sd, int n, int nt, double rx, double rt, double beta, double eta, const double* ge,
                           const double* dphi, double* out, double* const* vec, double* dd, double* hh, RedWs ws,
                           cudaStream_t s);
// csrc/timestep.cu
long long st_run_timestepping(const Geom& g0, const MatsDev& md, const st_source_t& src, double tau, double T0,
                              const double* rho, int nsteps, double rtol, int maxit, int coarse_max_nodes,
                              const Geom& gdense, double* Tout, cudaStream_t s, double* ms_out, long long* launches,
                              int* max_its);

namespace {
thread_local std::string g_last_error;

struct StErr {
  int code;
  std::string msg;
};

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      throw StErr{e_ == cudaErrorMemoryAllocation ? ST_E_OOM : ST_E_CUDA,               \
                  std::string(#call) + ": " + cudaGetErrorString(e_)};                  \
  } while (0)

struct Level {
  Geom g{};              // local geometry: a time slab (dist) or the whole level (replicated)
  int kind = KIND_FINE;
  OpDesc op{};
  double* st = nullptr;  // owned stencil storage (null if shared / RHO)
  bool st_owned = false;
  long long st_elems = 0;
  double *x = nullptr, *b = nullptr, *r = nullptr, *t = nullptr;
  bool dense = false;
  double *A = nullptr, *Ainv = nullptr;
  int* info = nullptr;
  int nf = 0;                                  // dense: free nodes (not pad, not constrained)
  int *fidx = nullptr, *fpos = nullptr;        // dense: free stored indices [nf]; stored -> free position [N]
  // time slabs
  int ntg = 0;           // global element layers of the level
  bool dist = false;     // distributed in time slabs (else replicated on every rank)
  int nloc = 0, a = 0;   // dist: owned element layers [a, a + nloc) = node planes (a, a + nloc]
  bool gather_in = false;  // first replicated level below a distributed one
  Geom gs{};             // gather_in: this level in slab form (restriction / stencils before gather)
  double omega = 0.0;    // damped-Jacobi weight of this level (per design)
  double lam_max = 0.0;  // power-iteration estimate of |lambda|_max(D^-1 A) of this level
  double* bpart = nullptr;
  double* stpart = nullptr;
  long long stpart_elems = 0;
  // full space-time coarsening of a time-varying level: the parent's stencils coarsened in space
  // only (mid_ns stencils per parent layer on this level's spatial grid), then in time
  double* mid = nullptr;
  long long mid_elems = 0;
  int mid_ns = 0;
  // GMRES(k) smoother (ST_SMOOTH_GMRES) / GMRES coarsest solve (cgm): k+1 basis vectors with leading
  // dimension gld
  double* gv = nullptr;
  long long gld = 0;
  bool cgm = false;      // coarsest level solved by GMRES(<= coarse_maxit)-Jacobi (ST_COARSE_GMRES)
};
}  // namespace

struct st_ctx {
  st_grid_t grid{};
  st_materials_t mats{};
  st_bcs_t bcs{};
  st_source_t src{};
  st_options_t opt{};
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int sd = 2;
  bool tc = true;
  MatsDev md{};
  std::vector<Level> lv;
  long long N = 0, Nd = 0, ndesign = 0, ld = 0;   // N: internal (padded) storage, Nd: nodes
  long long guard = 0;                              // zeroed front guard of internal vectors
  std::vector<double*> vallocs;                     // guarded allocations (raw bases)
  Geom gd0{};                                      // level-0 geometry in the caller's dense layout
  // level-0 vectors (memory plan): the right-hand side of the current solve, the
  // iterate, and the Krylov pool V[0..m] | Z[0..nz) that doubles as scratch for the test hooks and the
  // V-cycle's level-0 residual (no other full-length vector is allocated)
  double *rhs = nullptr, *xint = nullptr;
  double *V = nullptr, *Z = nullptr;
  int nz = 0;                                       // Z slots: m (FGMRES) or 1 (GMRES: z = M v_j)
  RedWs ws{};
  double* dsmall = nullptr;
  double* hsmall = nullptr;
  double* rho_stage = nullptr;
  double* kt = nullptr;          // padded k~ table of a (2+1)D space-time design (launch_ktilde; tv2d)
  bool kt_design = false;        // kt belongs to the cached design (rho_ck); test hooks may rebuild it
  double* io_stage[4] = {nullptr, nullptr, nullptr, nullptr};
  long long io_n[4] = {0, 0, 0, 0};
  unsigned long long rho_fp[2] = {0ull, 0ull};  // design fingerprint of the cached operators
  bool have_ops = false;
  st_stats_t stats{};
  long long launches = 0;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  // st_design_step with host vectors: the side stream that copies results back while the next phase
  // computes, and its ordering events (created on first use)
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_rdy[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr};
  // time slabs: rank, owned fine planes [o0, o0 + nown) of the local vector (o0 = 0 on rank 0,
  // else 1: local plane 0 is the ghost copy of the previous rank's last plane)
  Comm comm;
  int o0 = 0, nown = 0;
  long long voff = 0, Nown = 0;   // owned range of an internal fine vector (offset, count)
  int n_dist = 0;                 // distributed levels
  // CUDA graphs of the small-level part of the V-cycle (levels >= gl0, replicated and fixed
  // buffers): one per direction, captured after one eager run, valid for the context lifetime
  int gl0 = -1;
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};
  // DGKS: re-orthogonalise when ||w'||^2 < eta^2 ||w||^2 (options dgks_eta, default 0.1). With the
  // V-cycle preconditioner ||w'|| / ||w|| stays above 0.1, and the measured iteration counts and true
  // residuals equal those of eta^2 = 0.5 (which re-orthogonalised every step) on configs 2-4
  // (profiles/r01/dgks_threshold.log); the pass remains a safety net for severe cancellation.
  double dgks_eta2 = 0.01;
  double* gsm = nullptr;  // GMRES smoother: device Hessenberg / Givens (1024 doubles) + dots (1024)
  double* cgs = nullptr;  // GMRES coarsest solve: device state gm_layout(coarse_maxit) + dots
  long long coarse_its = 0;
  // config-5 design update buffers (st_filter / st_oc_update), allocated on first use
  double *fbuf = nullptr, *fw = nullptr;
  long long gkernels[2] = {0, 0};
  int geager[2] = {0, 0};
};

namespace {

void L(st_ctx* c, long long n = 1) { c->launches += n; }

void check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw StErr{ST_E_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e)};
}

template <class T> void dalloc(T** p, size_t count) {
  CK(cudaMalloc((void**)p, std::max<size_t>(count, 1) * sizeof(T)));
}
// zero-initialised (pad entries of internal vectors must stay zero)
void dzalloc(double** p, size_t count) {
  dalloc(p, count);
  CK(cudaMemset(*p, 0, std::max<size_t>(count, 1) * sizeof(double)));
}

// pad = true: internal layout with an even x1 row pitch (16-byte aligned rows and planes).
// nt: local element layers; ntg (> 0): global layers of the level (dt = 1/ntg), pg0: global
// index of local plane 0.
// row-pitch alignment (doubles) of the padded internal layout while a context is being set up
// (st_options_t pitch_align; st_setup / st_plan set it around build_hierarchy and assign_slabs)
thread_local int t_pitch_align = 2;

Geom make_geom(int sd, int n, int nt, int plo, int phi, bool pad = true, int ntg = 0, int pg0 = 0) {
  Geom g{};
  g.sd = sd;
  g.n = n;
  g.nn = n + 1;
  g.nt = nt;
  g.pr = pad ? (g.nn + t_pitch_align - 1) / t_pitch_align * t_pitch_align : g.nn;
  g.P = g.pr;
  for (int d = 1; d < sd; ++d) g.P *= g.nn;
  g.N = g.P * (nt + 1);
  g.plo = plo;
  g.phi = phi;
  g.dx = 1.0 / n;
  g.dt = 1.0 / (ntg > 0 ? ntg : nt);
  g.pg0 = pg0;
  return g;
}

int nc_of(int sd) { return sd == 2 ? 5 : 14; }
long long nodes_of(const Geom& g) {
  long long v = g.nt + 1;
  for (int d = 0; d < g.sd; ++d) v *= g.nn;
  return v;
}
Geom dense_of(const Geom& g) {
  Geom d = make_geom(g.sd, g.n, g.nt, g.plo, g.phi, false, (int)std::lround(1.0 / g.dt), g.pg0);
  d.walls = g.walls;
  return d;
}

// E' = W0^T E W0 + W1^T E W1 (linear-in-time prolongation, two fine layers per coarse layer)
void time_coarsen_factor(const double E[2][2], double out[2][2]) {
  const double W[2][2][2] = {{{1.0, 0.0}, {0.5, 0.5}}, {{0.5, 0.5}, {0.0, 1.0}}};
  for (int A = 0; A < 2; ++A)
    for (int B = 0; B < 2; ++B) {
      double v = 0.0;
      for (int f = 0; f < 2; ++f)
        for (int a = 0; a < 2; ++a)
          for (int b = 0; b < 2; ++b) v += W[f][a][A] * W[f][b][B] * E[a][b];
      out[A][B] = v;
    }
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a{};
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

double* stage(st_ctx* c, int slot, long long n) {
  if (c->io_n[slot] < n) {
    if (c->io_stage[slot]) cudaFree(c->io_stage[slot]);
    dalloc(&c->io_stage[slot], (size_t)n);
    c->io_n[slot] = n;
  }
  return c->io_stage[slot];
}

const double* in_ptr(st_ctx* c, const double* p, long long n, int slot) {
  if (!p) throw StErr{ST_E_INVALID_ARG, "null pointer"};
  if (is_device_ptr(p)) return p;
  double* d = stage(c, slot, n);
  CK(cudaMemcpyAsync(d, p, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  return d;
}

// ---------------------------------------------------------------------------------------
// Algorithm 1
void build_hierarchy(st_ctx* c) {
  const st_materials_t& m = c->mats;
  const double scale = c->grid.tau / (c->grid.L * c->grid.L);
  const double kc = m.k_con * scale, ki = m.k_ins * scale;
  const double D = std::sqrt(kc * ki / (m.C_con * m.C_ins));
  int n = (int)c->grid.n, nt = (int)c->grid.nt;
  // sink patch on the fine level: nodes j with |j/n - center| <= halfwidth (R-4)
  int plo = 1, phi = 0;
  if (c->bcs.has_patch && !c->bcs.all_walls) {  // all_walls takes precedence (as the oracle's dirichlet)
    plo = n + 1;
    phi = -1;
    for (int j = 0; j <= n; ++j) {
      if (std::fabs((double)j / n - c->bcs.center) <= c->bcs.halfwidth * (1.0 + 1e-12)) {
        plo = std::min(plo, j);
        phi = std::max(phi, j);
      }
    }
  }
  c->lv.clear();
  Level L0;
  L0.g = make_geom(c->sd, n, nt, plo, phi);
  L0.kind = KIND_FINE;
  c->lv.push_back(L0);
  const int maxl = c->opt.max_levels > 0 ? c->opt.max_levels : 64;
  while ((int)c->lv.size() < maxl) {
    const Geom& g = c->lv.back().g;
    if (nodes_of(g) <= c->opt.coarse_max_nodes) break;
    double lam = D * g.dt / (g.dx * g.dx);
    int kind;
    bool ok;
    if (c->opt.full_coarsening) {
      kind = KIND_FULL;
      ok = (g.n % 2 == 0) && (g.nt % 2 == 0) && g.n >= 2 && g.nt >= 2;
    } else if (lam < c->opt.lambda_crit) {
      kind = KIND_TIME;
      ok = (g.nt % 2 == 0) && g.nt >= 2;
    } else {
      kind = KIND_SPACE;
      ok = (g.n % 2 == 0) && g.n >= 2;
    }
    if (!ok) break;
    int n2 = g.n, nt2 = g.nt, plo2 = g.plo, phi2 = g.phi;
    if (kind == KIND_SPACE || kind == KIND_FULL) {
      n2 /= 2;
      plo2 = (g.plo + 1) / 2;  // coarse J with 2J in [plo, phi] (injection)
      phi2 = g.phi >= 0 ? g.phi / 2 : -1;
    }
    if (kind == KIND_TIME || kind == KIND_FULL) nt2 /= 2;
    Level Ln;
    Ln.g = make_geom(c->sd, n2, nt2, plo2, phi2);
    Ln.kind = kind;
    c->lv.push_back(Ln);
  }
  // the dense coarsest inverse is one CTA's O(n^3) Gauss-Jordan on the free nodes (misc.cu): <= 4096
  // stored nodes (n^3 element updates at ~1.5e9 / s in one CTA: ~10 ms at config 4's 248 free nodes, a few
  // seconds per design near the limit); larger coarsest levels need the iterative coarsest solve
  // (ST_COARSE_GMRES)
  if (c->opt.coarse_solver == ST_COARSE_DENSE && c->lv.back().g.N > 4096)
    throw StErr{ST_E_DIVISIBILITY, "coarsest level too large for the dense solve (" +
                                       std::to_string(c->lv.back().g.N) +
                                       " stored nodes > 4096): grid not divisible enough; use coarse_solver = "
                                       "ST_COARSE_GMRES (the paper's GMRES coarsest solve)"};
  for (auto& Lv : c->lv) {
    Lv.ntg = Lv.g.nt;
    Lv.g.walls = c->bcs.all_walls ? 1 : 0;  // coarse walls = injection of the fine walls (R-23)
  }
}

// Time slabs: the leading levels whose time extent splits into G equal
// slabs (and that still have >= agg_nodes nodes per rank) are distributed; the next level is
// gathered onto every rank (it must split too: it is produced in slab form, then gathered) and
// every coarser level, including the dense coarsest one, is replicated.
void assign_slabs(st_ctx* c) {
  const int G = c->comm.size, r = c->comm.rank;
  const int nl = (int)c->lv.size();
  int nd = 0;
  if (G > 1) {
    auto splits = [&](int l) { return c->lv[l].ntg % G == 0 && c->lv[l].ntg / G >= 1; };
    auto big = [&](int l) { return nodes_of(c->lv[l].g) / G >= c->opt.agg_nodes; };
    nd = 1;  // the fine level is always distributed (validated in st_setup)
    while (nd < nl - 1 && splits(nd) && big(nd)) ++nd;
    // the first replicated level must split too (slab-form restriction before the gather)
    while (nd > 1 && nd < nl && !splits(nd)) --nd;
    if (nd < nl && !splits(nd)) throw StErr{ST_E_DIVISIBILITY, "time slabs: level 1 does not split over the ranks"};
  }
  c->n_dist = nd;
  for (int l = 0; l < nl; ++l) {
    Level& Lv = c->lv[l];
    const Geom g = Lv.g;  // global geometry
    if (l < nd) {
      Lv.dist = true;
      Lv.nloc = Lv.ntg / G;
      Lv.a = r * Lv.nloc;
      const int ntl = Lv.nloc + (r < G - 1 ? 1 : 0);  // + ghost layer (except the last rank)
      Lv.g = make_geom(g.sd, g.n, ntl, g.plo, g.phi, true, Lv.ntg, Lv.a);
      Lv.g.walls = g.walls;
    } else if (l == nd && nd > 0) {
      Lv.gather_in = true;
      const int nlc = Lv.ntg / G, ac = r * nlc;
      Lv.gs = make_geom(g.sd, g.n, nlc + (r < G - 1 ? 1 : 0), g.plo, g.phi, true, Lv.ntg, ac);
      Lv.gs.walls = g.walls;
    }
  }
}

void setup_forms(st_ctx* c) {
  const int NC = nc_of(c->sd);
  for (size_t l = 0; l < c->lv.size(); ++l) {
    Level& Lv = c->lv[l];
    OpDesc& op = Lv.op;
    op.g = Lv.g;
    op.m = c->md;
    op.family = c->opt.kernel_family;
    op.chunk = c->opt.chunk_planes;
    op.max_ctas = c->opt.max_ctas;
    if (l == 0) {
      op.form = FORM_RHO;
      op.nl = c->tc ? 1 : Lv.g.nt;
      op.tvl = c->tc ? 0 : 1;
      op.rho_tc = c->tc ? 1 : 0;
      op.U[0][0] = 0.0; op.U[0][1] = 0.0; op.U[1][0] = -1.0; op.U[1][1] = 1.0;
      double s = Lv.g.dt / 6.0;
      op.Tm[0][0] = 2 * s; op.Tm[0][1] = s; op.Tm[1][0] = s; op.Tm[1][1] = 2 * s;
      continue;
    }
    const Level& Pv = c->lv[l - 1];
    const OpDesc& po = Pv.op;
    // uniform capacity: every time-constant Galerkin level keeps C_ins x the Q1 mass of its own
    // grid (nested spaces: P^T M_h P = M_H), applied separably by the lean kernel
    op.msep = 0;
    op.msc = 0.0;
    // stored layers: 1 (time-constant design) or every local layer of the level
    const bool tv = po.tvl != 0;  // explicit: a slab of a time-varying level may hold one layer
    op.tvl = tv ? 1 : 0;
    int ns = 2;
    if (Lv.kind == KIND_FULL) {
      // P = P_t (x) P_s: Galerkin P^T K P = time coarsening of the space coarsening (the capacity
      // re-stabilised under the time step as on a KIND_TIME level, R-22)
      if (Lv.dist || Pv.dist) throw StErr{ST_E_UNSUPPORTED, "full space-time coarsening on time slabs"};
      op.U[0][0] = 0.0; op.U[0][1] = 0.0; op.U[1][0] = -1.0; op.U[1][1] = 1.0;
      Lv.st_owned = true;
      if (!tv) {
        op.form = FORM_MK;
        op.nl = 1;
        time_coarsen_factor(po.Tm, op.Tm);
        ns = 2;
      } else {
        op.form = FORM_B4;
        op.nl = Lv.g.nt;
        ns = 5;
        Lv.mid_ns = (po.form == FORM_B4) ? 5 : 2;
        Lv.mid_elems = (long long)Pv.g.nt * Lv.mid_ns * NC * Lv.g.P;
      }
    } else if (Lv.kind == KIND_SPACE) {
      op.nl = tv ? Lv.g.nt : 1;
      memcpy(op.U, po.U, sizeof(op.U));
      if (po.form == FORM_RHO || po.form == FORM_MK) {
        op.form = FORM_MK;
        memcpy(op.Tm, po.Tm, sizeof(op.Tm));
        ns = 2;
      } else {
        op.form = FORM_B4;
        ns = 5;
      }
      Lv.st_owned = true;
    } else {  // KIND_TIME: Galerkin conduction, re-stabilised (upwind) capacity in time
      op.U[0][0] = 0.0; op.U[0][1] = 0.0; op.U[1][0] = -1.0; op.U[1][1] = 1.0;
      if (!tv && po.form == FORM_RHO && c->sd == 3) {
        // (3+1)D, time-constant design: the time-coarsened level is the fine discretisation on the
        // doubled time step (nested spaces: the Galerkin time factor of the conduction term equals
        // the coarse T_m; the capacity is re-stabilised, R-22), so it stays matrix-free from rho and
        // runs the element-layer kernel (tc3r) instead of 2 x 27 stored weights per node (tc3d)
        op.form = FORM_RHO;
        op.rho_tc = 1;
        op.nl = 1;
        time_coarsen_factor(po.Tm, op.Tm);
        Lv.st_owned = false;
        ns = 2;
      } else if (!tv) {
        op.form = FORM_MK;
        op.nl = 1;
        time_coarsen_factor(po.Tm, op.Tm);
        Lv.st_owned = (po.form == FORM_RHO);  // else: the same spatial stencils as the finer level
        ns = 2;
      } else {
        op.form = FORM_B4;
        op.nl = Lv.g.nt;
        Lv.st_owned = true;
        ns = 5;
      }
    }
    Lv.st_elems = Lv.st_owned ? (long long)op.nl * ns * NC * Lv.g.P : 0;
    if (Lv.gather_in && tv) Lv.stpart_elems = (long long)Lv.gs.nt * ns * NC * Lv.gs.P;
    if (op.form == FORM_MK && c->md.dC == 0.0) {  // time-constant or per-layer (M is C_ins x Q1 mass)
      op.msep = 1;
      op.msc = c->md.Cins * Lv.g.dx * Lv.g.dx / 36.0;
    }
  }
}

// internal nodal vector: zeroed, with a zeroed front guard of c->guard entries so that the
// TMA x-tile maps (based pr + 2 entries before the data)
// only ever see non-negative box coordinates and finite data
double* vec_alloc(st_ctx* c, long long count) {
  double* base = nullptr;
  dzalloc(&base, (size_t)(count + 2 * c->guard));
  c->vallocs.push_back(base);
  return base + c->guard;
}

// slot k of the level-0 pool V[0..m] | Z[0..nz): scratch vectors of the hooks (outside a solve)
double* pool(st_ctx* c, int k) {
  const int m = c->opt.restart;
  if (k < 0 || k > m + c->nz) throw StErr{ST_E_INVALID_ARG, "internal: pool slot"};
  return k <= m ? c->V + (long long)k * c->ld : c->Z + (long long)(k - m - 1) * c->ld;
}

void allocate(st_ctx* c) {
  const long long N = c->N;
  const int m = c->opt.restart;
  // zeroed front guard: the TMA x maps are based one row (2D) / one slice + one row (3D) + 2
  // entries before the data
  {
    const Geom& g0 = c->lv[0].g;
    const long long need = (c->sd == 3 ? (long long)g0.pr * g0.nn : 0) + g0.pr + 2;
    c->guard = (need + 31) / 32 * 32;
  }
  c->ld = (N + c->guard + 31) / 32 * 32;   // vector j's guard = tail of slot j-1 (never written)
  c->rhs = vec_alloc(c, N);
  c->xint = vec_alloc(c, N);
  c->nz = c->opt.krylov == ST_KRYLOV_GMRES ? 1 : m;
  c->V = vec_alloc(c, (m + 1) * c->ld);
  c->Z = vec_alloc(c, c->nz * c->ld);
  dalloc(&c->ws.partial, (size_t)kRedBlocks * kMaxDots);
  dalloc(&c->ws.counter, 1);
  CK(cudaMemsetAsync(c->ws.counter, 0, sizeof(unsigned), c->stream));
  dalloc(&c->dsmall, 512);
  {
    const double one = 1.0;  // dsmall[510]: unit coefficient of x += M u (GMRES)
    CK(cudaMemcpy(c->dsmall + 510, &one, sizeof(double), cudaMemcpyHostToDevice));
  }
  if (c->opt.smoother == ST_SMOOTH_GMRES) {  // the paper's smoother: basis per level
    const int k = std::max(c->opt.nu_pre, c->opt.nu_post);
    dzalloc(&c->gsm, 2048);
    for (auto& Lv : c->lv) {
      if (&Lv == &c->lv.back()) break;  // the coarsest level has its own solve
      Lv.gld = (Lv.g.N + 31) / 32 * 32;
      dzalloc(&Lv.gv, (long long)(k + 1) * Lv.gld);  // zero pads: the dots run over the padded length
    }
  }
  CK(cudaMallocHost((void**)&c->hsmall, 512 * sizeof(double)));
  if ((long long)c->comm.size * (long long)c->lv.size() > 140) throw StErr{ST_E_INVALID_ARG, "too many ranks x levels"};
  for (size_t l = 0; l < c->lv.size(); ++l) {
    Level& Lv = c->lv[l];
    const long long n = Lv.g.N;
    if (l == 0) {
      Lv.t = vec_alloc(c, n);  // Jacobi ping-pong; the residual goes to a Krylov-pool slot
    } else {
      Lv.x = vec_alloc(c, n);
      Lv.b = vec_alloc(c, n);
      Lv.r = vec_alloc(c, n);
      Lv.t = vec_alloc(c, n);
      if (Lv.st_owned) {
        dalloc(&Lv.st, Lv.st_elems);
        Lv.op.st = Lv.st;
        if (Lv.mid_elems > 0) dalloc(&Lv.mid, Lv.mid_elems);
      } else {
        Lv.op.st = c->lv[l - 1].op.st;  // resolved again after build (shared)
      }
      if (Lv.gather_in) {
        Lv.bpart = vec_alloc(c, Lv.gs.N);
        if (Lv.stpart_elems > 0) dalloc(&Lv.stpart, Lv.stpart_elems);
      }
    }
  }
  Level& Lc = c->lv.back();
  if (c->opt.coarse_solver == ST_COARSE_GMRES) {  // the paper's GMRES coarsest solve
    const int k = c->opt.coarse_maxit;
    Lc.cgm = true;
    Lc.gld = (Lc.g.N + 31) / 32 * 32;
    dzalloc(&Lc.gv, (long long)(k + 1) * Lc.gld);
    dzalloc(&c->cgs, (size_t)gm_y_offset(k) + k + 32 + kMaxBasis + 64);
  } else {
    Lc.dense = true;
    // the free nodes of the coarsest level (host replica of pdecode / is_cons; the level is replicated:
    // plane 0 is the initial-condition plane): the dense inverse excludes pad entries and the identity
    // rows of constrained nodes (config 4: 248 of 600 stored entries, configs 2 / 3: 96 of 200)
    const Geom& g = Lc.g;
    std::vector<int> fidx, fpos((size_t)g.N, -1);
    for (long long e = 0; e < g.N; ++e) {
      const int p = (int)(e / g.P);
      const long long pn = e % g.P;
      const int c0 = (int)(pn % g.pr);
      const long long t = pn / g.pr;
      const int c1 = (int)(t % g.nn), c2 = c->sd == 3 ? (int)(t / g.nn) : 0;
      if (c0 >= g.nn || p + g.pg0 == 0) continue;
      bool patch;
      if (g.walls) {
        patch = c0 == 0 || c0 == g.n || c1 == 0 || c1 == g.n || (c->sd == 3 && (c2 == 0 || c2 == g.n));
      } else {
        patch = c0 == 0 && c1 >= g.plo && c1 <= g.phi && (c->sd == 2 || (c2 >= g.plo && c2 <= g.phi));
      }
      if (patch) continue;
      fpos[(size_t)e] = (int)fidx.size();
      fidx.push_back((int)e);
    }
    Lc.nf = (int)fidx.size();
    dalloc(&Lc.A, (size_t)g.N * g.N);
    dalloc(&Lc.Ainv, (size_t)std::max(Lc.nf, 1) * std::max(Lc.nf, 1));
    dalloc(&Lc.info, 1);
    dalloc(&Lc.fidx, std::max<size_t>(fidx.size(), 1));
    dalloc(&Lc.fpos, (size_t)g.N);
    if (!fidx.empty()) CK(cudaMemcpy(Lc.fidx, fidx.data(), fidx.size() * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(Lc.fpos, fpos.data(), fpos.size() * sizeof(int), cudaMemcpyHostToDevice));
  }
  CK(cudaEventCreate(&c->e0));
  CK(cudaEventCreate(&c->e1));
  c->gl0 = -1;
  // every replicated coarse level (level 0 takes the FGMRES vectors: not capturable); measured on
  // config 2: 563.8 MDOF/s vs ~558 with levels < 2^19 nodes only; options graph_max_nodes bounds it
  const long long gmax = c->opt.graph_max_nodes > 0 ? c->opt.graph_max_nodes : (1LL << 62);
  // host decisions inside the cycle (iterative coarsest solve, smoother with an inner rtol): no graph
  const bool host_sync = c->opt.coarse_solver == ST_COARSE_GMRES ||
                         (c->opt.smoother == ST_SMOOTH_GMRES && c->opt.smoother_rtol > 0.0);
  for (size_t l = 1; l + 1 < c->lv.size() && !host_sync; ++l) {
    const Level& Lv = c->lv[l];
    if (!Lv.dist && nodes_of(Lv.g) < gmax) {
      c->gl0 = (int)l;
      break;
    }
  }
}

void op_launch(st_ctx* c, int l, int mode, bool trans, bool mask, const double* x, const double* b, double* y) {
  launch_op(c->lv[l].op, mode, trans, mask, x, b, y, c->lv[l].omega > 0.0 ? c->lv[l].omega : c->opt.omega, c->stream);
  L(c);
}

// ---- time-slab communication -------------------------------------------
template <class F> void comm_call(F&& f) {
  try {
    f();
  } catch (const CommError& e) {
    throw StErr{ST_E_NCCL, e.msg};
  }
}
// refresh the two ghost planes of a vector of distributed level l
void halo(st_ctx* c, int l, double* v) {
  const Level& Lv = c->lv[l];
  if (!Lv.dist || c->comm.size <= 1) return;
  const long long P = Lv.g.P;
  comm_call([&] { comm_halo(c->comm, v + P, v, v + (long long)Lv.nloc * P, v + (long long)(Lv.nloc + 1) * P, P, c->stream); });
}
void allreduce(st_ctx* c, double* d, long long n) {
  if (c->comm.size <= 1) return;
  comm_call([&] { comm_allreduce(c->comm, d, n, c->stream); });
}
// owned planes 1..nlc of a slab-form vector of level Nx -> planes 1..ntg of its replicated copy
void gather_planes(st_ctx* c, const Level& Nx, const double* part, double* full) {
  const int nlc = Nx.ntg / c->comm.size;
  const long long P = Nx.g.P;
  comm_call([&] { comm_allgather(c->comm, part + P, full + P, (long long)nlc * P, c->stream); });
}

// level-0 rho binding; a (2+1)D space-time fine level also gets its k~ table (one pass over the
// design, read by tv2d instead of rho: the same bytes per sweep, no per-sweep rho^p)
// every matrix-free level reads the design itself (level 0; (3+1)D time-constant: also the leading
// time-coarsened levels). Captured V-cycle graphs hold the pointer: a new pointer drops them.
void set_level_rho(st_ctx* c, const double* rho) {
  bool coarse_moved = false;
  for (size_t l = 0; l < c->lv.size(); ++l)
    if (c->lv[l].op.form == FORM_RHO) {
      if (l > 0 && c->lv[l].op.rho != rho) coarse_moved = true;
      c->lv[l].op.rho = rho;
    }
  if (coarse_moved)
    for (int d = 0; d < 2; ++d) {
      if (c->gexec[d]) cudaGraphExecDestroy(c->gexec[d]);
      c->gexec[d] = nullptr;
      c->geager[d] = 0;
    }
}

void set_fine_rho(st_ctx* c, const double* rho) {
  set_level_rho(c, rho);
  if (c->kt) {
    launch_ktilde(rho, c->grid.n, c->lv[0].g.nt, c->lv[0].op.m, c->kt, c->stream);
    L(c);
    c->lv[0].op.kt = c->kt;
  }
}

// a host design is staged through a context buffer allocated on first use (device designs cost nothing)
const double* rho_device(st_ctx* c, const double* rho) {
  if (!rho) throw StErr{ST_E_INVALID_ARG, "null rho"};
  if (is_device_ptr(rho)) return rho;
  if (!c->rho_stage) dalloc(&c->rho_stage, c->ndesign);
  CK(cudaMemcpyAsync(c->rho_stage, rho, c->ndesign * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  return c->rho_stage;
}

// rho -> level-0 operator pointer; returns true if rho changed since the last full setup
bool bind_rho(st_ctx* c, const double* rho_in) {
  const double* rho = rho_device(c, rho_in);
  set_level_rho(c, rho);  // the per-design tables follow in prepare() when rho changed
  // exact change detection: 128 bits of hash over the bit patterns (launch_fingerprint)
  unsigned long long* fp = reinterpret_cast<unsigned long long*>(c->dsmall + 500);
  launch_fingerprint(rho, c->ndesign, fp, c->stream);
  L(c);
  CK(cudaMemcpyAsync(c->hsmall + 500, fp, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  unsigned long long h[2];
  memcpy(h, c->hsmall + 500, sizeof(h));
  int local_changed = !(c->have_ops && h[0] == c->rho_fp[0] && h[1] == c->rho_fp[1]);
  c->rho_fp[0] = h[0];
  c->rho_fp[1] = h[1];
  // one decision on every rank (a rank whose slab changed makes every rank rebuild)
  if (c->comm.size > 1) {
    c->hsmall[500] = local_changed ? 1.0 : 0.0;
    CK(cudaMemcpyAsync(c->dsmall + 500, c->hsmall + 500, sizeof(double), cudaMemcpyHostToDevice, c->stream));
    allreduce(c, c->dsmall + 500, 1);
    CK(cudaMemcpyAsync(c->hsmall + 500, c->dsmall + 500, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    local_changed = c->hsmall[500] > 0.0;
  }
  return local_changed != 0;
}

// Per-level Jacobi weight: the capacity term is an upwind difference in time,
// so on capacity-dominated levels the spectrum of D^-1 A fills a disk through 0 of diameter
// R = |lambda|_max (R = 2 x mass row-sum / diagonal: 4.5 in 2D, 6.75 in 3D) and damped Jacobi is
// stable iff omega R / 2 < 1. R is bounded by the row-wise Gershgorin ratio max_i sum_j |A_ij| /
// |A_ii| (one pass over the level's stencils, every design); omega_l = min(omega_cap, 1.9 / R).
constexpr double kOmegaFactor = 1.9;
void estimate_omegas(st_ctx* c) {
  unsigned long long* d = reinterpret_cast<unsigned long long*>(c->dsmall + 320);
  const int nl = (int)c->lv.size();
  CK(cudaMemsetAsync(d, 0, nl * sizeof(double), c->stream));
  for (int l = 0; l < nl; ++l) {
    const Level& Lv = c->lv[l];
    if (Lv.dense) continue;
    // time-constant: interior row type (plane 1) and the last plane; else every local row
    // (ghost planes of a slab: row 0 is skipped by pa = 1; the top ghost row is not a real row)
    const int pa = 1, pb = Lv.g.nt - ((Lv.dist && c->comm.rank < c->comm.size - 1) ? 1 : 0);
    if (!Lv.op.tvl && !(Lv.op.form == FORM_RHO && !Lv.op.rho_tc)) {
      launch_gersh(Lv.op, 1, std::min(2, Lv.g.nt), d + l, c->stream);
      launch_gersh(Lv.op, Lv.g.nt, Lv.g.nt, d + l, c->stream);
      L(c, 2);
    } else {
      launch_gersh(Lv.op, pa, pb, d + l, c->stream);
      L(c);
    }
  }
  check_launch();
  // max over ranks: gather every rank's values (the host transport has sums and gathers only)
  const int G = c->comm.size;
  double* gat = c->dsmall + 352;  // G * nl doubles (G * nl <= 160)
  if (G > 1) comm_call([&] { comm_allgather(c->comm, c->dsmall + 320, gat, nl, c->stream); });
  CK(cudaMemcpyAsync(c->hsmall + 352, G > 1 ? gat : c->dsmall + 320, (size_t)G * nl * sizeof(double),
                     cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  for (int l = 0; l < nl; ++l) {
    Level& Lv = c->lv[l];
    double R = 0.0;
    for (int r = 0; r < G; ++r) R = std::max(R, c->hsmall[352 + r * nl + l]);
    Lv.lam_max = R;
    // 1.9: stable (omega R / 2 < 1) with a 5 % margin; measured 1.5 / 1.8 / 1.9 / 1.95 on configs 2-5
    // (profiles/r01/omega_factor.log; options omega_factor)
    const double fac = c->opt.omega_factor > 0.0 ? c->opt.omega_factor : kOmegaFactor;
    Lv.omega = (R > 0.0 && std::isfinite(R)) ? std::min(c->opt.omega, fac / R) : c->opt.omega;
  }
}

// rho-dependent setup: Galerkin coarse operators, dense coarsest inverse,
// eliminated right-hand side b.
void build_ops(st_ctx* c) {
  CK(cudaEventRecord(c->e0, c->stream));
  // the per-level Jacobi weights are re-estimated per design: drop captured V-cycle graphs
  for (int d = 0; d < 2; ++d) {
    if (c->gexec[d]) cudaGraphExecDestroy(c->gexec[d]);
    c->gexec[d] = nullptr;
    c->geager[d] = 0;
  }
  const int NC = nc_of(c->sd);
  for (size_t l = 1; l < c->lv.size(); ++l) {
    Level& Lv = c->lv[l];
    const Level& Pv = c->lv[l - 1];
    const int ns = Lv.op.form == FORM_B4 ? 5 : 2;
    const bool tv = Lv.op.tvl != 0;
    const long long layer = (long long)ns * NC * Lv.g.P;  // stencil doubles per layer
    if (Lv.kind == KIND_SPACE) {
      if (Lv.gather_in && tv) {  // slab form, then gather the owned layers
        launch_rap_space(Pv.op, Lv.gs, Lv.gs.nt, ns, Lv.stpart, c->stream);
        L(c);
        comm_call([&] { comm_allgather(c->comm, Lv.stpart, Lv.st, (long long)(Lv.ntg / c->comm.size) * layer, c->stream); });
      } else {
        launch_rap_space(Pv.op, Lv.g, Lv.op.nl, ns, Lv.st, c->stream);
        L(c);
      }
    } else if (Lv.kind == KIND_FULL) {
      if (!tv) {  // spatial stencils coarsened in space; the time factor is in op.Tm
        launch_rap_space(Pv.op, Lv.g, 1, 2, Lv.st, c->stream);
        L(c);
      } else {  // space coarsening of every parent layer into mid, then time coarsening of mid
        OpDesc mop = Pv.op;
        t_pitch_align = c->opt.pitch_align;
        mop.g = make_geom(c->sd, Lv.g.n, Pv.g.nt, Lv.g.plo, Lv.g.phi);
        t_pitch_align = 2;
        mop.g.walls = Lv.g.walls;
        mop.form = Lv.mid_ns == 5 ? FORM_B4 : FORM_MK;
        mop.nl = Pv.g.nt;
        mop.tvl = 1;
        mop.rho = nullptr;
        mop.kt = nullptr;
        mop.msep = 0;
        mop.st = Lv.mid;
        launch_rap_space(Pv.op, mop.g, Pv.g.nt, Lv.mid_ns, Lv.mid, c->stream);
        launch_rap_time(mop, Lv.g.nt, Lv.st, c->stream);
        L(c, 2);
      }
    } else if (Lv.kind == KIND_TIME) {
      if (!tv) {
        if (Lv.op.form == FORM_RHO) {
          // matrix-free from rho (set_level_rho): nothing to build
        } else if (Pv.op.form == FORM_RHO) {
          launch_rho_to_mk(Pv.op, 0, Lv.st, c->stream);
          L(c);
        } else {
          Lv.op.st = Pv.op.st;
        }
      } else if (Lv.gather_in) {
        const int nlc = Lv.ntg / c->comm.size;
        launch_rap_time(Pv.op, nlc, Lv.stpart, c->stream);
        L(c);
        comm_call([&] { comm_allgather(c->comm, Lv.stpart, Lv.st, (long long)nlc * layer, c->stream); });
      } else if (Lv.dist) {
        // owned coarse layers from owned fine layer pairs; the ghost layer (first layer of the
        // next slab) comes from the next rank
        launch_rap_time(Pv.op, Lv.nloc, Lv.st, c->stream);
        L(c);
        comm_call([&] { comm_shift_down(c->comm, Lv.st, Lv.st + (long long)Lv.nloc * layer, layer, c->stream); });
      } else {
        launch_rap_time(Pv.op, Lv.op.nl, Lv.st, c->stream);
        L(c);
      }
    }
    check_launch();
  }
  Level& Lc = c->lv.back();
  const long long Nc = Lc.g.N;
  if (Lc.dense) {
    CK(cudaMemsetAsync(Lc.A, 0, (size_t)Nc * Nc * sizeof(double), c->stream));
    launch_dense_assemble(Lc.op, Lc.A, c->stream);
    if (Lc.nf > 0) launch_dense_invert(Lc.A, Nc, Lc.fidx, Lc.nf, Lc.Ainv, Lc.info, c->stream);
    else CK(cudaMemsetAsync(Lc.info, 0, sizeof(int), c->stream));
    L(c, 2);
    check_launch();
  }
  estimate_omegas(c);
  CK(cudaEventRecord(c->e1, c->stream));
  CK(cudaEventSynchronize(c->e1));
  int info = 0;
  if (Lc.dense) CK(cudaMemcpy(&info, Lc.info, sizeof(int), cudaMemcpyDeviceToHost));
  if (info != 0) throw StErr{ST_E_BREAKDOWN, "coarsest-level matrix singular (pivot " + std::to_string(info) + ")"};
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, c->e0, c->e1));
  c->stats.setup_ms = ms;
  c->stats.setups += 1;
  c->have_ops = true;
}

// source vector f (Q~ = Q tau) into `out` (one write pass, per call: no
// full-length vector is kept for it)
void make_source(st_ctx* c, double* out) {
  // UNIFORM / SIN: Q~ = Q tau; EX1 / EX2: Q0 is given already rescaled
  const bool ex = c->src.kind == ST_SRC_EX1 || c->src.kind == ST_SRC_EX2;
  launch_source(c->lv[0].g, c->src, ex ? c->src.Q0 : c->src.Q0 * c->grid.tau, c->grid.tau, out, c->stream);
  L(c);
  check_launch();
}

// eliminated forward RHS b = m_f (f - K xD) + m_c xD (R-1) into `out`; needs the level-0
// operator bound (prepare) when T0 != 0; pool slots 0 and 1 are scratch
void make_forward_rhs(st_ctx* c, double* out) {
  const Geom& g0 = c->lv[0].g;
  make_source(c, out);
  if (c->bcs.T0 != 0.0) {
    double* xd = pool(c, 0);
    double* kxd = pool(c, 1);
    launch_xd(g0, c->bcs.T0, xd, c->stream);
    op_launch(c, 0, MODE_APPLY, false, false, xd, nullptr, kxd);
    launch_rhs_combine(g0, out, kxd, c->bcs.T0, out, c->stream);
    L(c, 2);
  } else {
    launch_rhs_combine(g0, out, nullptr, 0.0, out, c->stream);
    L(c);
  }
  check_launch();
}

void prepare(st_ctx* c, const double* rho) {
  const bool changed = bind_rho(c, rho);
  if (changed || !c->kt_design) {  // k~ table (once per design, not per call)
    set_fine_rho(c, c->lv[0].op.rho);
    c->kt_design = true;
  }
  if (changed) build_ops(c);
}

// ---------------------------------------------------------------------------------------
// V-cycle: damped-Jacobi pre-smoothing from zero, residual,
// restriction, recursion, prolongation + correction, post-smoothing; coarsest: exact.
// r0: scratch for the level-0 residual (a free Krylov-pool slot; level 0 owns no residual vector)
void vcycle(st_ctx* c, int l, bool trans, const double* b, double* x, bool in_graph = false, double* r0 = nullptr);

// levels >= gl0 as one CUDA graph launch (launch latency dominates there)
bool vcycle_graph(st_ctx* c, int l, bool trans, const double* b, double* x) {
  if (!c->opt.use_graphs || l != c->gl0 || c->gl0 < 0) return false;
  Level& Lv = c->lv[l];
  if (b != Lv.b || x != Lv.x) return false;
  const int d = trans ? 1 : 0;
  if (!c->gexec[d]) {
    if (c->geager[d]++ < 1) return false;  // first run eager: kernel attributes / occupancy cached
    cudaGraph_t graph = nullptr;
    const long long l0 = c->launches;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed));
    vcycle(c, l, trans, b, x, true);
    CK(cudaStreamEndCapture(c->stream, &graph));
    c->gkernels[d] = c->launches - l0;
    c->launches = l0;
    CK(cudaGraphInstantiate(&c->gexec[d], graph, 0));
    cudaGraphDestroy(graph);
  }
  CK(cudaGraphLaunch(c->gexec[d], c->stream));
  L(c, c->gkernels[d]);
  return true;
}

// GMRES(k) with right Jacobi preconditioning on level l: the paper's smoother
// (option ST_SMOOTH_GMRES, k = nu_pre from x = 0 / nu_post from x) and the paper's coarsest-level
// solve (option ST_COARSE_GMRES: k = coarse_maxit <= 200 from x = 0, stop at coarse_rtol = 1e-6).
// x <- x + D^-1 V y with V the Arnoldi basis of A D^-1 from r0 = b - A x and y minimising
// ||beta e1 - H y|| (classical Gram-Schmidt). The Hessenberg, Givens rotations and the triangular
// solve stay on the device (gm_*_kernel, csrc/krylov.cu). rtol = 0: exactly k steps, no host
// synchronisation (the small levels keep their CUDA graph); rtol > 0: the residual estimate |g_{j+1}|
// is read back every `chk` steps and the iteration stops once |g_{j+1}| <= rtol ||r0|| (host
// decisions: no graph). Vectors: the basis Lv.gv, z = D^-1 V_j in Lv.t (read as the x tile of the
// apply), u = V y in the first unused basis slot. st: device state (gm_layout(k)); dd: dot scratch
// (k + 2 doubles, then the norm at dd[kMaxBasis + 8] and ||r0||^2 at dd[kMaxBasis + 16]).
// Returns the steps taken.
int gmres_jacobi(st_ctx* c, int l, bool trans, const double* b, double* x, bool from_zero, int k, double rtol,
                 double* st, double* dd, double* rl, int chk = 4) {
  Level& Lv = c->lv[l];
  if (k <= 0) return 0;
  const long long N = Lv.g.N, ld = Lv.gld;
  double* V = Lv.gv;
  double* z = Lv.t;
  double* dn = dd + kMaxBasis + 8;
  double* d0 = dd + kMaxBasis + 16;
  const double* r0 = b;
  if (!from_zero) {
    op_launch(c, l, MODE_RESID, trans, true, x, b, rl);
    r0 = rl;
  }
  launch_mdot(r0, nullptr, 0, 0, N, d0, c->ws, c->stream);
  launch_gm_init(st, k, d0, c->stream);
  launch_scale_dev(r0, V, d0, N, c->stream);
  L(c, 3);
  int jend = k;
  for (int j = 0; j < k; ++j) {
    double* vj = V + (long long)j * ld;
    double* w = V + (long long)(j + 1) * ld;
    launch_op(Lv.op, MODE_JAC0, trans, true, nullptr, vj, z, 1.0, c->stream);  // z = D^-1 V_j
    op_launch(c, l, MODE_APPLY, trans, true, z, nullptr, w);                   // w = A z
    launch_mdot(w, V, ld, j + 1, N, dd, c->ws, c->stream);                     // h = V^T w
    launch_maxpy_norm(w, V, ld, j + 1, dd, nullptr, N, dn, c->ws, c->stream);  // w -= V h, ||w||^2
    launch_gm_col(st, k, j, dd, dn, c->stream);
    launch_scale_dev(w, w, dn, N, c->stream);                                  // V_{j+1} = w / ||w||
    L(c, 5 + (j + 16) / 16);
    if (rtol > 0.0 && ((j + 1) % chk == 0 || j + 1 == k)) {
      CK(cudaMemcpyAsync(c->hsmall + 470, st + j + 1, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaMemcpyAsync(c->hsmall + 471, d0, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      const double res = std::fabs(c->hsmall[470]), beta = std::sqrt(std::max(c->hsmall[471], 0.0));
      if (!(res > rtol * beta)) {  // converged (or a non-finite estimate: stop and use what we have)
        jend = j + 1;
        break;
      }
    }
  }
  launch_gm_solve(st, k, jend, c->stream);
  double* u = V + (long long)jend * ld;
  CK(cudaMemsetAsync(u, 0, (size_t)N * sizeof(double), c->stream));
  launch_lincomb(u, V, ld, jend, st + gm_y_offset(k), N, c->stream);           // u = V y
  L(c, 2);
  if (from_zero) {
    launch_op(Lv.op, MODE_JAC0, trans, true, nullptr, u, x, 1.0, c->stream);   // x = D^-1 u
    L(c);
  } else {
    launch_op(Lv.op, MODE_JAC0, trans, true, nullptr, u, z, 1.0, c->stream);
    launch_lincomb(x, z, 0, 1, c->dsmall + 510, N, c->stream);                 // x += z (dsmall[510] = 1)
    L(c, 2);
  }
  check_launch();
  return jend;
}

void gmres_smooth(st_ctx* c, int l, bool trans, const double* b, double* x, bool from_zero, double* rl) {
  const int k = from_zero ? c->opt.nu_pre : c->opt.nu_post;
  gmres_jacobi(c, l, trans, b, x, from_zero, k, c->opt.smoother_rtol, c->gsm, c->gsm + 1024, rl, 1);
}

void vcycle(st_ctx* c, int l, bool trans, const double* b, double* x, bool in_graph, double* r0) {
  Level& Lv = c->lv[l];
  double* rl = l == 0 ? r0 : Lv.r;
  if (!rl) throw StErr{ST_E_INVALID_ARG, "internal: level-0 V-cycle without a residual scratch vector"};
  if (!in_graph && vcycle_graph(c, l, trans, b, x)) return;
  if (Lv.dense) {
    launch_dense_solve(Lv.Ainv, Lv.nf, Lv.fidx, Lv.fpos, Lv.g.N, trans, b, x, c->stream);
    L(c);
    return;
  }
  if (Lv.cgm) {  // the paper's coarsest solve: GMRES(<= coarse_maxit)-Jacobi to coarse_rtol
    c->coarse_its += gmres_jacobi(c, l, trans, b, x, true, c->opt.coarse_maxit, c->opt.coarse_rtol, c->cgs,
                                  c->cgs + gm_y_offset(c->opt.coarse_maxit) + c->opt.coarse_maxit + 32, Lv.r);
    return;
  }
  Level& Nx = c->lv[l + 1];
  if (c->opt.smoother == ST_SMOOTH_GMRES) {  // one replicated level (slabs are rejected at setup)
    gmres_smooth(c, l, trans, b, x, true, rl);
    op_launch(c, l, MODE_RESID, trans, true, x, b, rl);
    launch_restrict(Lv.g, Nx.g, Nx.kind, rl, Nx.b, c->stream);
    L(c);
    vcycle(c, l + 1, trans, Nx.b, Nx.x, in_graph);
    launch_prolong_add(Lv.g, Nx.g, Nx.kind, Nx.x, x, c->stream);
    L(c);
    gmres_smooth(c, l, trans, b, x, false, rl);
    return;
  }
  // sweep counts: nu_pre / nu_post on the fine level (and on coarse levels of >= nu_fine_nodes global
  // nodes), nu_coarse on the other coarse levels
  const long long gnodes = (long long)(Lv.ntg + 1) * (c->sd == 2 ? (long long)Lv.g.nn * Lv.g.nn
                                                                 : (long long)Lv.g.nn * Lv.g.nn * Lv.g.nn);
  const bool coarse_nu = l > 0 && c->opt.nu_coarse > 0 &&
                         !(c->opt.nu_fine_nodes > 0 && gnodes >= c->opt.nu_fine_nodes);
  const int npre = coarse_nu ? c->opt.nu_coarse : c->opt.nu_pre;
  const int npost = coarse_nu ? c->opt.nu_coarse : c->opt.nu_post;
  const int total = npre + npost;
  double* cur = (total % 2 == 1) ? x : Lv.t;
  double* oth = (cur == x) ? Lv.t : x;
  op_launch(c, l, MODE_JAC0, trans, true, nullptr, b, cur);
  halo(c, l, cur);
  for (int s = 1; s < npre; ++s) {
    op_launch(c, l, MODE_JAC, trans, true, cur, b, oth);
    halo(c, l, oth);
    std::swap(cur, oth);
  }
  op_launch(c, l, MODE_RESID, trans, true, cur, b, rl);
  if (Nx.kind == KIND_TIME) halo(c, l, rl);  // time restriction reads the next slab's first plane
  if (Nx.gather_in) {  // agglomeration: restrict in slab form, gather onto every rank
    launch_restrict(Lv.g, Nx.gs, Nx.kind, rl, Nx.bpart, c->stream);
    L(c);
    gather_planes(c, Nx, Nx.bpart, Nx.b);
  } else {
    launch_restrict(Lv.g, Nx.g, Nx.kind, rl, Nx.b, c->stream);
    L(c);
  }
  vcycle(c, l + 1, trans, Nx.b, Nx.x, in_graph);
  // prolongation + correction, fused into the first post-sweep where the level kernel can read
  // x + P e itself (tc2d, space-coarsened next level, one GPU; options fuse_prolong = 0: separate kernels)
  int s0 = 0;
  // not on level 0: there the fused sweep costs more than sweep + prolongation — tc2d: 201 vs 90 + 45 us
  // (profiles/r01/launches_c2_v42_summary.txt), the correction pass weighs on an issue-bound kernel; the
  // same fusion in tv2d (r02): config 3 689 -> 671 MDOF/s, the 512^2 x 512 slab 562 -> 556
  // (profiles/r02/ab_r2.log)
  if (l > 0 && npost > 0 && c->opt.fuse_prolong && Nx.kind == KIND_SPACE && c->comm.size <= 1 &&
      c->opt.kernel_family == ST_KERNELS_TMA &&
      launch_op_tc2d_pro(Lv.op, Nx.g, trans, cur, Nx.x, b, oth, Lv.omega > 0.0 ? Lv.omega : c->opt.omega, c->stream)) {
    L(c);
    std::swap(cur, oth);
    s0 = 1;
  } else {
    launch_prolong_add(Lv.g, Nx.g, Nx.kind, Nx.x, cur, c->stream);
    L(c);
    if (npost == 0) halo(c, l, cur);
  }
  for (int s = s0; s < npost; ++s) {
    op_launch(c, l, MODE_JAC, trans, true, cur, b, oth);
    halo(c, l, oth);
    std::swap(cur, oth);
  }
}

void sync_small(st_ctx* c, int off, int n) {
  CK(cudaMemcpyAsync(c->hsmall + off, c->dsmall + off, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
}

// FGMRES(m), right preconditioned by one V-cycle (Saad 1993); with options krylov =
// ST_KRYLOV_GMRES the same Arnoldi process without the Z vectors: z_j = M V_j goes to one scratch
// vector and the cycle ends with x += M (V y) (one more V-cycle; M is a fixed linear map). Classical
// Gram-Schmidt (fused multi-dot + fused multi-AXPY) with one conditional re-orthogonalisation
// (DGKS, eta = 0.1: st_ctx::dgks_eta2). Convergence on the TRUE relative residual ||b - A x|| / ||b|| <= rtol (R-14).
// The Arnoldi vectors are stored unnormalised, v_i = sg_i V_i: the V-cycle and the operator are
// linear, so z_j = sg_j M V_j and A z_j = sg_j A (M V_j), and every scale is folded into the
// host-side Hessenberg / the device-side AXPY weights (no separate scaling pass over memory).
int fgmres(st_ctx* c, bool trans, const double* b, double* x) {
  const long long N = c->Nown;      // inner products and updates over this rank's owned planes
  const long long vo = c->voff;
  const int m = c->opt.restart;
  const double rtol = c->opt.rtol;
  const long long ld = c->ld;
  double* dh = c->dsmall;        // [0..63] g, [64..127] reorth g, [128..191] y, [256..319] sg^2
  double* hh = c->hsmall;
  double* ds2 = dh + 256;
  const bool flex = c->opt.krylov == ST_KRYLOV_FGMRES;
  std::vector<double> H((size_t)(m + 1) * m, 0.0), cs(m), sn(m), gv(m + 1), y(m), sg(m + 1);
  CK(cudaEventRecord(c->e0, c->stream));
  // ||b||
  launch_mdot(b + vo, nullptr, 0, 0, N, dh + 200, c->ws, c->stream);
  L(c);
  allreduce(c, dh + 200, 1);
  sync_small(c, 200, 1);
  const double bnorm = std::sqrt(hh[200]);
  int its = 0, restarts = 0, status = ST_OK, nvc = 0;
  double relres = 0.0;
  bool conv = false;
  if (bnorm == 0.0) {
    CK(cudaMemsetAsync(x, 0, c->N * sizeof(double), c->stream));
    conv = true;
  }
  while (!conv) {
    // true residual r = b - A x into V_0
    op_launch(c, 0, MODE_RESID, trans, true, x, b, c->V);
    launch_mdot(c->V + vo, nullptr, 0, 0, N, dh + 200, c->ws, c->stream);
    L(c);
    allreduce(c, dh + 200, 1);
    sync_small(c, 200, 1);
    const double beta = std::sqrt(hh[200]);
    relres = beta / bnorm;
    if (!std::isfinite(beta)) { status = ST_E_BREAKDOWN; break; }
    if (relres <= rtol) { conv = true; break; }
    if (its >= c->opt.maxit) { status = ST_E_NOT_CONVERGED; break; }
    sg[0] = 1.0 / beta;
    hh[256] = sg[0] * sg[0];
    CK(cudaMemcpyAsync(ds2, hh + 256, sizeof(double), cudaMemcpyHostToDevice, c->stream));
    std::fill(gv.begin(), gv.end(), 0.0);
    gv[0] = beta;
    int jend = 0;
    for (int j = 0; j < m; ++j) {
      double* vj = c->V + (long long)j * ld;
      double* zj = flex ? c->Z + (long long)j * ld : c->Z;
      double* w = c->V + (long long)(j + 1) * ld;
      vcycle(c, 0, trans, vj, zj, false, w);                             // Z_j = M V_j (W: scratch)
      ++nvc;
      op_launch(c, 0, MODE_APPLY, trans, true, zj, nullptr, w);         // W = A Z_j
      launch_mdot(w + vo, c->V + vo, ld, j + 1, N, dh, c->ws, c->stream);  // g_i = V_i . W, ||W||^2
      allreduce(c, dh, j + 2);
      // W -= sum sg_i^2 g_i V_i; with it (j + 1 <= 16) the DGKS coefficients V_i . W and ||W||^2
      const bool fused = launch_maxpy_dots(w + vo, c->V + vo, ld, j + 1, dh, ds2, N, dh + 64, c->ws, c->stream);
      if (fused) {
        allreduce(c, dh + 64, j + 2);
      } else {
        launch_maxpy_norm(w + vo, c->V + vo, ld, j + 1, dh, ds2, N, dh + 196, c->ws, c->stream);
        allreduce(c, dh + 196, 1);
      }
      L(c, (j + 16) / 16 + 1);
      check_launch();
      CK(cudaMemcpyAsync(hh, dh, (j + 2) * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      if (fused) CK(cudaMemcpyAsync(hh + 64, dh + 64, (j + 2) * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      else CK(cudaMemcpyAsync(hh + 196, dh + 196, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      double* hcol = &H[(size_t)j * (m + 1)];
      for (int i = 0; i <= j; ++i) hcol[i] = sg[i] * sg[j] * hh[i];  // h_ij = v_i . (A z_j)
      double ww = hh[j + 1], w2 = fused ? hh[64 + j + 1] : hh[196];
      if (w2 < c->dgks_eta2 * ww) {  // DGKS re-orthogonalisation
        if (!fused) {
          launch_mdot(w + vo, c->V + vo, ld, j + 1, N, dh + 64, c->ws, c->stream);
          allreduce(c, dh + 64, j + 1);
        }
        launch_maxpy_norm(w + vo, c->V + vo, ld, j + 1, dh + 64, ds2, N, dh + 196, c->ws, c->stream);
        allreduce(c, dh + 196, 1);
        L(c, (j + 16) / 16 + 1);
        CK(cudaMemcpyAsync(hh + 64, dh + 64, (j + 1) * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(hh + 196, dh + 196, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        for (int i = 0; i <= j; ++i) hcol[i] += sg[i] * sg[j] * hh[64 + i];
        w2 = hh[196];
      }
      const double hn = sg[j] * std::sqrt(std::max(w2, 0.0));  // ||A z_j - V h||
      hcol[j + 1] = hn;
      ++its;
      if (hn > 0.0) {
        sg[j + 1] = sg[j] / hn;
        hh[257 + j] = sg[j + 1] * sg[j + 1];
        CK(cudaMemcpyAsync(ds2 + j + 1, hh + 257 + j, sizeof(double), cudaMemcpyHostToDevice, c->stream));
      }
      // Givens rotations
      for (int i = 0; i < j; ++i) {
        double t = cs[i] * hcol[i] + sn[i] * hcol[i + 1];
        hcol[i + 1] = -sn[i] * hcol[i] + cs[i] * hcol[i + 1];
        hcol[i] = t;
      }
      double den = std::hypot(hcol[j], hcol[j + 1]);
      if (den == 0.0) { status = ST_E_BREAKDOWN; jend = j; break; }
      cs[j] = hcol[j] / den;
      sn[j] = hcol[j + 1] / den;
      hcol[j] = den;
      hcol[j + 1] = 0.0;
      gv[j + 1] = -sn[j] * gv[j];
      gv[j] = cs[j] * gv[j];
      jend = j + 1;
      if (!std::isfinite(gv[j + 1])) { status = ST_E_BREAKDOWN; break; }
      if (std::fabs(gv[j + 1]) <= rtol * bnorm || hn == 0.0 || its >= c->opt.maxit) break;
    }
    if (status == ST_E_BREAKDOWN && jend == 0) break;
    // back substitution H y = g, x += sum_i y_i z_i = sum_i (y_i sg_i) Z_i
    for (int i = jend - 1; i >= 0; --i) {
      double s = gv[i];
      for (int k = i + 1; k < jend; ++k) s -= H[(size_t)k * (m + 1) + i] * y[k];
      y[i] = s / H[(size_t)i * (m + 1) + i];
    }
    for (int i = 0; i < jend; ++i) hh[128 + i] = y[i] * sg[i];
    CK(cudaMemcpyAsync(dh + 128, hh + 128, jend * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    if (flex) {
      launch_lincomb(x + vo, c->Z + vo, ld, jend, dh + 128, N, c->stream);
      L(c);
    } else {  // u = V (y sg) into the z scratch, then x += M u (V_0 receives M u, V_1 is scratch)
      double* u = c->Z;
      CK(cudaMemsetAsync(u, 0, (size_t)c->N * sizeof(double), c->stream));
      launch_lincomb(u + vo, c->V + vo, ld, jend, dh + 128, N, c->stream);
      L(c);
      vcycle(c, 0, trans, u, c->V, false, c->V + ld);
      ++nvc;
      launch_lincomb(x + vo, c->V + vo, 0, 1, dh + 510, N, c->stream);  // dsmall[510] = 1
      L(c);
    }
    check_launch();
    halo(c, 0, x);
    ++restarts;
    if (status == ST_E_BREAKDOWN) status = ST_OK;  // lucky/hard breakdown: re-check true residual
  }
  CK(cudaEventRecord(c->e1, c->stream));
  CK(cudaEventSynchronize(c->e1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, c->e0, c->e1));
  c->stats.solve_ms = ms;
  c->stats.iterations = its;
  c->stats.restarts = restarts;
  c->stats.vcycles = nvc;
  c->stats.rel_residual = relres;
  c->stats.converged = conv ? 1 : 0;
  c->stats.n_levels = (int)c->lv.size();
  if (!conv && status == ST_OK) status = ST_E_NOT_CONVERGED;
  return conv ? ST_OK : status;
}

double* out_ptr(st_ctx* c, double* p, long long n, int slot, bool copy_in, bool* staged) {
  if (!p) throw StErr{ST_E_INVALID_ARG, "null pointer"};
  if (is_device_ptr(p)) {
    *staged = false;
    return p;
  }
  double* d = stage(c, slot, n);
  if (copy_in) CK(cudaMemcpyAsync(d, p, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  *staged = true;
  return d;
}

void copy_back(st_ctx* c, double* host, const double* dev, long long n) {
  CK(cudaMemcpyAsync(host, dev, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
}

// owned planes of an internal fine vector, as a geometry starting at plane o0
Geom owned_geom(const st_ctx* c) {
  Geom g = c->lv[0].g;
  g.nt = c->nown - 1;
  g.N = g.P * c->nown;
  g.pg0 += c->o0;
  return g;
}
// caller vector (dense layout of the owned planes, host or device) -> internal padded vector;
// ghost = true refreshes the ghost planes (vectors read through the stencil)
// Host vectors of the nodal calls share ONE staging buffer (slot 0): every use is stream-ordered (the
// relayout kernel reading staged data precedes the next copy into the buffer) — config 3's e2e path
// then stages through one 8.6 GB buffer instead of four.
void pack_in(st_ctx* c, const double* user, double* internal, int /*slot*/, bool ghost = false) {
  const double* d = in_ptr(c, user, c->Nd, 0);
  launch_relayout(c->gd0, d, c->lv[0].g, internal + c->voff, c->stream);
  L(c);
  if (ghost) halo(c, 0, internal);
}
// internal padded vector -> caller vector (dense layout, host or device); synchronises
void unpack_out(st_ctx* c, const double* internal, double* user, int /*slot*/) {
  const int slot = 0;
  if (!user) throw StErr{ST_E_INVALID_ARG, "null pointer"};
  const Geom go = owned_geom(c);
  if (is_device_ptr(user)) {
    launch_relayout(go, internal + c->voff, c->gd0, user, c->stream);
    L(c);
    CK(cudaStreamSynchronize(c->stream));
  } else {
    double* d = stage(c, slot, c->Nd);
    launch_relayout(go, internal + c->voff, c->gd0, d, c->stream);
    L(c);
    copy_back(c, user, d, c->Nd);
  }
}

template <class F> int guarded(F&& f) {
  try {
    return f();
  } catch (const StErr& e) {
    g_last_error = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return ST_E_CUDA;
  } catch (...) {
    g_last_error = "unknown error";
    return ST_E_CUDA;
  }
}

void free_ctx(st_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  for (auto& Lv : c->lv) {
    if (Lv.st_owned && Lv.st) cudaFree(Lv.st);
    cudaFree(Lv.mid);
    cudaFree(Lv.gv);
    cudaFree(Lv.A); cudaFree(Lv.Ainv); cudaFree(Lv.info); cudaFree(Lv.fidx); cudaFree(Lv.fpos);
  }
  for (double* p : c->vallocs) cudaFree(p);
  cudaFree(c->ws.partial); cudaFree(c->ws.counter);
  cudaFree(c->dsmall);
  if (c->hsmall) cudaFreeHost(c->hsmall);
  cudaFree(c->rho_stage);
  cudaFree(c->gsm);
  cudaFree(c->cgs);
  cudaFree(c->kt);
  comm_release(c->comm);
  cudaFree(c->fbuf);
  cudaFree(c->fw);
  for (auto& Lv : c->lv) cudaFree(Lv.stpart);
  for (int i = 0; i < 4; ++i) cudaFree(c->io_stage[i]);
  for (int d = 0; d < 2; ++d)
    if (c->gexec[d]) cudaGraphExecDestroy(c->gexec[d]);
  if (c->e0) cudaEventDestroy(c->e0);
  if (c->e1) cudaEventDestroy(c->e1);
  for (int k = 0; k < 2; ++k) {
    if (c->ev_rdy[k]) cudaEventDestroy(c->ev_rdy[k]);
    if (c->ev_done[k]) cudaEventDestroy(c->ev_done[k]);
  }
  if (c->cstream) cudaStreamDestroy(c->cstream);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

// entries of dJ this rank writes (owned element layers; time-constant: the spatial design)
long long sens_count(const st_ctx* c) {
  const Level& L0 = c->lv[0];
  long long nsp = 1;
  for (int d = 0; d < c->sd; ++d) nsp *= c->grid.n;
  return c->tc ? nsp : nsp * (L0.dist ? L0.nloc : L0.g.nt);
}

// dJ (device, sens_count entries) from the internal T and lambda (ghost planes refreshed)
void sens_core(st_ctx* c, const double* r, const double* Ti, const double* li, double* dj) {
  const Level& L0 = c->lv[0];
  OpDesc op = L0.op;
  op.rho = r;
  op.g.nt = L0.dist ? L0.nloc : L0.g.nt;  // owned element layers
  launch_sensitivity(op, Ti, li, dj, c->stream);
  L(c);
  check_launch();
  if (c->tc) allreduce(c, dj, sens_count(c));  // time-constant design: sum through time over all slabs
}

// caller vector (host or device, dense owned planes) -> internal vector; a host vector is copied into
// `scratch` (a free device buffer of >= Nd entries) first
void pack_in_via(st_ctx* c, const double* user, double* internal, double* scratch, bool ghost) {
  if (!user) throw StErr{ST_E_INVALID_ARG, "null pointer"};
  const double* d = user;
  if (!is_device_ptr(user)) {
    CK(cudaMemcpyAsync(scratch, user, c->Nd * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    d = scratch;
  }
  launch_relayout(c->gd0, d, c->lv[0].g, internal + c->voff, c->stream);
  L(c);
  if (ghost) halo(c, 0, internal);
}

// side-stream copies of st_design_step: slot k's copy starts once the library stream reaches this
// point (ev_rdy[k]) and runs beside whatever the library stream does next; side_wait(k) makes the
// library stream wait for it (ev_done[k])
void side_copy(st_ctx* c, int k, void* dst, const void* src, long long n, cudaMemcpyKind kind) {
  if (!c->cstream) {
    CK(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      CK(cudaEventCreateWithFlags(&c->ev_rdy[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_done[i], cudaEventDisableTiming));
    }
  }
  CK(cudaEventRecord(c->ev_rdy[k], c->stream));
  CK(cudaStreamWaitEvent(c->cstream, c->ev_rdy[k], 0));
  CK(cudaMemcpyAsync(dst, src, n * sizeof(double), kind, c->cstream));
  CK(cudaEventRecord(c->ev_done[k], c->cstream));
}
void side_wait(st_ctx* c, int k) { CK(cudaStreamWaitEvent(c->stream, c->ev_done[k], 0)); }

}  // namespace

// =======================================================================================
extern "C" {

int st_abi_version(void) { return ST_ABI_VERSION; }

void st_default_options(st_options_t* o) {
  if (!o) return;
  memset(o, 0, sizeof(*o));
  o->design_mode = ST_SPACE_TIME;
  o->rtol = 1e-8;
  o->maxit = 500;
  o->restart = 16;
  o->smoother = ST_SMOOTH_JACOBI;
  // measured over configs 2-5 (profiles/r01/nu_sweep.log, nu_split*.log): the
  // fine-level sweeps are the expensive ones, the coarse ones buy the convergence
  o->nu_pre = 2;
  o->nu_post = 2;
  o->nu_coarse = 5;
  o->omega = 0.75;
  o->lambda_crit = 0.5;
  o->coarse_max_nodes = 400;
  o->max_levels = 0;
  o->full_coarsening = 0;
  o->use_graphs = 1;
  o->verbose = 0;
  // 256 Ki nodes per rank: below that a distributed level's sweep (a few us per rank) costs less than
  // the halo exchange each sweep needs (two NCCL plane messages, ~10-20 us), while the replicated
  // level costs one all-gather per V-cycle; config 3 on 8 ranks gathers level 6 (65^2 x 257 nodes, 8.7 MB)
  // instead of level 9 — 33 fewer exchanges per V-cycle
  o->agg_nodes = 262144;
  o->krylov = ST_KRYLOV_FGMRES;
  o->coarse_solver = ST_COARSE_DENSE;
  o->coarse_rtol = 1e-6;
  o->coarse_maxit = 200;
  o->kernel_family = ST_KERNELS_TMA;
  o->chunk_planes = 0;
  o->max_ctas = 0;
  o->fuse_prolong = 1;
  o->omega_factor = 1.9;
  o->dgks_eta = 0.1;
  o->graph_max_nodes = 0;
  o->smoother_rtol = 0.0;
  // coarse levels of >= 1e7 nodes sweep like the fine level (2+2): measured config 3 511 -> 607 MDOF/s
  // (levels 1-3: 2.7e8, 6.8e7, 1.7e7 nodes), config 5 247 -> 271, the 512^2 x 512 slab 486 -> 551;
  // configs 2 / 4 have no such coarse level (profiles/r02/nu_fine_nodes.log)
  o->nu_fine_nodes = 10000000;
  // 32-byte rows: every TMA box row and every tile-row store starts on a DRAM sector (config-3 fine
  // residual 7.80 -> 7.61 ms, sweep 6.79 -> 6.78 ms; 16 doubles: 7.44 / 6.76 ms but +1.4 % memory;
  // profiles/r02/kbench_pitch.log)
  o->pitch_align = 4;
}

const char* st_strerror(int code) {
  switch (code) {
    case ST_OK: return "ok";
    case ST_E_INVALID_ARG: return "invalid argument";
    case ST_E_DIVISIBILITY: return "grid not divisible along the coarsening direction";
    case ST_E_NOT_CONVERGED: return "solver did not converge";
    case ST_E_BREAKDOWN: return "Krylov breakdown";
    case ST_E_OOM: return "out of device memory";
    case ST_E_CUDA: return "CUDA error";
    case ST_E_NCCL: return "NCCL error";
    case ST_E_UNSUPPORTED: return "unsupported option";
    default: return "unknown";
  }
}

const char* st_last_error(void) { return g_last_error.c_str(); }

int st_setup(const st_grid_t* grid, const st_materials_t* mats, const st_bcs_t* bcs, const st_source_t* src,
             const st_options_t* opts, const st_dist_t* dist, st_ctx_t** out) {
  return guarded([&]() -> int {
    if (!grid || !mats || !bcs || !src || !out) throw StErr{ST_E_INVALID_ARG, "null argument"};
    *out = nullptr;
    if (grid->sdim != 2 && grid->sdim != 3) throw StErr{ST_E_INVALID_ARG, "sdim must be 2 or 3"};
    if (grid->n < 2 || grid->nt < 2) throw StErr{ST_E_INVALID_ARG, "n and nt must be >= 2"};
    if (!(grid->L > 0) || !(grid->tau > 0)) throw StErr{ST_E_INVALID_ARG, "L and tau must be > 0"};
    if (grid->n > (1 << 20) || grid->nt > (1 << 24)) throw StErr{ST_E_INVALID_ARG, "grid too large"};
    if (!(mats->C_ins > 0) || !(mats->C_con > 0) || !(mats->k_ins > 0) || !(mats->k_con > 0))
      throw StErr{ST_E_INVALID_ARG, "material constants must be > 0"};
    if (bcs->has_patch && bcs->face != 0) throw StErr{ST_E_UNSUPPORTED, "only face 0 (x1 = 0) supported"};
    if (src->kind < ST_SRC_UNIFORM || src->kind > ST_SRC_EX2) throw StErr{ST_E_UNSUPPORTED, "source kind"};
    if (src->kind == ST_SRC_EX2 && (grid->sdim != 2 || !(src->sigma > 0)))
      throw StErr{ST_E_INVALID_ARG, "ST_SRC_EX2: (2+1)D grid and sigma > 0"};
    if (dist && dist->size > 1) {
      if (dist->rank < 0 || dist->rank >= dist->size) throw StErr{ST_E_INVALID_ARG, "rank out of range"};
      if (grid->nt % dist->size != 0) throw StErr{ST_E_DIVISIBILITY, "time slabs: nt must be divisible by the rank count"};
      if (dist->transport == ST_COMM_NCCL && !dist->nccl_comm) throw StErr{ST_E_INVALID_ARG, "NCCL transport needs nccl_comm"};
      if (dist->transport == ST_COMM_NCCL) {  // the communicator must be the one the slabs assume
        int cnt = -1, r = -1;
        if (nccl_comm_count(dist->nccl_comm, &cnt, &r) != 0)
          throw StErr{ST_E_NCCL, "ncclCommCount / ncclCommUserRank failed"};
        if (cnt != dist->size || r != dist->rank)
          throw StErr{ST_E_NCCL, "NCCL communicator has " + std::to_string(cnt) + " ranks (rank " + std::to_string(r) +
                                     "), st_dist_t says " + std::to_string(dist->size) + " (rank " +
                                     std::to_string(dist->rank) + ")"};
        if (dist->rank == 0 || (opts && opts->verbose))
          fprintf(stderr, "libst: time slabs over NCCL: ncclCommCount = %d, rank %d of %d, device %d\n", cnt, r,
                  dist->size, dist->device);
      }
      if (dist->transport == ST_COMM_HOST &&
          (!dist->host.sendrecv || !dist->host.allreduce_sum || !dist->host.allgather))
        throw StErr{ST_E_INVALID_ARG, "host transport needs sendrecv, allreduce_sum and allgather"};
      if (dist->transport != ST_COMM_NCCL && dist->transport != ST_COMM_HOST)
        throw StErr{ST_E_INVALID_ARG, "size > 1 needs a transport (ST_COMM_NCCL or ST_COMM_HOST)"};
      if (opts && (opts->smoother == ST_SMOOTH_GMRES || opts->full_coarsening))
        throw StErr{ST_E_UNSUPPORTED, "time slabs: Jacobi smoother and semi-coarsening only"};
    }
    st_ctx* c = new st_ctx();
    try {
      c->grid = *grid;
      c->mats = *mats;
      c->bcs = *bcs;
      c->src = *src;
      if (opts) c->opt = *opts;
      else st_default_options(&c->opt);
      if (c->opt.restart < 1 || c->opt.restart > 60) throw StErr{ST_E_INVALID_ARG, "restart must be in [1, 60]"};
      if (c->opt.nu_pre < 1 || c->opt.nu_post < 0 || c->opt.nu_coarse < 0)
        throw StErr{ST_E_INVALID_ARG, "nu_pre >= 1, nu_post >= 0, nu_coarse >= 0"};
      if (c->opt.smoother != ST_SMOOTH_JACOBI && c->opt.smoother != ST_SMOOTH_GMRES)
        throw StErr{ST_E_UNSUPPORTED, "smoother: ST_SMOOTH_JACOBI or ST_SMOOTH_GMRES"};
      if (c->opt.smoother == ST_SMOOTH_GMRES && (c->opt.nu_pre > 24 || c->opt.nu_post > 24))
        throw StErr{ST_E_INVALID_ARG, "GMRES smoother: nu_pre, nu_post <= 24"};
      if (c->opt.coarse_max_nodes < 8) c->opt.coarse_max_nodes = 8;
      if (c->opt.kernel_family < ST_KERNELS_TMA || c->opt.kernel_family > ST_KERNELS_TMA2D)
        throw StErr{ST_E_INVALID_ARG, "kernel_family: ST_KERNELS_*"};
      if (c->opt.krylov != ST_KRYLOV_FGMRES && c->opt.krylov != ST_KRYLOV_GMRES)
        throw StErr{ST_E_INVALID_ARG, "krylov: ST_KRYLOV_FGMRES or ST_KRYLOV_GMRES"};
      if (c->opt.krylov == ST_KRYLOV_GMRES && c->opt.smoother != ST_SMOOTH_JACOBI)
        throw StErr{ST_E_UNSUPPORTED, "ST_KRYLOV_GMRES needs a fixed linear preconditioner (ST_SMOOTH_JACOBI)"};
      if (c->opt.coarse_solver != ST_COARSE_DENSE && c->opt.coarse_solver != ST_COARSE_GMRES)
        throw StErr{ST_E_INVALID_ARG, "coarse_solver: ST_COARSE_DENSE or ST_COARSE_GMRES"};
      if (c->opt.krylov == ST_KRYLOV_GMRES && c->opt.coarse_solver != ST_COARSE_DENSE)
        throw StErr{ST_E_UNSUPPORTED, "ST_KRYLOV_GMRES needs a fixed linear preconditioner (ST_COARSE_DENSE)"};
      if (c->opt.coarse_rtol <= 0.0) c->opt.coarse_rtol = 1e-6;
      if (c->opt.coarse_maxit <= 0) c->opt.coarse_maxit = 200;
      if (c->opt.coarse_maxit >= kMaxBasis) throw StErr{ST_E_INVALID_ARG, "coarse_maxit must be < 256"};
      if (c->opt.dgks_eta == 0.0) c->opt.dgks_eta = 0.1;
      c->dgks_eta2 = c->opt.dgks_eta > 0.0 ? c->opt.dgks_eta * c->opt.dgks_eta : 0.0;
      CK(cudaGetDevice(&c->device));
      if (dist && dist->device >= 0) {
        c->device = dist->device;
        CK(cudaSetDevice(c->device));
      }
      if (dist && dist->cuda_stream) {
        c->stream = (cudaStream_t)dist->cuda_stream;
      } else {
        // blocking stream: ordered with work the caller enqueues on the legacy default stream
        // (e.g. PyTorch's default stream), so caller-side fills / copies never race the library
        CK(cudaStreamCreate(&c->stream));
        c->own_stream = true;
      }
      c->sd = grid->sdim;
      c->tc = (c->opt.design_mode == ST_TIME_CONSTANT);
      if (c->opt.agg_nodes <= 0) c->opt.agg_nodes = 262144;
      if (dist && dist->size > 1) {
        c->comm.rank = dist->rank;
        c->comm.size = dist->size;
        c->comm.kind = dist->transport;
        c->comm.nccl = dist->nccl_comm;
        c->comm.host = dist->host;
      }
      const double scale = grid->tau / (grid->L * grid->L);
      c->md.Cins = mats->C_ins;
      c->md.dC = mats->C_con - mats->C_ins;
      c->md.pc = mats->p_c;
      c->md.kins = mats->k_ins * scale;
      c->md.dk = (mats->k_con - mats->k_ins) * scale;
      c->md.pk = mats->p_k;
      if (c->opt.pitch_align <= 0) c->opt.pitch_align = 4;
      if (c->opt.pitch_align % 2 != 0 || c->opt.pitch_align > 64)
        throw StErr{ST_E_INVALID_ARG, "pitch_align: an even number of doubles <= 64"};
      t_pitch_align = c->opt.pitch_align;
      build_hierarchy(c);
      assign_slabs(c);
      t_pitch_align = 2;
      setup_forms(c);
      const Level& L0 = c->lv[0];
      c->N = L0.g.N;
      c->o0 = (L0.dist && c->comm.rank > 0) ? 1 : 0;
      c->nown = L0.dist ? L0.nloc + (c->comm.rank == 0 ? 1 : 0) : L0.g.nt + 1;
      c->voff = (long long)c->o0 * L0.g.P;
      c->Nown = (long long)c->nown * L0.g.P;
      c->gd0 = make_geom(c->sd, L0.g.n, c->nown - 1, L0.g.plo, L0.g.phi, false, L0.ntg, L0.g.pg0 + c->o0);
      c->gd0.walls = L0.g.walls;
      c->Nd = nodes_of(c->gd0);
      long long nsp = 1;
      for (int d = 0; d < c->sd; ++d) nsp *= grid->n;
      c->ndesign = c->tc ? nsp : nsp * L0.g.nt;   // space-time: owned layers + the ghost layer
      allocate(c);
      if (c->sd == 2 && !c->tc)  // padded k~ table (launch_ktilde)
        dalloc(&c->kt, (long long)(grid->n + 2) * (grid->n + 2) * (L0.g.nt + 1));
      CK(cudaStreamSynchronize(c->stream));
    } catch (...) {
      free_ctx(c);
      throw;
    }
    *out = c;
    return ST_OK;
  });
}

void st_destroy(st_ctx_t* ctx) { free_ctx(ctx); }

int st_solve(st_ctx_t* c, const double* rho, double* T) {
  return guarded([&]() -> int {
    if (!c) throw StErr{ST_E_INVALID_ARG, "null ctx"};
    CK(cudaSetDevice(c->device));
    prepare(c, rho);
    make_forward_rhs(c, c->rhs);
    pack_in(c, T, c->xint, 0);
    launch_set_bc_values(c->lv[0].g, c->bcs.T0, c->xint, c->stream);  // x_c = xD
    L(c, 2);
    halo(c, 0, c->xint);
    int rc = fgmres(c, false, c->rhs, c->xint);
    unpack_out(c, c->xint, T, 0);
    return rc;
  });
}

int st_adjoint(st_ctx_t* c, const double* rho, const double* dJdT, double* lambda) {
  return guarded([&]() -> int {
    if (!c) throw StErr{ST_E_INVALID_ARG, "null ctx"};
    CK(cudaSetDevice(c->device));
    prepare(c, rho);
    if (dJdT) pack_in(c, dJdT, c->rhs, 1);
    else make_source(c, c->rhs);  // null dJdT: the compliance f^T T, dphi/dT = f (R-8)
    launch_mask_free(c->lv[0].g, c->rhs, c->rhs, c->stream);  // RHS m_f g
    pack_in(c, lambda, c->xint, 0);
    launch_set_bc_values(c->lv[0].g, 0.0, c->xint, c->stream);  // lambda_c = 0
    L(c, 4);
    halo(c, 0, c->xint);
    int rc = fgmres(c, true, c->rhs, c->xint);
    unpack_out(c, c->xint, lambda, 0);
    return rc;
  });
}

int st_sensitivity(st_ctx_t* c, const double* rho, const double* T, const double* lambda, double* dJ) {
  return guarded([&]() -> int {
    if (!c) throw StErr{ST_E_INVALID_ARG, "null ctx"};
    CK(cudaSetDevice(c->device));
    const double* r = rho_device(c, rho);
    // T and lambda into internal slab vectors with ghost planes (element layers of this rank)
    double* Ti = pool(c, 0);
    double* li = pool(c, 1);
    pack_in(c, T, Ti, 1, true);
    pack_in(c, lambda, li, 2, true);
    const long long ndj = sens_count(c);
    bool staged = false;
    double* dj = out_ptr(c, dJ, ndj, 0, false, &staged);  // after the packs' relayouts (stream order)
    sens_core(c, r, Ti, li, dj);
    if (staged) copy_back(c, dJ, dj, ndj);
    else CK(cudaStreamSynchronize(c->stream));
    return ST_OK;
  });
}

int st_design_step(st_ctx_t* c, const double* rho, const double* dJdT, double* T, double* lambda, double* dJ,
                   st_stats_t* fwd_stats) {
  return guarded([&]() -> int {
    if (!c) throw StErr{ST_E_INVALID_ARG, "null ctx"};
    if (!T || !lambda || !dJ) throw StErr{ST_E_INVALID_ARG, "null pointer"};
    CK(cudaSetDevice(c->device));
    const bool hT = !is_device_ptr(T), hl = !is_device_ptr(lambda), hj = !is_device_ptr(dJ);
    // host initial guesses go through the staging buffer S0 on the side stream: T0 while the design-
    // dependent setup runs, lambda0 while the forward solve runs
    double* S0 = (hT || hl) ? stage(c, 0, c->Nd) : nullptr;
    if (hT) side_copy(c, 0, S0, T, c->Nd, cudaMemcpyHostToDevice);
    // ---- forward solve (as st_solve); rho is bound (a host design uploaded) once for the whole step
    prepare(c, rho);
    const double* r = c->lv[0].op.rho;
    make_forward_rhs(c, c->rhs);
    if (hT) side_wait(c, 0);
    launch_relayout(c->gd0, hT ? S0 : T, c->lv[0].g, c->xint + c->voff, c->stream);
    L(c);
    if (hl) side_copy(c, 1, S0, lambda, c->Nd, cudaMemcpyHostToDevice);  // after T0 left S0
    launch_set_bc_values(c->lv[0].g, c->bcs.T0, c->xint, c->stream);
    L(c);
    halo(c, 0, c->xint);
    const int rc1 = fgmres(c, false, c->rhs, c->xint);
    st_stats_t s1 = c->stats;
    // lambda0 (host) -> its internal layout in pool slot 1, freeing S0
    if (hl) {
      side_wait(c, 1);
      launch_relayout(c->gd0, S0, c->lv[0].g, pool(c, 1) + c->voff, c->stream);
      L(c);
    }
    // T -> its dense layout: the caller's device vector, or S0 (kept until the sensitivities; its
    // copy to the host runs on the side stream during the adjoint solve)
    const Geom go = owned_geom(c);
    double* Td = hT ? S0 : T;
    launch_relayout(go, c->xint + c->voff, c->gd0, Td, c->stream);
    L(c);
    if (hT) side_copy(c, 0, T, Td, c->Nd, cudaMemcpyDeviceToHost);
    // ---- adjoint solve (as st_adjoint)
    // (a pool slot used as a DENSE buffer is zeroed again afterwards: the level kernels read the pad
    // entries of internal vectors, which must stay zero)
    if (dJdT) {
      pack_in_via(c, dJdT, c->rhs, pool(c, 0), false);
      if (!is_device_ptr(dJdT)) CK(cudaMemsetAsync(pool(c, 0), 0, c->Nd * sizeof(double), c->stream));
    } else {
      make_source(c, c->rhs);
    }
    launch_mask_free(c->lv[0].g, c->rhs, c->rhs, c->stream);
    L(c);
    if (hl) CK(cudaMemcpyAsync(c->xint, pool(c, 1), c->N * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    else {
      launch_relayout(c->gd0, lambda, c->lv[0].g, c->xint + c->voff, c->stream);
      L(c);
    }
    launch_set_bc_values(c->lv[0].g, 0.0, c->xint, c->stream);
    L(c);
    halo(c, 0, c->xint);
    const int rc2 = fgmres(c, true, c->rhs, c->xint);
    // lambda -> dense (the caller's device vector, or pool slot 0 copied back on the side stream)
    double* ld = hl ? pool(c, 0) : lambda;
    launch_relayout(go, c->xint + c->voff, c->gd0, ld, c->stream);
    L(c);
    if (hl) side_copy(c, 1, lambda, ld, c->Nd, cudaMemcpyDeviceToHost);
    // ---- sensitivities from the internal lambda (xint) and T re-laid out from its dense copy
    halo(c, 0, c->xint);
    double* Ti = pool(c, 1);
    launch_relayout(c->gd0, Td, c->lv[0].g, Ti + c->voff, c->stream);
    L(c);
    halo(c, 0, Ti);
    const long long ndj = sens_count(c);
    double* dj = hj ? pool(c, 2) : dJ;
    sens_core(c, r, Ti, c->xint, dj);
    if (hj) {
      CK(cudaMemcpyAsync(dJ, dj, ndj * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaMemsetAsync(dj, 0, ndj * sizeof(double), c->stream));
    }
    if (hl) {
      side_wait(c, 1);
      CK(cudaMemsetAsync(ld, 0, c->Nd * sizeof(double), c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    if (c->cstream) CK(cudaStreamSynchronize(c->cstream));
    if (fwd_stats) *fwd_stats = s1;
    return rc1 != ST_OK ? rc1 : rc2;
  });
}

// eliminated operator on an arbitrary input: the level kernels assume x = 0 at constrained
// nodes (true for every vector of the solver), so mask first and restore the identity rows
void masked_level_apply(st_ctx* c, int l, const double* x, double* xm, double* y, bool trans, bool bc) {
  const Geom& g = c->lv[l].g;
  if (bc) {
    launch_mask_free(g, x, xm, c->stream);
    op_launch(c, l, MODE_APPLY, trans, true, xm, nullptr, y);
    launch_copy_cons(g, x, y, c->stream);
    L(c, 2);
  } else {
    op_launch(c, l, MODE_APPLY, trans, false, x, nullptr, y);
  }
  check_launch();
}

int st_apply(st_ctx_t* c, const double* rho, const double* x, double* y, int transpose, int bc) {
  return guarded([&]() -> int {
    if (!c) throw StErr{ST_E_INVALID_ARG, "null ctx"};
    CK(cudaSetDevice(c->device));
    const double* r = rho_device(c, rho);
    set_fine_rho(c, r);
    c->kt_design = false;  // the table now follows r, not necessarily the cached design
    pack_in(c, x, pool(c, 0), 1, true);
    masked_level_apply(c, 0, pool(c, 0), pool(c, 1), pool(c, 2), transpose != 0, bc != 0);
    unpack_out(c, pool(c, 2), y, 2);
    return ST_OK;
  });
}

int st_level_apply(st_ctx_t* c, const double* rho, int level, const double* x, double* y, int transpose) {
  return guarded([&]() -> int {
    if (!c) throw StErr{ST_E_INVALID_ARG, "null ctx"};
    if (level < 0 || level >= (int)c->lv.size()) throw StErr{ST_E_INVALID_ARG, "level out of range"};
    if (c->comm.size > 1) throw StErr{ST_E_UNSUPPORTED, "st_level_apply: single-rank contexts only"};
    CK(cudaSetDevice(c->device));
    prepare(c, rho);
    Level& Lv = c->lv[level];
    const Geom gd = dense_of(Lv.g);
    const long long nd = nodes_of(Lv.g);
    double* xi = level == 0 ? pool(c, 0) : Lv.x;
    double* xm = level == 0 ? pool(c, 1) : Lv.b;
    const double* xd = in_ptr(c, x, nd, 1);
    launch_relayout(gd, xd, Lv.g, xi, c->stream);
    L(c);
    masked_level_apply(c, level, xi, xm, Lv.t, transpose != 0, true);
    bool staged = false;
    double* yd = out_ptr(c, y, nd, 2, false, &staged);
    launch_relayout(Lv.g, Lv.t, gd, yd, c->stream);
    L(c);
    check_launch();
    if (staged) copy_back(c, y, yd, nd);
    else CK(cudaStreamSynchronize(c->stream));
    return ST_OK;
  });
}

int st_level_transfer(st_ctx_t* c, const double* rho, int level, const double* in, double* out, int restrict_) {
  return guarded([&]() -> int {
    if (!c) throw StErr{ST_E_INVALID_ARG, "null ctx"};
    if (level < 0 || level + 1 >= (int)c->lv.size()) throw StErr{ST_E_INVALID_ARG, "level out of range"};
    if (c->comm.size > 1) throw StErr{ST_E_UNSUPPORTED, "st_level_transfer: single-rank contexts only"};
    CK(cudaSetDevice(c->device));
    prepare(c, rho);
    Level& Lv = c->lv[level];
    Level& Nx = c->lv[level + 1];
    const Geom gdf = dense_of(Lv.g), gdc = dense_of(Nx.g);
    const long long nf = nodes_of(Lv.g), ncn = nodes_of(Nx.g);
    double* fine = level == 0 ? pool(c, 0) : Lv.x;
    double* coarse = Nx.b;
    bool staged = false;
    if (restrict_) {  // out (level + 1) = m_c P^T in (level)
      launch_relayout(gdf, in_ptr(c, in, nf, 1), Lv.g, fine, c->stream);
      launch_restrict(Lv.g, Nx.g, Nx.kind, fine, coarse, c->stream);
      double* od = out_ptr(c, out, ncn, 2, false, &staged);
      launch_relayout(Nx.g, coarse, gdc, od, c->stream);
      L(c, 3);
      check_launch();
      if (staged) copy_back(c, out, od, ncn);
    } else {  // out (level) = m_f P in (level + 1): the correction added to a zero vector
      launch_relayout(gdc, in_ptr(c, in, ncn, 1), Nx.g, coarse, c->stream);
      CK(cudaMemsetAsync(fine, 0, (size_t)Lv.g.N * sizeof(double), c->stream));
      launch_prolong_add(Lv.g, Nx.g, Nx.kind, coarse, fine, c->stream);
      double* od = out_ptr(c, out, nf, 2, false, &staged);
      launch_relayout(Lv.g, fine, gdf, od, c->stream);
      L(c, 3);
      check_launch();
      if (staged) copy_back(c, out, od, nf);
    }
    if (!staged) CK(cudaStreamSynchronize(c->stream));
    return ST_OK;
  });
}

int st_vcycle(st_ctx_t* c, const double* rho, const double* b, double* z, int transpose) {
  return guarded([&]() -> int {
    if (!c) throw StErr{ST_E_INVALID_ARG, "null ctx"};
    CK(cudaSetDevice(c->device));
    prepare(c, rho);
    pack_in(c, b, pool(c, 1), 1);
    launch_mask_free(c->lv[0].g, pool(c, 1), pool(c, 1), c->stream);  // the solver's vectors vanish there
    L(c);
    vcycle(c, 0, transpose != 0, pool(c, 1), pool(c, 0), false, pool(c, 2));
    unpack_out(c, pool(c, 0), z, 2);
    return ST_OK;
  });
}

// ---- config-5 design update (R-13) --------------------------------------------------
namespace {
struct DesignShape {
  long long nsp;    // elements per layer (spatial field)
  int nloc;         // owned layers (time-constant: 1)
  int out_layers;   // layers of the filtered field st_solve takes (owned + ghost)
  long long nglob;  // elements over all ranks
  bool tv;
};
DesignShape design_shape(const st_ctx* c) {
  DesignShape d{};
  d.nsp = 1;
  for (int k = 0; k < c->sd; ++k) d.nsp *= c->grid.n;
  const Level& L0 = c->lv[0];
  d.tv = !c->tc;
  d.nloc = d.tv ? (L0.dist ? L0.nloc : L0.g.nt) : 1;
  d.out_layers = d.tv ? L0.g.nt : 1;
  d.nglob = d.tv ? d.nsp * c->grid.nt : d.nsp;
  return d;
}
void ensure_design_bufs(st_ctx* c, const DesignShape& d) {
  if (!c->fbuf) {
    dzalloc(&c->fbuf, (size_t)d.nsp * (d.nloc + 2));
    dzalloc(&c->fw, (size_t)d.nsp * d.nloc);
  }
}
}  // namespace

int st_filter(st_ctx_t* c, const double* in, double* out, int transpose, double radius) {
  return guarded([&]() -> int {
    if (!c || !in || !out) throw StErr{ST_E_INVALID_ARG, "null argument"};
    if (!(radius > 0)) throw StErr{ST_E_INVALID_ARG, "radius must be > 0"};
    CK(cudaSetDevice(c->device));
    const DesignShape d = design_shape(c);
    ensure_design_bufs(c, d);
    const bool slab = d.tv && c->lv[0].dist;
    const int lo_ok = slab && c->comm.rank > 0, hi_ok = slab && c->comm.rank < c->comm.size - 1;
    const int tdir = d.tv ? 1 : 0;
    const long long nown = d.nsp * d.nloc;
    const double* src = in_ptr(c, in, nown, 1);
    if (transpose) launch_filter_w(c->sd, (int)c->grid.n, d.nloc, tdir, lo_ok, hi_ok, radius, c->fw, c->stream);
    launch_filter_pack(nown, src, transpose ? c->fw : nullptr, c->fbuf + d.nsp, c->stream);
    L(c, transpose ? 2 : 1);
    if (slab)
      comm_call([&] {
        comm_halo(c->comm, c->fbuf + d.nsp, c->fbuf, c->fbuf + (long long)d.nloc * d.nsp,
                  c->fbuf + (long long)(d.nloc + 1) * d.nsp, d.nsp, c->stream);
      });
    const long long nout = transpose ? nown : d.nsp * d.out_layers;
    bool staged = false;
    double* dst = out_ptr(c, out, nout, 3, false, &staged);
    launch_filter(c->sd, (int)c->grid.n, d.nloc, tdir, lo_ok, hi_ok, radius, c->fbuf, dst, transpose ? 1 : 0,
                  c->stream);
    L(c);
    check_launch();
    if (!transpose && slab)  // the solver's ghost layer: the next slab's first filtered layer (all ranks take part)
      comm_call([&] { comm_shift_down(c->comm, dst, dst + (long long)d.nloc * d.nsp, d.nsp, c->stream); });
    if (staged) copy_back(c, out, dst, nout);
    else CK(cudaStreamSynchronize(c->stream));
    return ST_OK;
  });
}

int st_oc_update(st_ctx_t* c, const double* rho, const double* dJ, double volfrac, double move, double rho_min,
                 double* rho_new, double* lambda_out) {
  return guarded([&]() -> int {
    if (!c || !rho || !dJ || !rho_new) throw StErr{ST_E_INVALID_ARG, "null argument"};
    if (!(volfrac > 0 && volfrac <= 1) || !(move > 0) || !(rho_min >= 0 && rho_min < 1))
      throw StErr{ST_E_INVALID_ARG, "volfrac / move / rho_min"};
    CK(cudaSetDevice(c->device));
    const DesignShape d = design_shape(c);
    const long long nown = d.nsp * d.nloc;
    const double* r = in_ptr(c, rho, nown, 1);
    const double* g = in_ptr(c, dJ, nown, 2);
    const bool slab = d.tv && c->lv[0].dist;
    double* dsum = c->dsmall + 480;
    // bisection on Lambda (the oracle runs the same loop, oracle/design.py)
    double l1 = 0.0, l2 = 1e9;
    for (int it = 0; it < 200 && (l2 - l1) / (l1 + l2) > 1e-12; ++it) {
      const double lm = 0.5 * (l1 + l2);
      launch_oc_sum(r, g, nown, lm, move, rho_min, c->ws.partial, c->ws.counter, dsum, c->stream);
      L(c);
      if (slab) allreduce(c, dsum, 1);
      sync_small(c, 480, 1);
      if (c->hsmall[480] / (double)d.nglob > volfrac) l1 = lm;
      else l2 = lm;
    }
    const double lam = 0.5 * (l1 + l2);
    bool staged = false;
    double* dst = out_ptr(c, rho_new, nown, 3, false, &staged);
    launch_oc_apply(r, g, nown, lam, move, rho_min, dst, c->stream);
    L(c);
    check_launch();
    if (staged) copy_back(c, rho_new, dst, nown);
    else CK(cudaStreamSynchronize(c->stream));
    if (lambda_out) *lambda_out = lam;
    return ST_OK;
  });
}

int st_pnorm(st_ctx_t* c, const double* T, double P, double* phi, double* dphidT) {
  return guarded([&]() -> int {
    if (!c || !T || !phi) throw StErr{ST_E_INVALID_ARG, "null argument"};
    if (!(P >= 1.0)) throw StErr{ST_E_INVALID_ARG, "P must be >= 1"};
    CK(cudaSetDevice(c->device));
    double* Ti = pool(c, 0);
    pack_in(c, T, Ti, 1, true);  // with ghost planes: elements of the slab boundary planes
    const Level& L0 = c->lv[0];
    const int nl = L0.dist ? L0.nloc : L0.g.nt;
    launch_pnorm_sum(L0.g, nl, Ti, P, c->ws.partial, c->ws.counter, c->dsmall + 486, c->stream);
    L(c);
    allreduce(c, c->dsmall + 486, 1);
    sync_small(c, 486, 1);
    const double theta = c->hsmall[486];
    *phi = std::pow(theta, 1.0 / P);
    if (dphidT) {
      const double scale = std::pow(theta, (1.0 - P) / P) / (double)(1 << (c->sd + 1));
      launch_pnorm_grad(L0.g, c->o0, c->nown, L0.ntg, Ti, P, scale, pool(c, 1), c->stream);
      L(c);
      check_launch();
      unpack_out(c, pool(c, 1), dphidT, 2);
    } else {
      CK(cudaStreamSynchronize(c->stream));
    }
    return ST_OK;
  });
}

int st_dot(st_ctx_t* c, const double* x, const double* y, double* out) {
  return guarded([&]() -> int {
    if (!c || !x || !y || !out) throw StErr{ST_E_INVALID_ARG, "null argument"};
    CK(cudaSetDevice(c->device));
    const double* xd = in_ptr(c, x, c->Nd, 1);
    const double* yd = in_ptr(c, y, c->Nd, 2);
    launch_mdot(xd, yd, 0, 1, c->Nd, c->dsmall + 484, c->ws, c->stream);  // x . y and ||x||^2
    L(c);
    allreduce(c, c->dsmall + 484, 1);
    sync_small(c, 484, 1);
    *out = c->hsmall[484];
    return ST_OK;
  });
}

int st_rhs(st_ctx_t* c, const double* rho, double* f, double* b) {
  return guarded([&]() -> int {
    if (!c) throw StErr{ST_E_INVALID_ARG, "null ctx"};
    CK(cudaSetDevice(c->device));
    prepare(c, rho);
    if (f) {
      make_source(c, pool(c, 2));
      unpack_out(c, pool(c, 2), f, 2);
    }
    if (b) {
      make_forward_rhs(c, pool(c, 2));
      unpack_out(c, pool(c, 2), b, 2);
    }
    CK(cudaStreamSynchronize(c->stream));
    return ST_OK;
  });
}

int st_bench_op(st_ctx_t* c, const double* rho, int level, int mode, int transpose, int reps) {
  return guarded([&]() -> int {
    if (!c) throw StErr{ST_E_INVALID_ARG, "null ctx"};
    if (level < 0 || level >= (int)c->lv.size() || c->lv[level].dense) throw StErr{ST_E_INVALID_ARG, "level"};
    if (mode < 0 || mode > 3 || reps < 0) throw StErr{ST_E_INVALID_ARG, "mode/reps"};
    CK(cudaSetDevice(c->device));
    if (level == 0) {
      if (!is_device_ptr(rho)) throw StErr{ST_E_INVALID_ARG, "rho must be a device pointer"};
      if (c->lv[0].op.rho != rho || (c->kt && !c->lv[0].op.kt)) {  // st.h: same pointer = same rho
        set_fine_rho(c, rho);
        c->kt_design = false;
      }
    } else if (!c->have_ops || c->lv[0].op.rho != rho) {  // as level 0: same pointer = same design (st.h)
      prepare(c, rho);
    }
    Level& Lv = c->lv[level];
    double* x = level == 0 ? pool(c, 0) : Lv.x;
    double* b = level == 0 ? pool(c, 1) : Lv.b;
    for (int r = 0; r < reps; ++r) op_launch(c, level, mode, transpose != 0, true, x, b, Lv.t);
    check_launch();
    return ST_OK;
  });
}

int st_timestep(st_ctx_t* c, const double* rho, int32_t nsteps, double* T, st_ts_stats_t* stats) {
  return guarded([&]() -> int {
    if (!c || !rho || !T) throw StErr{ST_E_INVALID_ARG, "null argument"};
    if (nsteps < 1) throw StErr{ST_E_INVALID_ARG, "nsteps must be >= 1"};
    if (!c->tc) throw StErr{ST_E_UNSUPPORTED, "time stepping: time-constant designs only"};
    if (c->comm.size > 1) throw StErr{ST_E_UNSUPPORTED, "time stepping: one GPU"};
    if (c->src.kind == ST_SRC_EX2) throw StErr{ST_E_UNSUPPORTED, "time stepping: spatially uniform sources"};
    CK(cudaSetDevice(c->device));
    const double* r = rho_device(c, rho);
    const long long Pd = c->gd0.P;
    const long long nout = Pd * (nsteps + 1);
    double* Td = T;
    double* tmp = nullptr;
    const bool host = !is_device_ptr(T);
    if (host) {
      dalloc(&tmp, (size_t)nout);
      Td = tmp;
    }
    st_ts_stats_t st{};
    double ms = 0.0;
    long long nl = 0;
    int worst = 0;
    try {
      st.cg_iterations = st_run_timestepping(c->lv[0].g, c->md, c->src, c->grid.tau, c->bcs.T0, r, nsteps, c->opt.rtol,
                                             c->opt.maxit, (int)c->opt.coarse_max_nodes, c->gd0, Td, c->stream, &ms, &nl,
                                             &worst);
    } catch (const std::exception& e) {
      cudaFree(tmp);
      throw StErr{ST_E_CUDA, e.what()};
    }
    if (host) {
      CK(cudaMemcpyAsync(T, tmp, (size_t)nout * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      cudaFree(tmp);
    }
    st.steps = nsteps;
    st.ms = ms;
    st.launches = nl;
    st.max_step_iterations = worst;
    L(c, nl);
    if (stats) *stats = st;
    return ST_OK;
  });
}

// ---- PDE filter + Heaviside projection (csrc/pdefilter.cu) ------------------------
namespace {
// six work vectors of >= Nd doubles: Krylov-pool slots (re-zeroed by pf_release), else allocations
struct PfWork {
  double* v[6] = {};
  std::vector<double*> owned;
  bool pooled = false;
};
PfWork pf_acquire(st_ctx* c) {
  PfWork w;
  const int slots = c->opt.restart + 1 + c->nz;
  if (slots >= 6) {
    for (int k = 0; k < 6; ++k) w.v[k] = pool(c, k);
    w.pooled = true;
  } else {
    for (int k = 0; k < 6; ++k) {
      dalloc(&w.v[k], (size_t)c->Nd);
      w.owned.push_back(w.v[k]);
    }
  }
  return w;
}
void pf_release(st_ctx* c, PfWork& w) {
  if (w.pooled)  // the solver relies on zero pad entries in its pool vectors
    for (int k = 0; k < 6; ++k) CK(cudaMemsetAsync(w.v[k], 0, (size_t)c->N * sizeof(double), c->stream));
  CK(cudaStreamSynchronize(c->stream));
  for (double* p : w.owned) cudaFree(p);
}
void pf_check(st_ctx* c, double rx, double rt, double beta, double eta) {
  if (c->tc) throw StErr{ST_E_UNSUPPORTED, "PDE filter: space-time designs (a time-constant design is extruded)"};
  if (c->comm.size > 1) throw StErr{ST_E_UNSUPPORTED, "PDE filter: one GPU"};
  if (!(rx >= 0) || !(rt >= 0) || !(beta > 0) || !(eta > 0 && eta < 1))
    throw StErr{ST_E_INVALID_ARG, "PDE filter: rx, rt >= 0, beta > 0, 0 < eta < 1"};
}
}  // namespace

int st_pde_filter(st_ctx_t* c, const double* gamma, double rx, double rt, double beta, double eta, double* gamma_e,
                  double* gamma_bar) {
  return guarded([&]() -> int {
    if (!c || !gamma || !gamma_bar) throw StErr{ST_E_INVALID_ARG, "null argument"};
    pf_check(c, rx, rt, beta, eta);
    CK(cudaSetDevice(c->device));
    const long long ne = c->ndesign;
    const double* g = in_ptr(c, gamma, ne, 1);
    bool s1 = false, s2 = false;
    double* gb = out_ptr(c, gamma_bar, ne, 2, false, &s1);
    double* ge = gamma_e ? out_ptr(c, gamma_e, ne, 3, false, &s2) : nullptr;
    PfWork w = pf_acquire(c);
    const int its = st_run_pde_filter(c->sd, (int)c->grid.n, (int)c->grid.nt, rx, rt, beta, eta, g, ge, gb, w.v,
                                      c->dsmall + 400, c->hsmall + 400, c->ws, c->stream);
    L(c, 6 * its + 8);
    check_launch();
    pf_release(c, w);
    if (s1) copy_back(c, gamma_bar, gb, ne);
    if (s2) copy_back(c, gamma_e, ge, ne);
    c->stats.iterations = its;
    return ST_OK;
  });
}

int st_pde_filter_grad(st_ctx_t* c, const double* gamma_e, const double* dphi_dgbar, double rx, double rt, double beta,
                       double eta, double* dphi_dgamma) {
  return guarded([&]() -> int {
    if (!c || !gamma_e || !dphi_dgbar || !dphi_dgamma) throw StErr{ST_E_INVALID_ARG, "null argument"};
    pf_check(c, rx, rt, beta, eta);
    CK(cudaSetDevice(c->device));
    const long long ne = c->ndesign;
    const double* ge = in_ptr(c, gamma_e, ne, 1);
    const double* dp = in_ptr(c, dphi_dgbar, ne, 2);
    bool s1 = false;
    double* out = out_ptr(c, dphi_dgamma, ne, 3, false, &s1);
    PfWork w = pf_acquire(c);
    const int its = st_run_pde_filter_grad(c->sd, (int)c->grid.n, (int)c->grid.nt, rx, rt, beta, eta, ge, dp, out,
                                           w.v, c->dsmall + 400, c->hsmall + 400, c->ws, c->stream);
    L(c, 6 * its + 8);
    check_launch();
    pf_release(c, w);
    if (s1) copy_back(c, dphi_dgamma, out, ne);
    c->stats.iterations = its;
    return ST_OK;
  });
}

int st_get_stats(const st_ctx_t* c, st_stats_t* s) {
  if (!c || !s) return ST_E_INVALID_ARG;
  *s = c->stats;
  return ST_OK;
}

int st_get_hierarchy(const st_ctx_t* c, st_hierarchy_t* h) {
  if (!c || !h) return ST_E_INVALID_ARG;
  memset(h, 0, sizeof(*h));
  h->n_levels = (int)std::min<size_t>(c->lv.size(), 32);
  for (int l = 0; l < h->n_levels; ++l) {
    const Level& Lv = c->lv[l];
    h->n[l] = Lv.g.n;
    h->nt[l] = Lv.ntg;  // global extent (a rank holds a slab of distributed levels)
    h->kind[l] = Lv.kind;
    h->form[l] = Lv.dense ? FORM_DENSE : Lv.op.form;
    long long v = Lv.ntg + 1;
    for (int d = 0; d < Lv.g.sd; ++d) v *= Lv.g.nn;
    h->nodes[l] = v;
    h->omega[l] = Lv.omega;
    h->lam_max[l] = Lv.lam_max;
  }
  return ST_OK;
}

int st_local_layout(const st_ctx_t* c, st_layout_t* o) {
  if (!c || !o) return ST_E_INVALID_ARG;
  memset(o, 0, sizeof(*o));
  const Level& L0 = c->lv[0];
  o->rank = c->comm.rank;
  o->size = c->comm.size;
  o->plane0 = L0.g.pg0 + c->o0;
  o->n_planes = c->nown;
  o->layer0 = L0.g.pg0;
  o->n_layers = L0.dist ? L0.nloc : L0.g.nt;
  o->rho_layers = c->tc ? 0 : L0.g.nt;
  o->nodes_local = c->Nd;
  o->design_local = c->ndesign;
  o->n_levels = (int)c->lv.size();
  o->n_dist_levels = c->n_dist;
  return ST_OK;
}

int st_plan(const st_grid_t* grid, const st_materials_t* mats, const st_bcs_t* bcs, const st_options_t* opts,
            int32_t rank, int32_t size, st_plan_t* plan) {
  return guarded([&]() -> int {
    if (!grid || !mats || !bcs || !plan) throw StErr{ST_E_INVALID_ARG, "null argument"};
    if (grid->sdim != 2 && grid->sdim != 3) throw StErr{ST_E_INVALID_ARG, "sdim must be 2 or 3"};
    if (grid->n < 2 || grid->nt < 2) throw StErr{ST_E_INVALID_ARG, "n and nt must be >= 2"};
    if (size < 1 || rank < 0 || rank >= size) throw StErr{ST_E_INVALID_ARG, "rank / size"};
    if (grid->nt % size != 0) throw StErr{ST_E_DIVISIBILITY, "time slabs: nt must be divisible by the rank count"};
    st_ctx c;  // host-only: no device call below
    c.grid = *grid;
    c.mats = *mats;
    c.bcs = *bcs;
    if (opts) c.opt = *opts;
    else st_default_options(&c.opt);
    if (c.opt.coarse_max_nodes < 8) c.opt.coarse_max_nodes = 8;
    if (c.opt.agg_nodes <= 0) c.opt.agg_nodes = 262144;
    c.sd = grid->sdim;
    c.comm.rank = rank;
    c.comm.size = size;
    build_hierarchy(&c);
    assign_slabs(&c);
    memset(plan, 0, sizeof(*plan));
    plan->n_levels = (int)std::min<size_t>(c.lv.size(), 32);
    plan->n_dist_levels = c.n_dist;
    for (int l = 0; l < plan->n_levels; ++l) {
      const Level& Lv = c.lv[l];
      plan->n[l] = Lv.g.n;
      plan->nt[l] = Lv.ntg;
      plan->kind[l] = Lv.kind;
      plan->dist[l] = Lv.dist ? 1 : 0;
      plan->layer0[l] = Lv.dist ? Lv.a : 0;
      plan->n_layers[l] = Lv.dist ? Lv.nloc : Lv.ntg;
      plan->local_layers[l] = Lv.g.nt;
    }
    const Level& L0 = c.lv[0];
    const int o0 = (L0.dist && rank > 0) ? 1 : 0;
    plan->plane0 = L0.g.pg0 + o0;
    plan->n_planes = L0.dist ? L0.nloc + (rank == 0 ? 1 : 0) : L0.g.nt + 1;
    c.lv.clear();
    return ST_OK;
  });
}

int st_struct_sizes(int64_t out[11]) {
  if (!out) return ST_E_INVALID_ARG;
  out[0] = sizeof(st_grid_t); out[1] = sizeof(st_materials_t); out[2] = sizeof(st_bcs_t);
  out[3] = sizeof(st_source_t); out[4] = sizeof(st_options_t); out[5] = sizeof(st_dist_t);
  out[6] = sizeof(st_stats_t); out[7] = sizeof(st_hierarchy_t); out[8] = sizeof(st_layout_t);
  out[9] = sizeof(st_plan_t);
  out[10] = sizeof(st_ts_stats_t);
  return ST_OK;
}

int st_nccl_unique_id(char id[ST_NCCL_ID_BYTES]) {
  if (!id) return ST_E_INVALID_ARG;
  if (nccl_unique_id(id) != 0) {
    g_last_error = "libnccl.so.2 not available or ncclGetUniqueId failed";
    return ST_E_NCCL;
  }
  return ST_OK;
}

int st_nccl_comm_init(const char id[ST_NCCL_ID_BYTES], int32_t rank, int32_t size, void** comm) {
  if (!id || !comm || size < 1 || rank < 0 || rank >= size) return ST_E_INVALID_ARG;
  if (nccl_comm_init(id, rank, size, comm) != 0) {
    g_last_error = "ncclCommInitRank failed";
    return ST_E_NCCL;
  }
  return ST_OK;
}

int st_nccl_comm_destroy(void* comm) { return nccl_comm_destroy(comm) == 0 ? ST_OK : ST_E_NCCL; }

int st_nccl_selftest(void* comm, int32_t rank, int32_t size, int32_t* nranks) {
  return guarded([&]() -> int {
    if (!comm || size < 1 || rank < 0 || rank >= size) throw StErr{ST_E_INVALID_ARG, "comm / rank / size"};
    int cnt = -1, r = -1;
    if (nccl_comm_count(comm, &cnt, &r) != 0) throw StErr{ST_E_NCCL, "ncclCommCount / ncclCommUserRank failed"};
    if (nranks) *nranks = cnt;
    if (cnt != size || r != rank)
      throw StErr{ST_E_NCCL, "communicator has " + std::to_string(cnt) + " ranks (this is rank " + std::to_string(r) +
                                 "), expected " + std::to_string(size) + " / " + std::to_string(rank)};
    cudaStream_t s = nullptr;
    CK(cudaStreamCreate(&s));
    const std::string err = nccl_selftest(comm, rank, size, s);
    cudaStreamDestroy(s);
    if (!err.empty()) throw StErr{ST_E_NCCL, "NCCL self-test: " + err};
    return ST_OK;
  });
}

int64_t st_num_nodes(const st_ctx_t* c) { return c ? c->Nd : -1; }
int64_t st_num_design(const st_ctx_t* c) { return c ? c->ndesign : -1; }
int64_t st_kernel_launches(const st_ctx_t* c) { return c ? c->launches : -1; }

}  // extern "C"
