// timestep.cu — the GPU time-stepping baseline (sec. 4): the
// comparison method of the paper's space-time speed-up claims, on the same spatial
// Q1 mesh, design, materials, source and Dirichlet data as the space-time context.
//
// First-order backward difference in time:
//     (M_C / dt + K_k) T^{m+1} = (M_C / dt) T^m + F(t_{m+1}),   T^0 = T0 (0 on the sink),
// M_C, K_k the spatial Q1 capacity mass and conductivity stiffness of the time-constant design
// (C_e, k~_e per spatial element), F(t) = Q~(t) int N_a dx for the spatially uniform sources
// (UNIFORM, SIN, EX1; R-5), the sink / wall nodes held at 0 by symmetric elimination (R-1).
// Every step is solved to the same relative residual as the space-time solve by preconditioned CG
// (the eliminated matrix is SPD) with a spatial geometric-multigrid V-cycle: full spatial coarsening
// (as the paper's time-stepping runs), Galerkin coarse operators A_c = P^T A P with
// the bilinear / trilinear P of the space-time hierarchy, damped Jacobi 2 + 2, dense coarsest solve.
// All level operators are stored as full 9 / 27-point rows ([NOFF][P], coalesced per offset); the
// fine level of config 2 is 257^2 nodes, so a step is latency-bound: the whole PCG iteration is ONE
// CUDA graph launch (device-side alpha / beta; the host reads ||r||^2 once per iteration).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "st.h"
#include "common.cuh"
#include "kernels.h"

namespace st {
namespace ts {

constexpr int BLK = 256;

// row of the level-0 operator at node c, offset k: sum over the elements holding both nodes of
// C_e / dt M_e + k~_e K_e (Hamming-distance tables mtab / ktab, common.cuh)
template <int SD>
__global__ void assemble0_kernel(Geom g, const double* __restrict__ rho, MatsDev m, double idt, double* __restrict__ A) {
  constexpr int NOFF = SG<SD>::NOFF;
  const long long pn = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (pn >= g.P) return;
  int c[3] = {0, 0, 0};
  const bool node = pdecode<SD>(g, pn, c);
  const bool cons = node && is_patch<SD>(g, c);
  for (int k = 0; k < NOFF; ++k) {
    double w = 0.0;
    if (node && !cons) {
      int nb[3] = {0, 0, 0};
      bool ok = true;
      int h = 0;
      for (int d = 0; d < SD; ++d) {
        const int o = SG<SD>::od(k, d);
        nb[d] = c[d] + o;
        ok = ok && nb[d] >= 0 && nb[d] < g.nn;
        h += o != 0;
      }
      if (ok && !is_patch<SD>(g, nb)) {
        const double mh = mtab<SD>(h, g.dx), kh = ktab<SD>(h, g.dx);
        // element origins: per direction {c-1, c} when o = 0, else min(c, nb)
        int lo[3], cnt[3];
        for (int d = 0; d < SD; ++d) {
          const int o = SG<SD>::od(k, d);
          lo[d] = o == 0 ? c[d] - 1 : min(c[d], nb[d]);
          cnt[d] = o == 0 ? 2 : 1;
        }
        for (int e = 0; e < (1 << SD); ++e) {
          long long ei = 0, mul = 1;
          bool ve = true;
          for (int d = 0; d < SD; ++d) {
            const int bit = (e >> d) & 1;
            const int a = lo[d] + bit;
            ve = ve && bit < cnt[d] && a >= 0 && a < g.n;
            ei += (long long)a * mul;
            mul *= g.n;
          }
          if (!ve) continue;
          const double r = __ldg(rho + ei);
          const double Ce = m.Cins + m.dC * powp(r, m.pc);
          const double ke = m.kins + m.dk * powp(r, m.pk);
          w += Ce * idt * mh + ke * kh;
        }
      }
    } else if (node && k == SG<SD>::CEN) {
      w = 1.0;  // constrained row: identity (symmetric elimination, R-1)
    }
    A[(long long)k * g.P + pn] = w;
  }
}

// Galerkin A_c = P^T A P (P: bilinear / trilinear, rows of constrained fine nodes zero; constrained
// coarse nodes get identity rows). One thread per coarse node and offset.
template <int SD>
__global__ void rap_kernel(Geom gf, Geom gc, const double* __restrict__ Af, double* __restrict__ Ac) {
  constexpr int NOFF = SG<SD>::NOFF;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= gc.P * NOFF) return;
  const int K = (int)(t / gc.P);
  const long long pc = t % gc.P;
  int C[3] = {0, 0, 0};
  double out = 0.0;
  if (pdecode<SD>(gc, pc, C)) {
    if (is_patch<SD>(gc, C)) {
      out = K == SG<SD>::CEN ? 1.0 : 0.0;
    } else {
      int Cn[3] = {0, 0, 0};
      bool okc = true;
      for (int d = 0; d < SD; ++d) {
        Cn[d] = C[d] + SG<SD>::od(K, d);
        okc = okc && Cn[d] >= 0 && Cn[d] < gc.nn;
      }
      if (okc && !is_patch<SD>(gc, Cn)) {
        // fine nodes i with P(i, C) != 0: 2C + {-1, 0, 1} per direction
        for (int ki = 0; ki < NOFF; ++ki) {
          int fi[3] = {0, 0, 0};
          bool ok = true;
          double wi = 1.0;
          for (int d = 0; d < SD; ++d) {
            const int o = SG<SD>::od(ki, d);
            fi[d] = 2 * C[d] + o;
            ok = ok && fi[d] >= 0 && fi[d] < gf.nn;
            wi *= o == 0 ? 1.0 : 0.5;
          }
          if (!ok || is_patch<SD>(gf, fi)) continue;
          const long long pi = pidx<SD>(gf, fi);
          for (int kj = 0; kj < NOFF; ++kj) {
            const double a = __ldg(Af + (long long)kj * gf.P + pi);
            if (a == 0.0) continue;
            // P(j, Cn): fine j = fi + od(kj); weight prod over directions of (1 - |j - 2 Cn| / 2)
            double wj = 1.0;
            bool okj = true;
            for (int d = 0; d < SD; ++d) {
              const int j = fi[d] + SG<SD>::od(kj, d);
              const int dd = j - 2 * Cn[d];
              okj = okj && j >= 0 && j < gf.nn && dd >= -1 && dd <= 1;
              wj *= dd == 0 ? 1.0 : 0.5;
            }
            if (!okj) continue;
            int fj[3] = {0, 0, 0};
            for (int d = 0; d < SD; ++d) fj[d] = fi[d] + SG<SD>::od(kj, d);
            if (is_patch<SD>(gf, fj)) continue;
            out += wi * a * wj;
          }
        }
      }
    }
  }
  Ac[(long long)K * gc.P + pc] = out;
}

// y = A x (MODE_APPLY), b - A x (RESID), x + w D^-1 (b - A x) (JAC), w D^-1 b (JAC0)
template <int SD, int MODE>
__global__ void __launch_bounds__(BLK) op_kernel(Geom g, const double* __restrict__ A, const double* __restrict__ x,
                                                 const double* __restrict__ b, double* __restrict__ y, double omega) {
  constexpr int NOFF = SG<SD>::NOFF;
  const long long pn = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (pn >= g.P) return;
  int c[3] = {0, 0, 0};
  if (!pdecode<SD>(g, pn, c)) return;
  const double d = __ldg(A + (long long)SG<SD>::CEN * g.P + pn);
  double ax = 0.0;
  if (MODE != MODE_JAC0) {
    for (int k = 0; k < NOFF; ++k) {
      int nb[3] = {0, 0, 0};
      bool ok = true;
      for (int dd = 0; dd < SD; ++dd) {
        nb[dd] = c[dd] + SG<SD>::od(k, dd);
        ok = ok && nb[dd] >= 0 && nb[dd] < g.nn;
      }
      if (ok) ax += __ldg(A + (long long)k * g.P + pn) * __ldg(x + pidx<SD>(g, nb));
    }
  }
  double o;
  if (MODE == MODE_APPLY) o = ax;
  else if (MODE == MODE_RESID) o = __ldg(b + pn) - ax;
  else if (MODE == MODE_JAC) o = __ldg(x + pn) + omega * (__ldg(b + pn) - ax) / d;
  else o = omega * __ldg(b + pn) / d;
  y[pn] = o;
}

// max over rows of sum_j |A_ij| / |A_ii| (Gershgorin bound on |lambda|max(D^-1 A)), as positive bits
template <int SD>
__global__ void gersh_kernel(Geom g, const double* __restrict__ A, unsigned long long* out) {
  constexpr int NOFF = SG<SD>::NOFF;
  const long long pn = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double r = 0.0;
  int c[3] = {0, 0, 0};
  if (pn < g.P && pdecode<SD>(g, pn, c) && !is_patch<SD>(g, c)) {
    double s = 0.0;
    for (int k = 0; k < NOFF; ++k) s += fabs(__ldg(A + (long long)k * g.P + pn));
    r = s / fabs(__ldg(A + (long long)SG<SD>::CEN * g.P + pn));
  }
  for (int o = 16; o > 0; o >>= 1) r = fmax(r, __shfl_down_sync(0xffffffffu, r, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(r));
}

template <int SD>
__global__ void dense_kernel(Geom g, const double* __restrict__ A, double* __restrict__ D) {
  constexpr int NOFF = SG<SD>::NOFF;
  const long long pn = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (pn >= g.P) return;
  double* row = D + pn * g.P;
  int c[3] = {0, 0, 0};
  if (!pdecode<SD>(g, pn, c)) { row[pn] = 1.0; return; }  // pad: identity
  for (int k = 0; k < NOFF; ++k) {
    int nb[3] = {0, 0, 0};
    bool ok = true;
    for (int d = 0; d < SD; ++d) {
      nb[d] = c[d] + SG<SD>::od(k, d);
      ok = ok && nb[d] >= 0 && nb[d] < g.nn;
    }
    if (ok) row[pidx<SD>(g, nb)] += __ldg(A + (long long)k * g.P + pn);
  }
}

// F(t) = q~(t) int N_a dx (exact: (dx/2)^d per adjacent element), 0 at constrained nodes; plus
// rhs = (M_C / dt) T^m + F: y = b-part; the mass part comes from Mdt (stored rows of M_C / dt)
template <int SD>
__global__ void load_kernel(Geom g, double* __restrict__ L) {
  const long long pn = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (pn >= g.P) return;
  int c[3] = {0, 0, 0};
  double v = 0.0;
  if (pdecode<SD>(g, pn, c) && !is_patch<SD>(g, c)) {
    v = 1.0;
    for (int d = 0; d < SD; ++d) v *= 0.5 * g.dx * ((c[d] == 0 || c[d] == g.n) ? 1.0 : 2.0);
  }
  L[pn] = v;
}
template <int SD>
__global__ void mass_kernel(Geom g, const double* __restrict__ rho, MatsDev m, double idt, double* __restrict__ Mr) {
  // rows of M_C / dt (constrained rows and columns zero): the explicit part of the backward difference
  constexpr int NOFF = SG<SD>::NOFF;
  const long long pn = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (pn >= g.P) return;
  int c[3] = {0, 0, 0};
  const bool node = pdecode<SD>(g, pn, c);
  const bool cons = node && is_patch<SD>(g, c);
  for (int k = 0; k < NOFF; ++k) {
    double w = 0.0;
    if (node && !cons) {
      int nb[3] = {0, 0, 0};
      bool ok = true;
      int h = 0;
      for (int d = 0; d < SD; ++d) {
        const int o = SG<SD>::od(k, d);
        nb[d] = c[d] + o;
        ok = ok && nb[d] >= 0 && nb[d] < g.nn;
        h += o != 0;
      }
      if (ok) {
        int lo[3], cnt[3];
        for (int d = 0; d < SD; ++d) {
          const int o = SG<SD>::od(k, d);
          lo[d] = o == 0 ? c[d] - 1 : min(c[d], nb[d]);
          cnt[d] = o == 0 ? 2 : 1;
        }
        for (int e = 0; e < (1 << SD); ++e) {
          long long ei = 0, mul = 1;
          bool ve = true;
          for (int d = 0; d < SD; ++d) {
            const int bit = (e >> d) & 1;
            const int a = lo[d] + bit;
            ve = ve && bit < cnt[d] && a >= 0 && a < g.n;
            ei += (long long)a * mul;
            mul *= g.n;
          }
          if (!ve) continue;
          const double r = __ldg(rho + ei);
          w += (m.Cins + m.dC * powp(r, m.pc)) * idt * mtab<SD>(h, g.dx);
        }
      }
    }
    Mr[(long long)k * g.P + pn] = w;
  }
}
// rhs = Mr T^m + q L (constrained rows 0; the patch columns of Mr are multiplied by T^m = 0 there)
template <int SD>
__global__ void rhs_kernel(Geom g, const double* __restrict__ Mr, const double* __restrict__ Tm, const double* __restrict__ L,
                           const double* __restrict__ q, double* __restrict__ r) {
  constexpr int NOFF = SG<SD>::NOFF;
  const long long pn = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (pn >= g.P) return;
  int c[3] = {0, 0, 0};
  if (!pdecode<SD>(g, pn, c)) { r[pn] = 0.0; return; }
  double s = 0.0;
  for (int k = 0; k < NOFF; ++k) {
    int nb[3] = {0, 0, 0};
    bool ok = true;
    for (int d = 0; d < SD; ++d) {
      nb[d] = c[d] + SG<SD>::od(k, d);
      ok = ok && nb[d] >= 0 && nb[d] < g.nn;
    }
    if (ok) s += __ldg(Mr + (long long)k * g.P + pn) * __ldg(Tm + pidx<SD>(g, nb));
  }
  r[pn] = s + q[0] * __ldg(L + pn);
}

// device-side CG scalars: s[0] = rho_old, s[1] = rho_new, s[2] = p.q, s[3] = alpha, s[4] = beta
__global__ void cg_beta_kernel(double* s, const double* rz) {
  s[1] = rz[0];
  s[4] = s[0] != 0.0 ? s[1] / s[0] : 0.0;
}
__global__ void cg_alpha_kernel(double* s, const double* pq) {
  s[2] = pq[0];
  s[3] = s[2] != 0.0 ? s[1] / s[2] : 0.0;
  s[0] = s[1];
}
// p = z + beta p
__global__ void cg_p_kernel(long long n, const double* __restrict__ z, double* __restrict__ p, const double* s) {
  const double beta = s[4];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
}
// x += alpha p, r -= alpha q
__global__ void cg_xr_kernel(long long n, double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                             const double* __restrict__ q, const double* s) {
  const double a = s[3];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    x[i] += a * p[i];
    r[i] -= a * q[i];
  }
}
template <int SD>
__global__ void init_kernel(Geom g, double T0, double* __restrict__ x) {  // T^0: T0, 0 on the sink / pads
  const long long pn = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (pn >= g.P) return;
  int c[3] = {0, 0, 0};
  x[pn] = (pdecode<SD>(g, pn, c) && !is_patch<SD>(g, c)) ? T0 : 0.0;
}
__global__ void q_kernel(int kind, double qscale, double a, double w, double tau, double t, double* q) {
  double v = qscale;
  if (kind == 1) v = qscale * (1.0 + a * sin(w * tau * t));
  else if (kind == 2) v = 0.5 * qscale * (1.0 - t) * (1.0 + cos(50.0 * t));
  q[0] = v;
}

unsigned nb(long long n) { return (unsigned)std::max<long long>(1, (n + BLK - 1) / BLK); }

}  // namespace ts

// ------------------------------------------------------------------------------------------------
// host orchestration
struct TsLevel {
  Geom g{};
  double *A = nullptr, *x = nullptr, *b = nullptr, *r = nullptr, *t = nullptr;
  double omega = 0.8;
  double *D = nullptr, *Dinv = nullptr;
  int* info = nullptr;
  int *fidx = nullptr, *fpos = nullptr;  // dense coarsest: every stored entry is an unknown (identity maps)
};

struct TsRun {
  std::vector<TsLevel> lv;
  cudaStream_t s;
  int sd;
  double *Mr = nullptr, *L = nullptr, *xk = nullptr, *rk = nullptr, *zk = nullptr, *pk = nullptr, *qk = nullptr;
  double *sc = nullptr, *dots = nullptr;
  RedWs ws{};
  cudaGraphExec_t gx = nullptr;
  std::vector<void*> allocs;
  long long launches = 0;
  ~TsRun() {
    if (gx) cudaGraphExecDestroy(gx);
    for (void* p : allocs) cudaFree(p);
  }
  double* alloc(long long n) {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<long long>(n, 1) * sizeof(double)) != cudaSuccess)
      throw std::runtime_error("time stepping: cudaMalloc failed");
    cudaMemsetAsync(p, 0, std::max<long long>(n, 1) * sizeof(double), s);
    allocs.push_back(p);
    return (double*)p;
  }
};

static void ts_op(TsRun& R, const TsLevel& Lv, int mode, const double* x, const double* b, double* y, double omega) {
  const Geom& g = Lv.g;
  const unsigned grd = ts::nb(g.P);
#define TSOP(SD)                                                                                             \
  switch (mode) {                                                                                            \
    case MODE_APPLY: ts::op_kernel<SD, MODE_APPLY><<<grd, ts::BLK, 0, R.s>>>(g, Lv.A, x, b, y, omega); break; \
    case MODE_RESID: ts::op_kernel<SD, MODE_RESID><<<grd, ts::BLK, 0, R.s>>>(g, Lv.A, x, b, y, omega); break; \
    case MODE_JAC: ts::op_kernel<SD, MODE_JAC><<<grd, ts::BLK, 0, R.s>>>(g, Lv.A, x, b, y, omega); break;     \
    default: ts::op_kernel<SD, MODE_JAC0><<<grd, ts::BLK, 0, R.s>>>(g, Lv.A, x, b, y, omega); break;         \
  }
  if (R.sd == 2) { TSOP(2) } else { TSOP(3) }
#undef TSOP
  ++R.launches;
}

// V-cycle on level l: x = M b (damped Jacobi 2 + 2, Galerkin coarse levels, dense coarsest)
static void ts_vcycle(TsRun& R, int l, const double* b, double* x) {
  TsLevel& Lv = R.lv[l];
  if (Lv.Dinv) {
    launch_dense_solve(Lv.Dinv, (int)Lv.g.P, Lv.fidx, Lv.fpos, Lv.g.P, false, b, x, R.s);
    ++R.launches;
    return;
  }
  TsLevel& Nx = R.lv[l + 1];
  ts_op(R, Lv, MODE_JAC0, nullptr, b, x, Lv.omega);
  ts_op(R, Lv, MODE_JAC, x, b, Lv.t, Lv.omega);
  ts_op(R, Lv, MODE_RESID, Lv.t, b, Lv.r, 0.0);
  launch_restrict(Lv.g, Nx.g, KIND_SPACE, Lv.r, Nx.b, R.s);
  ts_vcycle(R, l + 1, Nx.b, Nx.x);
  launch_prolong_add(Lv.g, Nx.g, KIND_SPACE, Nx.x, Lv.t, R.s);
  ts_op(R, Lv, MODE_JAC, Lv.t, b, x, Lv.omega);
  ts_op(R, Lv, MODE_JAC, x, b, Lv.t, Lv.omega);
  cudaMemcpyAsync(x, Lv.t, Lv.g.P * sizeof(double), cudaMemcpyDeviceToDevice, R.s);
  R.launches += 2;
}

// one PCG iteration with device-side scalars (captured once into a CUDA graph)
static void ts_cg_iteration(TsRun& R) {
  TsLevel& L0 = R.lv[0];
  const long long P = L0.g.P;
  ts_vcycle(R, 0, R.rk, R.zk);                                          // z = M r
  launch_mdot(R.rk, R.zk, 0, 1, P, R.dots, R.ws, R.s);                  // r.z (and ||r||^2)
  ts::cg_beta_kernel<<<1, 1, 0, R.s>>>(R.sc, R.dots);
  ts::cg_p_kernel<<<ts::nb(P), ts::BLK, 0, R.s>>>(P, R.zk, R.pk, R.sc);  // p = z + beta p
  ts_op(R, L0, MODE_APPLY, R.pk, nullptr, R.qk, 0.0);                   // q = A p
  launch_mdot(R.pk, R.qk, 0, 1, P, R.dots + 2, R.ws, R.s);              // p.q
  ts::cg_alpha_kernel<<<1, 1, 0, R.s>>>(R.sc, R.dots + 2);
  ts::cg_xr_kernel<<<ts::nb(P), ts::BLK, 0, R.s>>>(P, R.xk, R.rk, R.pk, R.qk, R.sc);
  launch_mdot(R.rk, nullptr, 0, 0, P, R.dots + 4, R.ws, R.s);          // ||r||^2
  R.launches += 7;
}

}  // namespace st

using namespace st;

// Called by st_timestep (api.cu). Returns total PCG iterations; writes T (nsteps + 1 planes, dense
// caller layout on the device: gd, nn^sd per plane).
long long st_run_timestepping(const Geom& g0in, const MatsDev& md, const st_source_t& src, double tau, double T0,
                              const double* rho, int nsteps, double rtol, int maxit, int coarse_max_nodes,
                              const Geom& gdense, double* Tout, cudaStream_t s, double* ms_out, long long* launches,
                              int* max_its) {
  TsRun R;
  R.s = s;
  R.sd = g0in.sd;
  // spatial levels: one plane (nt = 0; pg0 = 1 so no plane is the initial-condition plane)
  auto plane_geom = [&](int n) {
    Geom g = g0in;
    g.n = n;
    g.nn = n + 1;
    g.nt = 0;
    g.pr = (g.nn % 2 == 1) ? g.nn + 1 : g.nn;
    g.P = g.pr;
    for (int d = 1; d < g.sd; ++d) g.P *= g.nn;
    g.N = g.P;
    g.dx = 1.0 / n;
    g.pg0 = 1;
    return g;
  };
  {
    int n = g0in.n, plo = g0in.plo, phi = g0in.phi;
    for (;;) {
      TsLevel L;
      L.g = plane_geom(n);
      L.g.plo = plo;
      L.g.phi = phi;
      R.lv.push_back(L);
      if (L.g.P <= coarse_max_nodes || n % 2 != 0 || n < 4) break;
      n /= 2;
      plo = (plo + 1) / 2;  // coarse J with 2J in the fine patch (injection, R-23)
      phi = phi >= 0 ? phi / 2 : -1;
    }
  }
  if (R.lv.back().g.P > 4096) throw std::runtime_error("time stepping: coarsest spatial level too large for the dense solve");
  const double dt = 1.0 / nsteps;  // rescaled time step
  const double idt = 1.0 / dt;
  for (auto& L : R.lv) {
    const long long P = L.g.P;
    L.A = R.alloc((long long)SG<3>::NOFF * P);
    L.x = R.alloc(P); L.b = R.alloc(P); L.r = R.alloc(P); L.t = R.alloc(P);
  }
  const long long P0 = R.lv[0].g.P;
  R.Mr = R.alloc((long long)SG<3>::NOFF * P0);
  R.L = R.alloc(P0);
  R.xk = R.alloc(P0); R.rk = R.alloc(P0); R.zk = R.alloc(P0); R.pk = R.alloc(P0); R.qk = R.alloc(P0);
  R.sc = R.alloc(16);
  R.dots = R.alloc(16);
  R.ws.partial = R.alloc((long long)kRedBlocks * kMaxDots);
  R.ws.counter = (unsigned*)R.alloc(1);
  double* qd = R.alloc(1);
  double* gsh = R.alloc(64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  // level 0 and the explicit mass rows, Galerkin coarse levels, per-level Jacobi weights, coarsest inverse
  const TsLevel& F = R.lv[0];
  if (R.sd == 2) {
    ts::assemble0_kernel<2><<<ts::nb(P0), ts::BLK, 0, s>>>(F.g, rho, md, idt, F.A);
    ts::mass_kernel<2><<<ts::nb(P0), ts::BLK, 0, s>>>(F.g, rho, md, idt, R.Mr);
    ts::load_kernel<2><<<ts::nb(P0), ts::BLK, 0, s>>>(F.g, R.L);
  } else {
    ts::assemble0_kernel<3><<<ts::nb(P0), ts::BLK, 0, s>>>(F.g, rho, md, idt, F.A);
    ts::mass_kernel<3><<<ts::nb(P0), ts::BLK, 0, s>>>(F.g, rho, md, idt, R.Mr);
    ts::load_kernel<3><<<ts::nb(P0), ts::BLK, 0, s>>>(F.g, R.L);
  }
  for (size_t l = 1; l < R.lv.size(); ++l) {
    const Geom& gf = R.lv[l - 1].g;
    const Geom& gc = R.lv[l].g;
    const long long tot = gc.P * (R.sd == 2 ? 9 : 27);
    if (R.sd == 2) ts::rap_kernel<2><<<ts::nb(tot), ts::BLK, 0, s>>>(gf, gc, R.lv[l - 1].A, R.lv[l].A);
    else ts::rap_kernel<3><<<ts::nb(tot), ts::BLK, 0, s>>>(gf, gc, R.lv[l - 1].A, R.lv[l].A);
  }
  cudaMemsetAsync(gsh, 0, 64 * sizeof(double), s);
  for (size_t l = 0; l + 1 < R.lv.size(); ++l) {
    unsigned long long* o = reinterpret_cast<unsigned long long*>(gsh + l);
    if (R.sd == 2) ts::gersh_kernel<2><<<ts::nb(R.lv[l].g.P), ts::BLK, 0, s>>>(R.lv[l].g, R.lv[l].A, o);
    else ts::gersh_kernel<3><<<ts::nb(R.lv[l].g.P), ts::BLK, 0, s>>>(R.lv[l].g, R.lv[l].A, o);
  }
  {
    TsLevel& Lc = R.lv.back();
    const long long Pc = Lc.g.P;
    Lc.D = R.alloc(Pc * Pc);
    Lc.Dinv = R.alloc(Pc * Pc);
    Lc.info = (int*)R.alloc(1);
    Lc.fidx = (int*)R.alloc((Pc + 1) / 2);
    Lc.fpos = (int*)R.alloc((Pc + 1) / 2);
    {
      std::vector<int> iota((size_t)Pc);
      for (long long e = 0; e < Pc; ++e) iota[(size_t)e] = (int)e;
      cudaMemcpyAsync(Lc.fidx, iota.data(), Pc * sizeof(int), cudaMemcpyHostToDevice, s);
      cudaMemcpyAsync(Lc.fpos, iota.data(), Pc * sizeof(int), cudaMemcpyHostToDevice, s);
      cudaStreamSynchronize(s);  // the host staging vector goes out of scope
    }
    if (R.sd == 2) ts::dense_kernel<2><<<ts::nb(Pc), ts::BLK, 0, s>>>(Lc.g, Lc.A, Lc.D);
    else ts::dense_kernel<3><<<ts::nb(Pc), ts::BLK, 0, s>>>(Lc.g, Lc.A, Lc.D);
    launch_dense_invert(Lc.D, Pc, Lc.fidx, (int)Pc, Lc.Dinv, Lc.info, s);
  }
  double hg[64];
  cudaMemcpyAsync(hg, gsh, 64 * sizeof(double), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  for (size_t l = 0; l + 1 < R.lv.size(); ++l)  // SPD: damped Jacobi converges for omega < 2 / lambda_max
    R.lv[l].omega = hg[l] > 0.0 ? std::min(0.8, 1.6 / hg[l]) : 0.8;
  // T^0 into plane 0 of the output (dense caller layout), and the iterate
  const long long Pd = gdense.P;
  if (R.sd == 2) ts::init_kernel<2><<<ts::nb(P0), ts::BLK, 0, s>>>(F.g, T0, R.xk);
  else ts::init_kernel<3><<<ts::nb(P0), ts::BLK, 0, s>>>(F.g, T0, R.xk);
  Geom gd1 = gdense;
  gd1.nt = 0;
  gd1.N = Pd;
  gd1.pg0 = 1;
  Geom gi1 = F.g;
  launch_relayout(gi1, R.xk, gd1, Tout, s);
  double* Tprev = R.alloc(P0);
  long long total_its = 0;
  int worst = 0;
  for (int m = 0; m < nsteps; ++m) {
    // rhs = (M_C / dt) T^m + q(t_{m+1}) L ; warm start x = T^m
    cudaMemcpyAsync(Tprev, R.xk, P0 * sizeof(double), cudaMemcpyDeviceToDevice, s);
    ts::q_kernel<<<1, 1, 0, s>>>(src.kind, src.kind == ST_SRC_EX1 ? src.Q0 : src.Q0 * tau, src.a, src.w, tau,
                                 (m + 1) * dt, qd);
    double* bvec = R.lv[0].b;
    if (R.sd == 2) ts::rhs_kernel<2><<<ts::nb(P0), ts::BLK, 0, s>>>(F.g, R.Mr, Tprev, R.L, qd, bvec);
    else ts::rhs_kernel<3><<<ts::nb(P0), ts::BLK, 0, s>>>(F.g, R.Mr, Tprev, R.L, qd, bvec);
    // r = b - A x, ||b||, p = 0, rho_old = 0
    ts_op(R, F, MODE_RESID, R.xk, bvec, R.rk, 0.0);
    launch_mdot(bvec, nullptr, 0, 0, P0, R.dots + 6, R.ws, s);
    launch_mdot(R.rk, nullptr, 0, 0, P0, R.dots + 4, R.ws, s);
    cudaMemsetAsync(R.pk, 0, P0 * sizeof(double), s);
    cudaMemsetAsync(R.sc, 0, 8 * sizeof(double), s);
    double h[8];
    cudaMemcpyAsync(h, R.dots + 4, 4 * sizeof(double), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    const double bn = std::sqrt(h[2]);
    double rn = std::sqrt(h[0]);
    int its = 0;
    while (rn > rtol * bn && its < maxit) {
      if (!R.gx) {  // capture one PCG iteration (fixed buffers, device-side scalars)
        cudaGraph_t graph = nullptr;
        const long long l0 = R.launches;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed);
        ts_cg_iteration(R);
        cudaStreamEndCapture(s, &graph);
        cudaGraphInstantiate(&R.gx, graph, 0);
        cudaGraphDestroy(graph);
        R.launches = l0;
      }
      cudaGraphLaunch(R.gx, s);
      R.launches += 10 + 8 * (long long)R.lv.size();
      cudaMemcpyAsync(h, R.dots + 4, sizeof(double), cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      rn = std::sqrt(std::max(h[0], 0.0));
      ++its;
      if (!std::isfinite(rn)) throw std::runtime_error("time stepping: CG breakdown");
    }
    total_its += its;
    worst = std::max(worst, its);
    Geom gdm = gd1;
    launch_relayout(gi1, R.xk, gdm, Tout + (long long)(m + 1) * Pd, s);
  }
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("time stepping: ") + cudaGetErrorString(e));
  if (ms_out) *ms_out = ms;
  if (launches) *launches = R.launches;
  if (max_its) *max_its = worst;
  return total_its;
}
