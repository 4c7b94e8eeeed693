// pdefilter.cu — the paper's PDE filter and Heaviside projection of the space-time design
// (sec. 2.4.2), with the chain rule of the sensitivities.
//
//   filter      (K_f + M_f) g~ = T_f g on the Q1 space-time mesh of the state, natural boundaries,
//               d = diag(r_x^2/12 (spatial), r_t^2/12 (time)); element value of the
//               filtered field = mean of its nodes (R-25);
//   projection  g_bar = (tanh(b e) + tanh(b (g~ - e))) / (tanh(b e) + tanh(b (1 - e)));
//   chain rule  dphi/dg = T_f^T (K_f + M_f)^-1 A^T (dg_bar/dg~ .* dphi/dg_bar).
//
// B200 design: K_f + M_f on the regular mesh is a sum of Kronecker products of assembled 1D tridiagonal
// factors (mass m = h/6 [1 4 1], stiffness k = 1/h [-1 2 -1], one-sided at the ends), so the operator is
// applied matrix-free with the 27 / 81 weights of a node evaluated from its position (no stored matrix,
// 16 B per node and apply). With r ~ 2.4 h the preconditioned system has an h-independent condition
// number, so conjugate gradients with Jacobi preconditioning converge in a fixed ~20-40 iterations at any
// size: no multigrid is needed for the default radii. Vectors (dense caller node layout) live in the
// context's Krylov pool between solves; the slots are re-zeroed afterwards (their pad entries must stay
// zero for the solver). One GPU (time slabs: ST_E_UNSUPPORTED).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace st {
namespace pf {

constexpr int BLK = 256;

struct FGeom {
  int sd, n, nn, nt;
  long long P, N;   // nodes per plane (dense), nodes
  long long NE;     // elements
  double dx, dt, ax, at;  // ax = r_x^2 / 12, at = r_t^2 / 12
};

// assembled 1D factors at node i (0..n) of a line of n elements, step h, for neighbour offset o
__device__ __forceinline__ double m1(int i, int n, int o, double h) {
  if (o == 0) return (h / 3.0) * ((i > 0) + (i < n));
  const int j = i + o;
  return (j >= 0 && j <= n) ? h / 6.0 : 0.0;
}
__device__ __forceinline__ double k1(int i, int n, int o, double h) {
  if (o == 0) return (1.0 / h) * ((i > 0) + (i < n));
  const int j = i + o;
  return (j >= 0 && j <= n) ? -1.0 / h : 0.0;
}

template <int SD>
__device__ __forceinline__ void coords(const FGeom& g, long long idx, int* c) {  // c[0..SD-1] space, c[SD] time
  long long r = idx;
  for (int d = 0; d < SD; ++d) {
    c[d] = (int)(r % g.nn);
    r /= g.nn;
  }
  c[SD] = (int)r;
}

// weight of (node c, offset o[0..SD]) in K_f + M_f
template <int SD>
__device__ __forceinline__ double fweight(const FGeom& g, const int* c, const int* o) {
  double ms = 1.0;
  double mk[SD];
  for (int d = 0; d < SD; ++d) {
    mk[d] = m1(c[d], g.n, o[d], g.dx);
    ms *= mk[d];
  }
  const double mt = m1(c[SD], g.nt, o[SD], g.dt), kt = k1(c[SD], g.nt, o[SD], g.dt);
  double ks = 0.0;  // sum_d k_d prod_{d' != d} m_d'
  for (int d = 0; d < SD; ++d) {
    double t = k1(c[d], g.n, o[d], g.dx);
    for (int e = 0; e < SD; ++e)
      if (e != d) t *= mk[e];
    ks += t;
  }
  return mt * ms + g.ax * mt * ks + g.at * kt * ms;
}

// MODE 0: y = F x; MODE 1: y = b - F x and z = D^-1 y (Jacobi-preconditioned residual)
template <int SD, int MODE>
__global__ void __launch_bounds__(BLK) apply_kernel(FGeom g, const double* __restrict__ x, const double* __restrict__ b,
                                                    double* __restrict__ y, double* __restrict__ z) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= g.N) return;
  int c[SD + 1];
  coords<SD>(g, idx, c);
  constexpr int NO = SD == 2 ? 27 : 81;
  double acc = 0.0, diag = 0.0;
  for (int k = 0; k < NO; ++k) {
    int o[SD + 1];
    int r = k;
    bool ok = true;
    long long nb = 0, mul = 1;
    for (int d = 0; d <= SD; ++d) {
      o[d] = (r % 3) - 1;
      r /= 3;
      const int v = c[d] + o[d];
      ok = ok && v >= 0 && v <= (d < SD ? g.n : g.nt);
      nb += (long long)v * mul;
      mul *= (d < SD ? g.nn : 1);
    }
    if (!ok) continue;
    const double w = fweight<SD>(g, c, o);
    acc += w * __ldg(x + nb);
    if (k == NO / 2) diag = w;
  }
  if (MODE == 0) {
    y[idx] = acc;
  } else {
    const double rr = __ldg(b + idx) - acc;
    y[idx] = rr;
    z[idx] = rr / diag;
  }
}

template <int SD>
__global__ void diag_kernel(FGeom g, const double* __restrict__ r, double* __restrict__ z) {  // z = D^-1 r
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= g.N) return;
  int c[SD + 1], o[SD + 1] = {};
  coords<SD>(g, idx, c);
  z[idx] = r[idx] / fweight<SD>(g, c, o);
}

// node value = s * sum over the node's elements of v_e (T_f: s = |e| / 2^(d+1); A^T: s = 1 / 2^(d+1))
template <int SD>
__global__ void e2n_kernel(FGeom g, const double* __restrict__ v, double s, double* __restrict__ out) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= g.N) return;
  int c[SD + 1];
  coords<SD>(g, idx, c);
  double acc = 0.0;
  for (int e = 0; e < (1 << (SD + 1)); ++e) {
    long long ei = 0, mul = 1;
    bool ok = true;
    for (int d = 0; d <= SD; ++d) {
      const int a = c[d] - ((e >> d) & 1);
      ok = ok && a >= 0 && a < (d < SD ? g.n : g.nt);
      ei += (long long)a * mul;
      mul *= g.n;
    }
    if (ok) acc += __ldg(v + ei);
  }
  out[idx] = s * acc;
}

// element value = s * sum of its nodal values (A: s = 1 / 2^(d+1); T_f^T: s = |e| / 2^(d+1)); with
// PROJ the mean is also projected: ge = mean, gb = projection(ge)
template <int SD, bool PROJ>
__global__ void n2e_kernel(FGeom g, const double* __restrict__ u, double s, double* __restrict__ out,
                           double* __restrict__ gb, double beta, double eta) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= g.NE) return;
  int c[SD + 1];
  long long r = e;
  for (int d = 0; d < SD; ++d) {
    c[d] = (int)(r % g.n);
    r /= g.n;
  }
  c[SD] = (int)r;
  double acc = 0.0;
  for (int a = 0; a < (1 << (SD + 1)); ++a) {
    long long ni = 0, mul = 1;
    for (int d = 0; d <= SD; ++d) {
      ni += (long long)(c[d] + ((a >> d) & 1)) * mul;
      mul *= g.nn;
    }
    acc += __ldg(u + ni);
  }
  const double v = s * acc;
  if (out) out[e] = v;
  if (PROJ) {
    const double den = tanh(beta * eta) + tanh(beta * (1.0 - eta));
    gb[e] = (tanh(beta * eta) + tanh(beta * (v - eta))) / den;
  }
}

// w_e = dg_bar/dg~ (ge) * dphi/dg_bar
__global__ void dproj_kernel(long long n, const double* __restrict__ ge, const double* __restrict__ dphi, double beta,
                             double eta, double* __restrict__ w) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double den = tanh(beta * eta) + tanh(beta * (1.0 - eta));
  const double th = tanh(beta * (__ldg(ge + i) - eta));
  w[i] = beta * (1.0 - th * th) / den * __ldg(dphi + i);
}

// p = z + beta p, with beta = s[0] / s[1] (rz_new / rz_old)
__global__ void p_kernel(long long n, const double* __restrict__ z, double* __restrict__ p, const double* rz_new,
                         const double* rz_old, int first) {
  const double b = first ? 0.0 : rz_new[0] / rz_old[0];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = z[i] + b * p[i];
}
// x += a p, r -= a q, z = D^-1 r handled by the caller (diag_kernel); a = rz / pq
__global__ void xr_kernel(long long n, double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                          const double* __restrict__ q, const double* rz, const double* pq) {
  const double a = rz[0] / pq[0];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    x[i] += a * p[i];
    r[i] -= a * q[i];
  }
}

unsigned nb(long long n) { return (unsigned)((n + BLK - 1) / BLK); }
unsigned ew(long long n) { return (unsigned)std::min<long long>((n + BLK - 1) / BLK, 148LL * 16); }

}  // namespace pf

// Solve (K_f + M_f) x = b by Jacobi-preconditioned CG to rtol (relative residual), x = 0 start.
// Work vectors: r, z, p, q (N each). dd: >= 16 device doubles; hh: >= 16 pinned host doubles.
// Returns the iterations.
static int pf_cg(const pf::FGeom& g, const double* b, double* x, double* r, double* z, double* p, double* q,
                 double rtol, int maxit, double* dd, double* hh, RedWs ws, cudaStream_t s) {
  using namespace pf;
  const long long N = g.N;
  cudaMemsetAsync(x, 0, N * sizeof(double), s);
  cudaMemcpyAsync(r, b, N * sizeof(double), cudaMemcpyDeviceToDevice, s);
  if (g.sd == 2) diag_kernel<2><<<nb(N), BLK, 0, s>>>(g, r, z);
  else diag_kernel<3><<<nb(N), BLK, 0, s>>>(g, r, z);
  launch_mdot(r, nullptr, 0, 0, N, dd + 4, ws, s);  // ||b||^2
  launch_mdot(r, z, 0, 1, N, dd, ws, s);            // dd[0] = r.z
  cudaMemcpyAsync(hh, dd, 8 * sizeof(double), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  const double bn = std::sqrt(hh[4]);
  if (bn == 0.0) return 0;
  int it = 0;
  for (; it < maxit; ++it) {
    // p = z + (rz / rz_old) p ; q = F p ; pq ; x += a p, r -= a q ; z = D^-1 r ; rz_new, ||r||^2
    p_kernel<<<ew(N), BLK, 0, s>>>(N, z, p, dd, dd + 8, it == 0);
    cudaMemcpyAsync(dd + 8, dd, sizeof(double), cudaMemcpyDeviceToDevice, s);  // rz_old = rz
    if (g.sd == 2) apply_kernel<2, 0><<<nb(N), BLK, 0, s>>>(g, p, nullptr, q, nullptr);
    else apply_kernel<3, 0><<<nb(N), BLK, 0, s>>>(g, p, nullptr, q, nullptr);
    launch_mdot(p, q, 0, 1, N, dd + 2, ws, s);      // dd[2] = p.q
    xr_kernel<<<ew(N), BLK, 0, s>>>(N, x, r, p, q, dd + 8, dd + 2);
    if (g.sd == 2) diag_kernel<2><<<nb(N), BLK, 0, s>>>(g, r, z);
    else diag_kernel<3><<<nb(N), BLK, 0, s>>>(g, r, z);
    launch_mdot(r, z, 0, 1, N, dd, ws, s);          // dd[0] = r.z, dd[1] = ||r||^2
    cudaMemcpyAsync(hh, dd, 2 * sizeof(double), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if (!(std::sqrt(std::max(hh[1], 0.0)) > rtol * bn)) return it + 1;
  }
  return it;
}

}  // namespace st

using namespace st;

// entry points used by api.cu (st_pde_filter / st_pde_filter_grad). Dense node / element layouts.
// vec: 6 work vectors of >= N doubles; dd / hh scratch; returns CG iterations (or -1 on bad args).
int st_run_pde_filter(int sd, int n, int nt, double rx, double rt, double beta, double eta, const double* gamma,
                      double* ge, double* gb, double* const* vec, double* dd, double* hh, RedWs ws, cudaStream_t s) {
  using namespace pf;
  FGeom g{};
  g.sd = sd; g.n = n; g.nn = n + 1; g.nt = nt;
  g.P = 1;
  for (int d = 0; d < sd; ++d) g.P *= g.nn;
  g.N = g.P * (nt + 1);
  g.NE = 1;
  for (int d = 0; d < sd; ++d) g.NE *= n;
  g.NE *= nt;
  g.dx = 1.0 / n; g.dt = 1.0 / nt; g.ax = rx * rx / 12.0; g.at = rt * rt / 12.0;
  const double vol = std::pow(g.dx, sd) * g.dt, w = 1.0 / (1 << (sd + 1));
  double* b = vec[0];
  double* x = vec[1];
  if (sd == 2) e2n_kernel<2><<<nb(g.N), BLK, 0, s>>>(g, gamma, vol * w, b);   // T_f g
  else e2n_kernel<3><<<nb(g.N), BLK, 0, s>>>(g, gamma, vol * w, b);
  const int its = pf_cg(g, b, x, vec[2], vec[3], vec[4], vec[5], 1e-12, 500, dd, hh, ws, s);
  if (sd == 2) n2e_kernel<2, true><<<nb(g.NE), BLK, 0, s>>>(g, x, w, ge, gb, beta, eta);  // mean, projection
  else n2e_kernel<3, true><<<nb(g.NE), BLK, 0, s>>>(g, x, w, ge, gb, beta, eta);
  return its;
}

int st_run_pde_filter_grad(int sd, int n, int nt, double rx, double rt, double beta, double eta, const double* ge,
                           const double* dphi, double* out, double* const* vec, double* dd, double* hh, RedWs ws,
                           cudaStream_t s) {
  using namespace pf;
  FGeom g{};
  g.sd = sd; g.n = n; g.nn = n + 1; g.nt = nt;
  g.P = 1;
  for (int d = 0; d < sd; ++d) g.P *= g.nn;
  g.N = g.P * (nt + 1);
  g.NE = 1;
  for (int d = 0; d < sd; ++d) g.NE *= n;
  g.NE *= nt;
  g.dx = 1.0 / n; g.dt = 1.0 / nt; g.ax = rx * rx / 12.0; g.at = rt * rt / 12.0;
  const double vol = std::pow(g.dx, sd) * g.dt, w = 1.0 / (1 << (sd + 1));
  double* we = out;  // element scratch: w_e = dg_bar/dg~ dphi/dg_bar (overwritten by the result)
  dproj_kernel<<<nb(g.NE), BLK, 0, s>>>(g.NE, ge, dphi, beta, eta, we);
  double* b = vec[0];
  double* x = vec[1];
  if (sd == 2) e2n_kernel<2><<<nb(g.N), BLK, 0, s>>>(g, we, w, b);   // A^T w
  else e2n_kernel<3><<<nb(g.N), BLK, 0, s>>>(g, we, w, b);
  const int its = pf_cg(g, b, x, vec[2], vec[3], vec[4], vec[5], 1e-12, 500, dd, hh, ws, s);
  if (sd == 2) n2e_kernel<2, false><<<nb(g.NE), BLK, 0, s>>>(g, x, vol * w, out, nullptr, beta, eta);  // T_f^T
  else n2e_kernel<3, false><<<nb(g.NE), BLK, 0, s>>>(g, x, vol * w, out, nullptr, beta, eta);
  return its;
}
