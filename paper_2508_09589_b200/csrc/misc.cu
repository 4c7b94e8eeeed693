// misc.cu — source assembly, Dirichlet helpers, element sensitivities, dense coarsest solve.
#include <algorithm>

#include "st.h"
#include "common.cuh"
#include "kernels.h"

namespace st {

// ---------------------------------------------------------------------------------------
// f_a = sum_e int N_a Q~ dV for a spatially uniform source: exact spatial
// integrals (dx/2 per adjacent element and direction) times 2-point Gauss in time per
// element layer (R-5).
// Temporal factor of a spatially uniform source (R-5: 2-point Gauss per element layer):
// kind 0 UNIFORM, 1 SIN: qscale (1 + a sin(w tau t)); 2 EX1: 1/2 qscale (1 - t)(1 + cos 50 t)
// (Example 1, t rescaled). t: global rescaled time.
__device__ __forceinline__ double q_time(int kind, double qscale, double a, double w, double tau, double t) {
  if (kind == 1) return qscale * (1.0 + a * sin(w * tau * t));
  if (kind == 2) return 0.5 * qscale * (1.0 - t) * (1.0 + cos(50.0 * t));
  return qscale;
}

// Spatially uniform sources (kinds 0-2): one CTA row per time plane (blockIdx.y); the plane's
// temporal factor (4 Gauss points) is evaluated once per CTA, then the plane's nodes are written with
// a grid-stride loop (exact spatial integrals: dx/2 per adjacent element and direction).
template <int SD>
__global__ void source_kernel(Geom g, int kind, double qscale, double a, double w, double tau, double* __restrict__ f) {
  __shared__ double ft_s;
  for (int p = blockIdx.y; p <= g.nt; p += gridDim.y) {
    if (threadIdx.x == 0) {
      const double s = 0.5 / sqrt(3.0);
      double ft = 0.0;
      for (int side = 0; side < 2; ++side) {
        const int l = side == 0 ? p - 1 : p;  // layer; the node is its top (side 0) or bottom (side 1)
        if (l < 0 || l >= g.nt) continue;
        for (int gp = 0; gp < 2; ++gp) {
          const double sg = gp == 0 ? -s : s;
          const double tt = (l + g.pg0 + 0.5 + sg) * g.dt;  // global time of the Gauss point
          const double N = side == 0 ? (0.5 + sg) : (0.5 - sg);
          ft += 0.5 * g.dt * N * q_time(kind, qscale, a, w, tau, tt);
        }
      }
      ft_s = ft;
    }
    __syncthreads();
    const double ft = ft_s;
    double* fp = f + (long long)p * g.P;
    for (long long pn = blockIdx.x * (long long)blockDim.x + threadIdx.x; pn < g.P;
         pn += (long long)gridDim.x * blockDim.x) {
      int cc[3];
      if (!pdecode<SD>(g, pn, cc)) { fp[pn] = 0.0; continue; }
      double sx = 1.0;
#pragma unroll
      for (int d = 0; d < SD; ++d) sx *= 0.5 * g.dx * ((cc[d] == 0 || cc[d] == g.n) ? 1.0 : 2.0);
      fp[pn] = sx * ft;
    }
    __syncthreads();
  }
}

// Example 2's moving Gaussian, (2+1)D: f_a = sum over the node's adjacent elements of
// the 2 x 2 x 2-point Gauss quadrature of N_a Q~ (R-5), Q~ = Q0 exp(-|x - x0(t)|^2 / (2 s^2)),
// x0(t) = (1/2 + R cos(w tau t + pi/2), 1/2 + R sin(w tau t + pi/2)) in rescaled coordinates.
__global__ void source_ex2_kernel(Geom g, double q0, double w, double tau, double sig, double R, double* __restrict__ f) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= g.N) return;
  const int p = (int)(idx / g.P);
  int cc[3];
  if (!pdecode<2>(g, idx % g.P, cc)) { f[idx] = 0.0; return; }
  const double gq = 1.0 / sqrt(3.0);
  const double det = 0.125 * g.dx * g.dx * g.dt;  // (dx/2)^2 (dt/2)
  const double inv2s2 = 1.0 / (2.0 * sig * sig);
  const double hp = 1.5707963267948966;
  double acc = 0.0;
  for (int bt = 0; bt < 2; ++bt) {
    const int l = p - bt;  // element layer; the node's local time bit is bt
    if (l < 0 || l >= g.nt) continue;
    for (int qt = 0; qt < 2; ++qt) {
      const double st = qt ? gq : -gq;
      const double t = (l + g.pg0 + 0.5 * (1.0 + st)) * g.dt;
      const double Nt = bt ? 0.5 * (1.0 + st) : 0.5 * (1.0 - st);
      const double x10 = 0.5 + R * cos(w * tau * t + hp), x20 = 0.5 + R * sin(w * tau * t + hp);
      for (int b2 = 0; b2 < 2; ++b2) {
        const int e2 = cc[1] - b2;
        if (e2 < 0 || e2 >= g.n) continue;
        for (int b1 = 0; b1 < 2; ++b1) {
          const int e1 = cc[0] - b1;
          if (e1 < 0 || e1 >= g.n) continue;
          for (int q2 = 0; q2 < 2; ++q2) {
            const double s2 = q2 ? gq : -gq;
            const double x2 = (e2 + 0.5 * (1.0 + s2)) * g.dx;
            const double N2 = b2 ? 0.5 * (1.0 + s2) : 0.5 * (1.0 - s2);
            for (int q1 = 0; q1 < 2; ++q1) {
              const double s1 = q1 ? gq : -gq;
              const double x1 = (e1 + 0.5 * (1.0 + s1)) * g.dx;
              const double N1 = b1 ? 0.5 * (1.0 + s1) : 0.5 * (1.0 - s1);
              const double r2 = (x1 - x10) * (x1 - x10) + (x2 - x20) * (x2 - x20);
              acc += det * N1 * N2 * Nt * q0 * exp(-r2 * inv2s2);
            }
          }
        }
      }
    }
  }
  f[idx] = acc;
}

__global__ void ktilde_kernel(const double* __restrict__ rho, int n, int nl, MatsDev m, double* __restrict__ kt) {
  const long long w = n + 2, per = w * w, tot = per * (nl + 1);
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(idx / per);
    const long long r = idx - t * per;
    const int pj = (int)(r / w), pi = (int)(r - pj * w);
    double v = 0.0;
    if (t < nl && pi >= 1 && pi <= n && pj >= 1 && pj <= n)
      v = m.kins + m.dk * powp(__ldg(rho + ((long long)t * n + (pj - 1)) * n + (pi - 1)), m.pk);
    kt[idx] = v;
  }
}

void launch_ktilde(const double* rho, int n, int nl, const MatsDev& m, double* kt, cudaStream_t s) {
  const long long tot = (long long)(n + 2) * (n + 2) * (nl + 1);
  const long long blocks = std::min<long long>((tot + 255) / 256, 148LL * 16);
  ktilde_kernel<<<(unsigned)blocks, 256, 0, s>>>(rho, n, nl, m, kt);
}

void launch_source(const Geom& g, const st_source_t& src, double qscale, double tau, double* f, cudaStream_t s) {
  if (src.kind == ST_SRC_EX2) {
    source_ex2_kernel<<<(unsigned)((g.N + 255) / 256), 256, 0, s>>>(g, qscale, src.w, tau, src.sigma, src.R, f);
    return;
  }
  const long long bx = std::min<long long>((g.P + 255) / 256, 64);
  const unsigned by = (unsigned)std::min<long long>(g.nt + 1, 65535);
  if (g.sd == 2) source_kernel<2><<<dim3((unsigned)bx, by), 256, 0, s>>>(g, src.kind, qscale, src.a, src.w, tau, f);
  else source_kernel<3><<<dim3((unsigned)bx, by), 256, 0, s>>>(g, src.kind, qscale, src.a, src.w, tau, f);
}

// ---------------------------------------------------------------------------------------
// node of storage index idx; false for pad entries
template <int SD> __device__ __forceinline__ bool node_of(const Geom& g, long long idx, int* c, int& p) {
  p = (int)(idx / g.P);
  return pdecode<SD>(g, idx % g.P, c);
}

template <int SD> __global__ void mask_free_kernel(Geom g, const double* __restrict__ in, double* __restrict__ out) {
  long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= g.N) return;
  int c[3] = {0, 0, 0}, p;
  if (!node_of<SD>(g, idx, c, p)) { out[idx] = 0.0; return; }
  out[idx] = is_cons<SD>(g, c, p) ? 0.0 : in[idx];
}
template <int SD> __global__ void set_bc_kernel(Geom g, double T0, double* __restrict__ x) {
  long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= g.N) return;
  int c[3] = {0, 0, 0}, p;
  if (!node_of<SD>(g, idx, c, p)) return;
  if (is_cons<SD>(g, c, p)) x[idx] = (p + g.pg0 == 0 && !is_patch<SD>(g, c)) ? T0 : 0.0;
}
template <int SD> __global__ void xd_kernel(Geom g, double T0, double* __restrict__ x) {
  long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= g.N) return;
  int c[3] = {0, 0, 0}, p;
  if (!node_of<SD>(g, idx, c, p)) { x[idx] = 0.0; return; }
  x[idx] = (p + g.pg0 == 0 && !is_patch<SD>(g, c)) ? T0 : 0.0;
}
template <int SD>
__global__ void rhs_kernel(Geom g, const double* f, const double* __restrict__ KxD, double T0,
                           double* b) {  // b may alias f (elementwise)
  long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= g.N) return;
  int c[3] = {0, 0, 0}, p;
  if (!node_of<SD>(g, idx, c, p)) { b[idx] = 0.0; return; }
  if (is_cons<SD>(g, c, p)) b[idx] = (p + g.pg0 == 0 && !is_patch<SD>(g, c)) ? T0 : 0.0;
  else b[idx] = f[idx] - (KxD ? KxD[idx] : 0.0);
}

// relayout between two storage geometries of the same grid (dense caller layout <-> padded
// internal layout); iterates over the source storage, skips its pads
template <int SD>
__global__ void relayout_kernel(Geom gs, const double* __restrict__ src, Geom gd, double* __restrict__ dst) {
  long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= gs.N) return;
  int c[3] = {0, 0, 0}, p;
  if (!node_of<SD>(gs, idx, c, p)) return;
  dst[(long long)p * gd.P + pidx<SD>(gd, c)] = src[idx];
}
// dst_c = src_c at constrained nodes (identity rows of the eliminated operator)
template <int SD> __global__ void copy_cons_kernel(Geom g, const double* __restrict__ src, double* __restrict__ dst) {
  long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= g.N) return;
  int c[3] = {0, 0, 0}, p;
  if (!node_of<SD>(g, idx, c, p)) return;
  if (is_cons<SD>(g, c, p)) dst[idx] = src[idx];
}

void launch_relayout(const Geom& gs, const double* src, const Geom& gd, double* dst, cudaStream_t s) {
  unsigned grd = (unsigned)((gs.N + 255) / 256);
  if (gs.sd == 2) relayout_kernel<2><<<grd, 256, 0, s>>>(gs, src, gd, dst);
  else relayout_kernel<3><<<grd, 256, 0, s>>>(gs, src, gd, dst);
}

#define EW_LAUNCH(K, ...)                                                   \
  do {                                                                      \
    unsigned grd = (unsigned)((g.N + 255) / 256);                           \
    if (g.sd == 2) K<2><<<grd, 256, 0, s>>>(g, __VA_ARGS__);                \
    else K<3><<<grd, 256, 0, s>>>(g, __VA_ARGS__);                          \
  } while (0)

void launch_mask_free(const Geom& g, const double* in, double* out, cudaStream_t s) { EW_LAUNCH(mask_free_kernel, in, out); }
void launch_copy_cons(const Geom& g, const double* src, double* dst, cudaStream_t s) { EW_LAUNCH(copy_cons_kernel, src, dst); }
void launch_set_bc_values(const Geom& g, double T0, double* x, cudaStream_t s) { EW_LAUNCH(set_bc_kernel, T0, x); }
void launch_xd(const Geom& g, double T0, double* x, cudaStream_t s) { EW_LAUNCH(xd_kernel, T0, x); }  // x = xD
void launch_rhs_combine(const Geom& g, const double* f, const double* KxD, double T0, double* b, cudaStream_t s) {
  EW_LAUNCH(rhs_kernel, f, KxD, T0, b);
}

// ---------------------------------------------------------------------------------------
// Element sensitivities: dJ_e = -lambda_e^T (C' U(x)M_sp + k~' Tm(x)K_sp) T_e
// with lambda = 0 on constrained nodes and full T. Time-constant rho: sum over layers
// (transposed extrusion).
// the element's nodal values of plane q: T and lambda (lambda = 0 at constrained nodes)
template <int SD>
__device__ __forceinline__ void sens_plane(const Geom& g, const double* __restrict__ T, const double* __restrict__ lam,
                                           const int* a, int q, double* Tq, double* Lq) {
#pragma unroll
  for (int b = 0; b < SG<SD>::NE; ++b) {
    int c[3] = {0, 0, 0};
#pragma unroll
    for (int d = 0; d < SD; ++d) c[d] = a[d] + ((b >> d) & 1);
    const long long i = (long long)q * g.P + pidx<SD>(g, c);
    Tq[b] = __ldg(T + i);
    Lq[b] = is_cons<SD>(g, c, q) ? 0.0 : __ldg(lam + i);
  }
}

// dJ_e of element layer tau from the bottom (b) and top (t) nodal values
template <int SD>
__device__ __forceinline__ double elem_sens(const OpDesc& op, const double* Tb, const double* Tt, const double* Lb,
                                            const double* Lt, double r) {
  constexpr int NE = SG<SD>::NE;
  const Geom& g = op.g;
  double gG = 0.0, gK1 = 0.0, gK2 = 0.0;
#pragma unroll
  for (int b = 0; b < NE; ++b) {
#pragma unroll
    for (int q = 0; q < NE; ++q) {
      int h = __popc((unsigned)(b ^ q));
      double m = mtab<SD>(h, g.dx), k = ktab<SD>(h, g.dx);
      gG += Lt[b] * m * (Tt[q] - Tb[q]);
      gK1 += Lb[b] * k * (2.0 * Tb[q] + Tt[q]);
      gK2 += Lt[b] * k * (Tb[q] + 2.0 * Tt[q]);
    }
  }
  double gK = (g.dt / 6.0) * (gK1 + gK2);
  double dC = op.m.dC * dpowp(r, op.m.pc);
  double dk = op.m.dk * dpowp(r, op.m.pk);
  return -(dC * gG + dk * gK);
}

// one thread per (spatial element, chunk of kSensChunk layers), marching in time: the top plane's nodal
// values of layer tau are the bottom plane's of layer tau + 1 (half the loads of one thread per element
// and layer); time-constant rho: one chunk of all layers, summed
constexpr int kSensChunk = 8;
template <int SD>
__global__ void sens_kernel(OpDesc op, const double* __restrict__ T, const double* __restrict__ lam,
                            double* __restrict__ dJ) {
  constexpr int NE = SG<SD>::NE;
  const Geom& g = op.g;
  long long ne_sp = 1;
  for (int d = 0; d < SD; ++d) ne_sp *= g.n;
  const int K = op.rho_tc ? g.nt : kSensChunk;
  const long long nch = (g.nt + K - 1) / K;
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= ne_sp * nch) return;
  const long long e = idx % ne_sp;
  const int t0 = (int)(idx / ne_sp) * K, t1 = min(t0 + K, g.nt);
  int a[3] = {0, 0, 0};
  long long t = e;
  for (int d = 0; d < SD; ++d) { a[d] = (int)(t % g.n); t /= g.n; }
  double Tb[NE], Lb[NE], Tt[NE], Lt[NE];
  sens_plane<SD>(g, T, lam, a, t0, Tb, Lb);
  const double rtc = op.rho_tc ? __ldg(op.rho + e) : 0.0;
  double acc = 0.0;
  for (int tau = t0; tau < t1; ++tau) {
    sens_plane<SD>(g, T, lam, a, tau + 1, Tt, Lt);
    const long long ie = (long long)tau * ne_sp + e;
    const double v = elem_sens<SD>(op, Tb, Tt, Lb, Lt, op.rho_tc ? rtc : __ldg(op.rho + ie));
    if (op.rho_tc) acc += v;
    else dJ[ie] = v;
#pragma unroll
    for (int b = 0; b < NE; ++b) {
      Tb[b] = Tt[b];
      Lb[b] = Lt[b];
    }
  }
  if (op.rho_tc) dJ[e] = acc;
}

void launch_sensitivity(const OpDesc& op, const double* T, const double* lam, double* dJ, cudaStream_t s) {
  long long ne_sp = 1;
  for (int d = 0; d < op.g.sd; ++d) ne_sp *= op.g.n;
  const long long nch = op.rho_tc ? 1 : (op.g.nt + kSensChunk - 1) / kSensChunk;
  const unsigned grd = (unsigned)((ne_sp * nch + 127) / 128);
  if (op.g.sd == 2) sens_kernel<2><<<grd, 128, 0, s>>>(op, T, lam, dJ);
  else sens_kernel<3><<<grd, 128, 0, s>>>(op, T, lam, dJ);
}

// ---------------------------------------------------------------------------------------
// Dense coarsest level: the assembled eliminated operator restricted to the FREE nodes
// (no pad entries, no constrained identity rows: those unknowns are x_c = b_c), inverted once per design
// by Gauss-Jordan with partial pivoting in one CTA, then x = A^-1 b per V-cycle.
__global__ void dense_gather_kernel(const double* __restrict__ A, long long N, const int* __restrict__ fidx, int nf,
                                    double* __restrict__ Af) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)nf * nf) return;
  const int i = (int)(e / nf), j = (int)(e % nf);
  Af[e] = A[(long long)fidx[i] * N + fidx[j]];
}

// In-place Gauss-Jordan inversion with partial pivoting, the whole matrix in shared memory (n <= 160):
// step k swaps rows k and p_k, then with piv = a_kk, r_j = a_kj / piv (r_k = 1 / piv), c_i = a_ik:
// a_kj = r_j, and for i != k: a_ik = 0, a_ij -= c_i r_j. The row swaps are undone at the end as
// column swaps in reverse order. Same result as the augmented [A | I] elimination up to rounding,
// with every access in shared memory (~1 us per pivot instead of ~11 us through L2).
// SMEM = false (n <= 4096): the same steps in place on the global matrix (L2-resident), r and c in shared
// memory.
constexpr int kDenseSmemMax = 160;
constexpr int kDenseMax = 4096;
template <bool SMEM>
__global__ void __launch_bounds__(1024) dense_invert_kernel(const double* __restrict__ A, double* __restrict__ Ainv,
                                                            int n, int* info) {
  extern __shared__ double dsm[];  // SMEM: [n][n], then r[n], c[n]; else r[n], c[n]
  double* a = SMEM ? dsm : Ainv;
  double* r = SMEM ? dsm + n * n : dsm;
  double* c = r + n;
  __shared__ int perm[kDenseMax];
  __shared__ double bv[32];
  __shared__ int bi[32];
  const int tid = threadIdx.x, nth = blockDim.x;
  if (SMEM || A != Ainv)
    for (int e = tid; e < n * n; e += nth) a[e] = A[e];
  if (tid == 0) *info = 0;
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    double best = -1.0;
    int bidx = k;
    for (int i = k + tid; i < n; i += nth) {
      const double v = fabs(a[i * n + k]);
      if (v > best) { best = v; bidx = i; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_down_sync(0xffffffffu, best, o);
      const int oi = __shfl_down_sync(0xffffffffu, bidx, o);
      if (ov > best || (ov == best && oi < bidx)) { best = ov; bidx = oi; }
    }
    if ((tid & 31) == 0) { bv[tid >> 5] = best; bi[tid >> 5] = bidx; }
    __syncthreads();
    if (tid == 0) {
      double bb = bv[0];
      int ii = bi[0];
      for (int w = 1; w < nth / 32; ++w)
        if (bv[w] > bb || (bv[w] == bb && bi[w] < ii)) { bb = bv[w]; ii = bi[w]; }
      perm[k] = ii;
      if (!(bb > 0.0) && *info == 0) *info = k + 1;
    }
    __syncthreads();
    const int p = perm[k];
    if (p != k)
      for (int j = tid; j < n; j += nth) {
        const double t = a[k * n + j];
        a[k * n + j] = a[p * n + j];
        a[p * n + j] = t;
      }
    __syncthreads();
    const double piv = a[k * n + k];
    const double ip = (piv != 0.0) ? 1.0 / piv : 0.0;
    for (int j = tid; j < n; j += nth) r[j] = (j == k) ? ip : a[k * n + j] * ip;
    for (int i = tid; i < n; i += nth) c[i] = (i == k) ? 0.0 : a[i * n + k];
    __syncthreads();
    // rows strided over the warps, columns over the lanes (no per-element integer division)
    for (int i = tid >> 5; i < n; i += nth >> 5) {
      double* ai = a + i * n;
      const double ci = c[i];
      if (i == k) {
        for (int j = tid & 31; j < n; j += 32) ai[j] = r[j];
      } else {
        for (int j = tid & 31; j < n; j += 32) ai[j] = (j == k ? 0.0 : ai[j]) - ci * r[j];
      }
    }
    __syncthreads();
  }
  for (int k = n - 1; k >= 0; --k) {  // undo the row swaps as column swaps
    const int p = perm[k];
    if (p != k)
      for (int i = tid; i < n; i += nth) {
        const double t = a[i * n + k];
        a[i * n + k] = a[i * n + p];
        a[i * n + p] = t;
      }
    __syncthreads();
  }
  if (SMEM)
    for (int e = tid; e < n * n; e += nth) Ainv[e] = a[e];
}

// A: the assembled N x N operator; fidx: the nf free stored indices; Ainv: nf x nf inverse (out)
void launch_dense_invert(const double* A, long long N, const int* fidx, int nf, double* Ainv, int* info,
                         cudaStream_t s) {
  dense_gather_kernel<<<(unsigned)(((long long)nf * nf + 255) / 256), 256, 0, s>>>(A, N, fidx, nf, Ainv);
  if (nf <= kDenseSmemMax) {
    const size_t bytes = (size_t)(nf * nf + 2 * nf) * sizeof(double);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(dense_invert_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)((kDenseSmemMax * kDenseSmemMax + 2 * kDenseSmemMax) * sizeof(double)));
      attr = true;
    }
    dense_invert_kernel<true><<<1, 1024, bytes, s>>>(Ainv, Ainv, nf, info);
    return;
  }
  // in place through L2 (nf <= 4096: r, c 64 KB of dynamic shared memory)
  static bool attr2 = false;
  if (!attr2) {
    cudaFuncSetAttribute(dense_invert_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(2 * kDenseMax * sizeof(double)));
    attr2 = true;
  }
  dense_invert_kernel<false><<<1, 1024, 2 * nf * sizeof(double), s>>>(Ainv, Ainv, nf, info);
}

// x = A^-1 b on the free nodes (fpos[e] = free position of stored entry e, or -1), x_e = b_e elsewhere
// (constrained identity rows; pad entries, zero in both). One warp per stored entry.
__global__ void dense_solve_kernel(const double* __restrict__ Ainv, int nf, const int* __restrict__ fidx,
                                   const int* __restrict__ fpos, long long N, int trans, const double* __restrict__ b,
                                   double* __restrict__ x) {
  pdl_wait();
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= N) return;
  const int i = fpos[warp];
  if (i < 0) {
    if (lane == 0) x[warp] = b[warp];
    return;
  }
  double acc = 0.0;
  if (!trans)
    for (int j = lane; j < nf; j += 32) acc += Ainv[(long long)i * nf + j] * b[fidx[j]];
  else
    for (int j = lane; j < nf; j += 32) acc += Ainv[(long long)j * nf + i] * b[fidx[j]];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if (lane == 0) x[warp] = acc;
}

void launch_dense_solve(const double* Ainv, int nf, const int* fidx, const int* fpos, long long N, bool trans,
                        const double* b, double* x, cudaStream_t s) {
  const int thr = 256;
  const unsigned grd = (unsigned)((N * 32 + thr - 1) / thr);
  launch_pdl(dense_solve_kernel, dim3(grd), dim3(thr), 0, s, Ainv, nf, fidx, fpos, N, trans ? 1 : 0, b, x);
}

}  // namespace st
