// design.cu — the design-update kernels of BASELINE config 5 (R-13):
// the density filter and the optimality-criteria (OC) update. These are driver-level steps of a
// topology-optimisation loop, not the paper's method (the paper uses a PDE filter, projection and
// MMA); they sit beside the hot path so that config 5 runs entirely on the GPU.
//
// Density filter (R-13): on the element grid (x1, x2[, x3], t), rho~_i = sum_j w_ij rho_j / W_i with
// hat weights w_ij = max(0, r - |idx_i - idx_j|), r = 2 (the 3^(d+1) neighbourhood: 2, 1, 2 - sqrt2,
// 2 - sqrt3 [, 0]), W_i = sum_j w_ij over the elements that exist. Transpose (chain rule):
// (F^T g)_j = sum_i w_ij g_i / W_i. A time-constant design is filtered in space only.
// OC (R-13): rho_new = clip(rho sqrt(max(0, -dJ) / Lambda), [max(lo, rho - move), min(1, rho + move)])
// with Lambda from bisection so that the mean of rho_new is the volume fraction.
#include "common.cuh"
#include "kernels.h"

namespace st {

__device__ __forceinline__ double hat_w(int d0, int d1, int d2, double r) {
  const double d = sqrt((double)(d0 * d0 + d1 * d1 + d2 * d2));
  return fmax(0.0, r - d);
}

// in / out: element arrays [nl][n2][n1] (n2 = 1 for sdim = 1 slices is not used). `in` holds the
// owned layers with one ghost layer on each side (layers -1 .. nl; a missing neighbour layer is
// flagged by lo_ok / hi_ok = 0). mode 0: out_i = sum_j w_ij in_j / W_i; mode 1: out_j = sum_i w_ij in_i / W_i.
template <int SD>
__global__ void filter_kernel(int n, int nl, int tdir, int lo_ok, int hi_ok, double r, const double* __restrict__ in,
                              double* __restrict__ out, int mode) {
  long long nsp = 1;
  for (int d = 0; d < SD; ++d) nsp *= n;
  long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= nsp * nl) return;
  const int l = (int)(idx / nsp);
  long long e = idx % nsp;
  int c[3] = {0, 0, 0};
  for (int d = 0; d < SD; ++d) { c[d] = (int)(e % n); e /= n; }
  // neighbours: spatial offsets in {-1,0,1}^SD, time offset in {-1,0,1} (tdir = 1) or {0}
  auto exists = [&](const int* cc, int ll) {
    for (int d = 0; d < SD; ++d)
      if (cc[d] < 0 || cc[d] >= n) return false;
    if (ll < 0 && !lo_ok) return false;
    if (ll >= nl && !hi_ok) return false;
    return true;
  };
  double acc = 0.0, Wi = 0.0;
  for (int dt = -tdir; dt <= tdir; ++dt)
    for (int k = 0; k < (SD == 2 ? 9 : 27); ++k) {
      int o[3] = {k % 3 - 1, (k / 3) % 3 - 1, k / 9 - 1};
      if (SD == 2) o[2] = 0;
      int nb[3] = {0, 0, 0};
      for (int d = 0; d < SD; ++d) nb[d] = c[d] + o[d];
      const int ll = l + dt;
      if (!exists(nb, ll)) continue;
      // |offset| over (x1, x2[, x3], t)
      const double dist2 = (double)(o[0] * o[0] + o[1] * o[1] + (SD == 3 ? o[2] * o[2] : 0) + dt * dt);
      const double w = fmax(0.0, r - sqrt(dist2));
      if (w == 0.0) continue;
      long long j = 0, mul = 1;
      for (int d = 0; d < SD; ++d) { j += nb[d] * mul; mul *= n; }
      const double v = in[(long long)(ll + 1) * nsp + j];
      if (mode == 0) {
        acc += w * v;
        Wi += w;
      } else {
        // transpose: v is g_j / W_j already (pre-scaled by the caller pass)
        acc += w * v;
      }
    }
  out[idx] = (mode == 0) ? acc / Wi : acc;
}

// W_i of every element (owned layers) into out, for the transpose pre-scaling
template <int SD>
__global__ void filter_w_kernel(int n, int nl, int tdir, int lo_ok, int hi_ok, double r, double* __restrict__ out) {
  long long nsp = 1;
  for (int d = 0; d < SD; ++d) nsp *= n;
  long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= nsp * nl) return;
  const int l = (int)(idx / nsp);
  long long e = idx % nsp;
  int c[3] = {0, 0, 0};
  for (int d = 0; d < SD; ++d) { c[d] = (int)(e % n); e /= n; }
  double W = 0.0;
  for (int dt = -tdir; dt <= tdir; ++dt)
    for (int k = 0; k < (SD == 2 ? 9 : 27); ++k) {
      int o[3] = {k % 3 - 1, (k / 3) % 3 - 1, k / 9 - 1};
      if (SD == 2) o[2] = 0;
      bool ok = true;
      for (int d = 0; d < SD; ++d) ok = ok && c[d] + o[d] >= 0 && c[d] + o[d] < n;
      const int ll = l + dt;
      if (ll < 0 && !lo_ok) ok = false;
      if (ll >= nl && !hi_ok) ok = false;
      if (!ok) continue;
      const double dist2 = (double)(o[0] * o[0] + o[1] * o[1] + (SD == 3 ? o[2] * o[2] : 0) + dt * dt);
      W += fmax(0.0, r - sqrt(dist2));
    }
  out[idx] = W;
}

// copy owned layers into the ghosted buffer at layer offset 1 (optionally dividing by W)
__global__ void filter_pack_kernel(long long count, const double* __restrict__ src, const double* __restrict__ W,
                                   double* __restrict__ dst) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= count) return;
  dst[i] = W ? src[i] / W[i] : src[i];
}

void launch_filter(int sd, int n, int nl, int tdir, int lo_ok, int hi_ok, double r, const double* ghosted, double* out,
                   int mode, cudaStream_t s) {
  long long nsp = 1;
  for (int d = 0; d < sd; ++d) nsp *= n;
  const long long tot = nsp * nl;
  const unsigned grd = (unsigned)((tot + 255) / 256);
  if (sd == 2) filter_kernel<2><<<grd, 256, 0, s>>>(n, nl, tdir, lo_ok, hi_ok, r, ghosted, out, mode);
  else filter_kernel<3><<<grd, 256, 0, s>>>(n, nl, tdir, lo_ok, hi_ok, r, ghosted, out, mode);
}

void launch_filter_w(int sd, int n, int nl, int tdir, int lo_ok, int hi_ok, double r, double* out, cudaStream_t s) {
  long long nsp = 1;
  for (int d = 0; d < sd; ++d) nsp *= n;
  const long long tot = nsp * nl;
  const unsigned grd = (unsigned)((tot + 255) / 256);
  if (sd == 2) filter_w_kernel<2><<<grd, 256, 0, s>>>(n, nl, tdir, lo_ok, hi_ok, r, out);
  else filter_w_kernel<3><<<grd, 256, 0, s>>>(n, nl, tdir, lo_ok, hi_ok, r, out);
}

void launch_filter_pack(long long count, const double* src, const double* W, double* dst, cudaStream_t s) {
  filter_pack_kernel<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(count, src, W, dst);
}

// ---- OC ------------------------------------------------------------------------------------
__device__ __forceinline__ double oc_new(double rho, double dj, double lam, double move, double lo) {
  const double b = sqrt(fmax(0.0, -dj) / lam);
  const double v = rho * b;
  return fmin(fmin(1.0, rho + move), fmax(fmax(lo, rho - move), v));
}

// sum of rho_new(Lambda) (deterministic: per-block partials, last block sums in fixed order)
__global__ void __launch_bounds__(256) oc_sum_kernel(const double* __restrict__ rho, const double* __restrict__ dj,
                                                     long long n, double lam, double move, double lo,
                                                     double* __restrict__ partial, unsigned* counter,
                                                     double* __restrict__ out) {
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    acc += oc_new(rho[i], dj[i], lam, move, lo);
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  __shared__ double sm[8];
  __shared__ bool last;
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int w = 0; w < 8; ++w) a += sm[w];
    partial[blockIdx.x] = a;
    __threadfence();
    last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double a = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) a += ((volatile double*)partial)[b];
    *out = a;
    *counter = 0u;
  }
}

__global__ void oc_apply_kernel(const double* __restrict__ rho, const double* __restrict__ dj, long long n, double lam,
                                double move, double lo, double* __restrict__ out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] = oc_new(rho[i], dj[i], lam, move, lo);
}

void launch_oc_sum(const double* rho, const double* dj, long long n, double lam, double move, double lo,
                   double* partial, unsigned* counter, double* out, cudaStream_t s) {
  oc_sum_kernel<<<296, 256, 0, s>>>(rho, dj, n, lam, move, lo, partial, counter, out);
}

void launch_oc_apply(const double* rho, const double* dj, long long n, double lam, double move, double lo, double* out,
                     cudaStream_t s) {
  oc_apply_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(rho, dj, n, lam, move, lo, out);
}

}  // namespace st

namespace st {

// ---- p-norm objective (sec. 3.3.1; gradient PAPER.md:593-595) -------------------
// phi = (sum_e Tavg_e^P)^(1/P), Tavg_e = mean of the element's 2^(d+1) nodal temperatures.
template <int SD>
__device__ __forceinline__ double elem_avg(const Geom& g, const double* __restrict__ T, const int* e, int tau) {
  double s = 0.0;
  for (int b = 0; b < (1 << (SD + 1)); ++b) {
    int c[3] = {0, 0, 0};
    for (int d = 0; d < SD; ++d) c[d] = e[d] + ((b >> d) & 1);
    const int p = tau + ((b >> SD) & 1);
    s += __ldg(T + (long long)p * g.P + pidx<SD>(g, c));
  }
  return s / (double)(1 << (SD + 1));
}

// sum over the local element layers [0, nl) of Tavg^P (deterministic block partials)
template <int SD>
__global__ void __launch_bounds__(256) pnorm_sum_kernel(Geom g, int nl, const double* __restrict__ T, double P,
                                                        double* __restrict__ partial, unsigned* counter,
                                                        double* __restrict__ out) {
  long long nsp = 1;
  for (int d = 0; d < SD; ++d) nsp *= g.n;
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nsp * nl;
       i += (long long)gridDim.x * blockDim.x) {
    const int tau = (int)(i / nsp);
    long long r = i % nsp;
    int e[3] = {0, 0, 0};
    for (int d = 0; d < SD; ++d) { e[d] = (int)(r % g.n); r /= g.n; }
    acc += pow(elem_avg<SD>(g, T, e, tau), P);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  __shared__ double sm[8];
  __shared__ bool last;
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int w = 0; w < 8; ++w) a += sm[w];
    partial[blockIdx.x] = a;
    __threadfence();
    last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double a = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) a += ((volatile double*)partial)[b];
    *out = a;
    *counter = 0u;
  }
}

// dphi/dT_a = theta^((1-P)/P) / 2^(d+1) sum_{e adjacent to a} Tavg_e^(P-1) over the local planes
// [p0, p0 + np) (node-centric: the adjacent elements of slab-boundary planes use the ghost planes)
template <int SD>
__global__ void pnorm_grad_kernel(Geom g, int p0, int np, int ntg, const double* __restrict__ T, double P, double scale,
                                  double* __restrict__ out) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= g.P * (long long)np) return;
  const int p = p0 + (int)(idx / g.P);
  const long long pn = idx % g.P;
  int c[3] = {0, 0, 0};
  double* o = out + (long long)p * g.P + pn;
  if (!pdecode<SD>(g, pn, c)) { *o = 0.0; return; }
  double acc = 0.0;
  for (int b = 0; b < (1 << (SD + 1)); ++b) {  // element = node - bits of b
    int e[3] = {0, 0, 0};
    bool ok = true;
    for (int d = 0; d < SD; ++d) {
      e[d] = c[d] - ((b >> d) & 1);
      ok = ok && e[d] >= 0 && e[d] < g.n;
    }
    const int tau = p - ((b >> SD) & 1);
    ok = ok && tau >= 0 && tau + g.pg0 < ntg && tau < g.nt;
    if (ok) acc += pow(elem_avg<SD>(g, T, e, tau), P - 1.0);
  }
  *o = scale * acc;
}

void launch_pnorm_sum(const Geom& g, int nl, const double* T, double P, double* partial, unsigned* counter, double* out,
                      cudaStream_t s) {
  if (g.sd == 2) pnorm_sum_kernel<2><<<296, 256, 0, s>>>(g, nl, T, P, partial, counter, out);
  else pnorm_sum_kernel<3><<<296, 256, 0, s>>>(g, nl, T, P, partial, counter, out);
}

void launch_pnorm_grad(const Geom& g, int p0, int np, int ntg, const double* T, double P, double scale, double* out,
                       cudaStream_t s) {
  const long long tot = g.P * (long long)np;
  const unsigned grd = (unsigned)((tot + 255) / 256);
  if (g.sd == 2) pnorm_grad_kernel<2><<<grd, 256, 0, s>>>(g, p0, np, ntg, T, P, scale, out);
  else pnorm_grad_kernel<3><<<grd, 256, 0, s>>>(g, p0, np, ntg, T, P, scale, out);
}

}  // namespace st
