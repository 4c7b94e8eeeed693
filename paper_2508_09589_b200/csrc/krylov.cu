// krylov.cu — FGMRES building blocks (Saad 1993): fused multi-dot
// (classical Gram-Schmidt column h = V^T w together with ||w||^2), multi-AXPY with the new
// norm, the solution update x += Z y, scaling. HBM-bound; reductions are deterministic
// (fixed grid, per-block partials, last-block finalisation in fixed order).
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace st {

constexpr int kRedThreads = 256;

template <int NV>
__device__ __forceinline__ void block_partials(double (&acc)[NV], double* __restrict__ partial, RedWs ws,
                                               double* __restrict__ out) {
  __shared__ double sm[kRedThreads / 32][NV > 0 ? NV : 1];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    double a = acc[v];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
    if (lane == 0) sm[wid][v] = a;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double a = 0.0;
#pragma unroll
    for (int w = 0; w < kRedThreads / 32; ++w) a += sm[w][threadIdx.x];
    partial[(long long)blockIdx.x * NV + threadIdx.x] = a;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = atomicAdd(ws.counter, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // last block: sum partials over blocks in fixed order
  for (int v = 0; v < NV; ++v) {
    double a = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += kRedThreads) a += ((volatile double*)partial)[(long long)b * NV + v];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
    __syncthreads();
    if (lane == 0) sm[wid][0] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < kRedThreads / 32; ++w) s += sm[w][0];
      out[v] = s;
    }
  }
  if (threadIdx.x == 0) *ws.counter = 0u;
}

template <int J, bool NRM>
__global__ void __launch_bounds__(kRedThreads) mdot_kernel(const double* __restrict__ w, const double* __restrict__ V,
                                                           long long ldv, long long n, double* out, RedWs ws) {
  constexpr int NV = J + (NRM ? 1 : 0);
  double acc[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) acc[v] = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  // two elements per iteration: 2 (J + 1) independent loads in flight per thread
  for (; i + stride < n; i += 2 * stride) {
    double w0 = __ldg(w + i), w1 = __ldg(w + i + stride);
    double v0[J > 0 ? J : 1], v1[J > 0 ? J : 1];
#pragma unroll
    for (int j = 0; j < J; ++j) { v0[j] = __ldg(V + j * ldv + i); v1[j] = __ldg(V + j * ldv + i + stride); }
#pragma unroll
    for (int j = 0; j < J; ++j) acc[j] += v0[j] * w0 + v1[j] * w1;
    if (NRM) acc[NV - 1] += w0 * w0 + w1 * w1;
  }
  if (i < n) {
    double wi = __ldg(w + i);
#pragma unroll
    for (int j = 0; j < J; ++j) acc[j] += __ldg(V + j * ldv + i) * wi;
    if (NRM) acc[NV - 1] += wi * wi;
  }
  block_partials<NV>(acc, ws.partial, ws, out);
}

// 16-byte variant (every pointer 16-byte aligned, ldv even): one double2 of every vector per
// iteration, grid stride; the odd last element (n odd) is added by the last thread of the grid.
// Measured (scripts/dev/mdot_bench.cu, gpurun_out/mdot_bench.log): J = 11 at N = 17.0M 3.9 -> 6.9 TB/s,
// J = 6 5.2 -> 6.9 TB/s at the library's 888-CTA grid.
template <int J, bool NRM>
__global__ void __launch_bounds__(kRedThreads) mdot2_kernel(const double* __restrict__ w, const double* __restrict__ V,
                                                            long long ldv, long long n, double* out, RedWs ws) {
  constexpr int NV = J + (NRM ? 1 : 0);
  double acc[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) acc[v] = 0.0;
  const long long n2 = n >> 1;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const double2* w2 = reinterpret_cast<const double2*>(w);
  for (long long i = t0; i < n2; i += stride) {
    const double2 a = __ldg(w2 + i);
    double2 v[J > 0 ? J : 1];
#pragma unroll
    for (int j = 0; j < J; ++j) v[j] = __ldg(reinterpret_cast<const double2*>(V + j * ldv) + i);
#pragma unroll
    for (int j = 0; j < J; ++j) acc[j] += v[j].x * a.x + v[j].y * a.y;
    if (NRM) acc[NV - 1] += a.x * a.x + a.y * a.y;
  }
  if ((n & 1) && t0 == stride - 1) {
    const double wi = __ldg(w + n - 1);
#pragma unroll
    for (int j = 0; j < J; ++j) acc[j] += __ldg(V + j * ldv + n - 1) * wi;
    if (NRM) acc[NV - 1] += wi * wi;
  }
  block_partials<NV>(acc, ws.partial, ws, out);
}

__global__ void __launch_bounds__(kRedThreads) maxpy_norm_kernel(double* __restrict__ w, const double* __restrict__ V,
                                                                 long long ldv, int k, const double* __restrict__ h,
                                                                 const double* __restrict__ s2, long long n, double* out,
                                                                 RedWs ws) {
  __shared__ double hs[kMaxBasis];
  for (int j = threadIdx.x; j < k; j += blockDim.x) hs[j] = s2 ? h[j] * s2[j] : h[j];
  __syncthreads();
  double acc[1] = {0.0};
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + stride < n; i += 2 * stride) {
    double a0 = w[i], a1 = w[i + stride];
    int j = 0;
    for (; j + 4 <= k; j += 4) {
      double p0 = __ldg(V + (j + 0) * ldv + i), q0 = __ldg(V + (j + 0) * ldv + i + stride);
      double p1 = __ldg(V + (j + 1) * ldv + i), q1 = __ldg(V + (j + 1) * ldv + i + stride);
      double p2 = __ldg(V + (j + 2) * ldv + i), q2 = __ldg(V + (j + 2) * ldv + i + stride);
      double p3 = __ldg(V + (j + 3) * ldv + i), q3 = __ldg(V + (j + 3) * ldv + i + stride);
      a0 -= hs[j] * p0; a1 -= hs[j] * q0;
      a0 -= hs[j + 1] * p1; a1 -= hs[j + 1] * q1;
      a0 -= hs[j + 2] * p2; a1 -= hs[j + 2] * q2;
      a0 -= hs[j + 3] * p3; a1 -= hs[j + 3] * q3;
    }
    for (; j < k; ++j) { a0 -= hs[j] * __ldg(V + j * ldv + i); a1 -= hs[j] * __ldg(V + j * ldv + i + stride); }
    w[i] = a0;
    w[i + stride] = a1;
    acc[0] += a0 * a0 + a1 * a1;
  }
  if (i < n) {
    double a0 = w[i];
    for (int j = 0; j < k; ++j) a0 -= hs[j] * __ldg(V + j * ldv + i);
    w[i] = a0;
    acc[0] += a0 * a0;
  }
  block_partials<1>(acc, ws.partial, ws, out);
}

// Gram-Schmidt pass with the re-orthogonalisation coefficients of the next pass:
// w' = w - sum_j s2_j h_j V_j, then out[j] = V_j . w' (j < J) and out[J] = ||w'||^2, from the same
// V_j registers (saves the separate multi-dot pass over V and w' of the DGKS step).
template <int J>
__global__ void __launch_bounds__(kRedThreads) maxpy_dots_kernel(double* __restrict__ w, const double* __restrict__ V,
                                                                 long long ldv, const double* __restrict__ h,
                                                                 const double* __restrict__ s2, long long n,
                                                                 double* out, RedWs ws) {
  constexpr int U = J <= 8 ? 2 : 1;  // elements per iteration: (J + 1) U loads in flight
  __shared__ double hs[J];
  if (threadIdx.x < J) hs[threadIdx.x] = s2 ? h[threadIdx.x] * s2[threadIdx.x] : h[threadIdx.x];
  __syncthreads();
  double acc[J + 1];
#pragma unroll
  for (int v = 0; v <= J; ++v) acc[v] = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    double v[U][J], a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a[u] = w[i + u * stride];
#pragma unroll
      for (int j = 0; j < J; ++j) v[u][j] = __ldg(V + j * ldv + i + u * stride);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int j = 0; j < J; ++j) a[u] -= hs[j] * v[u][j];
      w[i + u * stride] = a[u];
#pragma unroll
      for (int j = 0; j < J; ++j) acc[j] += v[u][j] * a[u];
      acc[J] += a[u] * a[u];
    }
  }
  if (U == 2 && i < n) {
    double a = w[i];
    double v[J];
#pragma unroll
    for (int j = 0; j < J; ++j) v[j] = __ldg(V + j * ldv + i);
#pragma unroll
    for (int j = 0; j < J; ++j) a -= hs[j] * v[j];
    w[i] = a;
#pragma unroll
    for (int j = 0; j < J; ++j) acc[j] += v[j] * a;
    acc[J] += a * a;
  }
  block_partials<J + 1>(acc, ws.partial, ws, out);
}

template <int J>
__global__ void __launch_bounds__(kRedThreads) maxpy_dots2_kernel(double* __restrict__ w, const double* __restrict__ V,
                                                                  long long ldv, const double* __restrict__ h,
                                                                  const double* __restrict__ s2, long long n,
                                                                  double* out, RedWs ws) {
  __shared__ double hs[J];
  if (threadIdx.x < J) hs[threadIdx.x] = s2 ? h[threadIdx.x] * s2[threadIdx.x] : h[threadIdx.x];
  __syncthreads();
  double acc[J + 1];
#pragma unroll
  for (int v = 0; v <= J; ++v) acc[v] = 0.0;
  const long long n2 = n >> 1;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double2* w2 = reinterpret_cast<double2*>(w);
  for (long long i = t0; i < n2; i += stride) {
    double2 a = w2[i];
    double2 v[J];
#pragma unroll
    for (int j = 0; j < J; ++j) v[j] = __ldg(reinterpret_cast<const double2*>(V + j * ldv) + i);
#pragma unroll
    for (int j = 0; j < J; ++j) {
      a.x -= hs[j] * v[j].x;
      a.y -= hs[j] * v[j].y;
    }
    w2[i] = a;
#pragma unroll
    for (int j = 0; j < J; ++j) acc[j] += v[j].x * a.x + v[j].y * a.y;
    acc[J] += a.x * a.x + a.y * a.y;
  }
  if ((n & 1) && t0 == stride - 1) {
    double a = w[n - 1];
    double v[J];
#pragma unroll
    for (int j = 0; j < J; ++j) v[j] = __ldg(V + j * ldv + n - 1);
#pragma unroll
    for (int j = 0; j < J; ++j) a -= hs[j] * v[j];
    w[n - 1] = a;
#pragma unroll
    for (int j = 0; j < J; ++j) acc[j] += v[j] * a;
    acc[J] += a * a;
  }
  block_partials<J + 1>(acc, ws.partial, ws, out);
}

// x += sum_j y_j Z_j with 16-byte accesses (aligned pointers, even ldz)
__global__ void lincomb2_kernel(double* __restrict__ x, const double* __restrict__ Z, long long ldz, int k,
                                const double* __restrict__ y, long long n) {
  __shared__ double ys[kMaxBasis];
  for (int j = threadIdx.x; j < k; j += blockDim.x) ys[j] = y[j];
  __syncthreads();
  const long long n2 = n >> 1;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double2* x2 = reinterpret_cast<double2*>(x);
  for (long long i = t0; i < n2; i += stride) {
    double2 a = x2[i];
    int j = 0;
    for (; j + 4 <= k; j += 4) {
      double2 z[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) z[u] = __ldg(reinterpret_cast<const double2*>(Z + (j + u) * ldz) + i);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a.x += ys[j + u] * z[u].x;
        a.y += ys[j + u] * z[u].y;
      }
    }
    for (; j < k; ++j) {
      const double2 z = __ldg(reinterpret_cast<const double2*>(Z + j * ldz) + i);
      a.x += ys[j] * z.x;
      a.y += ys[j] * z.y;
    }
    x2[i] = a;
  }
  if ((n & 1) && t0 == stride - 1) {
    double a = x[n - 1];
    for (int j = 0; j < k; ++j) a += ys[j] * __ldg(Z + j * ldz + n - 1);
    x[n - 1] = a;
  }
}

__global__ void lincomb_kernel(double* __restrict__ x, const double* __restrict__ Z, long long ldz, int k,
                               const double* __restrict__ y, long long n) {
  __shared__ double ys[kMaxBasis];
  for (int j = threadIdx.x; j < k; j += blockDim.x) ys[j] = y[j];
  __syncthreads();
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    double xi = x[i];
    int j = 0;
    for (; j + 4 <= k; j += 4) {
      double z0 = __ldg(Z + (j + 0) * ldz + i), z1 = __ldg(Z + (j + 1) * ldz + i);
      double z2 = __ldg(Z + (j + 2) * ldz + i), z3 = __ldg(Z + (j + 3) * ldz + i);
      xi += ys[j] * z0 + ys[j + 1] * z1 + ys[j + 2] * z2 + ys[j + 3] * z3;
    }
    for (; j < k; ++j) xi += ys[j] * __ldg(Z + j * ldz + i);
    x[i] = xi;
  }
}

__global__ void scale_dev_kernel(const double* __restrict__ w, double* __restrict__ v, const double* nrm2, long long n) {
  const double a = nrm2[0] > 0.0 ? 1.0 / sqrt(nrm2[0]) : 0.0;  // a zero vector stays zero
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) v[i] = a * w[i];
}

__global__ void scale_kernel(const double* __restrict__ w, double* __restrict__ v, double a, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) v[i] = a * w[i];
}

// ---- GMRES(k) smoother bookkeeping on the device (one thread each; no host synchronisation) ----
// st layout (gm_layout): g[k+1] | cs[k] | sn[k] | H[k][k+1] (column j at H + j (k+1)) | y[k]
__device__ __forceinline__ void gm_layout(double* st, int k, double** g, double** cs, double** sn, double** H,
                                          double** y) {
  *g = st;
  *cs = st + (k + 1);
  *sn = *cs + k;
  *H = *sn + k;
  *y = *H + (long long)k * (k + 1);
}
__global__ void gm_init_kernel(double* st, int k, const double* nrm2) {
  double *g, *cs, *sn, *H, *y;
  gm_layout(st, k, &g, &cs, &sn, &H, &y);
  for (int i = 0; i <= k; ++i) g[i] = 0.0;
  g[0] = sqrt(fmax(nrm2[0], 0.0));
}
// column j: h_ij = V_i . w (i <= j, CGS), h_{j+1,j} = ||w'||; previous rotations, then a new one
__global__ void gm_col_kernel(double* st, int k, int j, const double* h, const double* nrm2w) {
  double *g, *cs, *sn, *H, *y;
  gm_layout(st, k, &g, &cs, &sn, &H, &y);
  double* col = H + (long long)j * (k + 1);
  for (int i = 0; i <= j; ++i) col[i] = h[i];
  col[j + 1] = sqrt(fmax(nrm2w[0], 0.0));
  for (int i = 0; i < j; ++i) {
    const double t = cs[i] * col[i] + sn[i] * col[i + 1];
    col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1];
    col[i] = t;
  }
  const double den = hypot(col[j], col[j + 1]);
  cs[j] = den > 0.0 ? col[j] / den : 1.0;
  sn[j] = den > 0.0 ? col[j + 1] / den : 0.0;
  col[j] = den;
  col[j + 1] = 0.0;
  g[j + 1] = -sn[j] * g[j];
  g[j] = cs[j] * g[j];
}
// y = R^-1 g over the first m columns (the rotated Hessenberg is upper triangular); a zero pivot
// (breakdown) gives y_i = 0
__global__ void gm_solve_kernel(double* st, int k, int mcols) {
  double *g, *cs, *sn, *H, *y;
  gm_layout(st, k, &g, &cs, &sn, &H, &y);
  for (int i = mcols - 1; i >= 0; --i) {
    double s = g[i];
    for (int m = i + 1; m < mcols; ++m) s -= H[(long long)m * (k + 1) + i] * y[m];
    const double d = H[(long long)i * (k + 1) + i];
    y[i] = d != 0.0 ? s / d : 0.0;
  }
}

// Design fingerprint (exact change detection): two independent 64-bit hashes of the
// element BIT PATTERNS, sum_i mix(bits(a_i), i) mod 2^64. Modular addition is order-free, so the
// block-level atomics give a deterministic result; a change of any single element changes each
// sum unless a 2^-64 collision occurs (no fp rounding can absorb a perturbation).
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ull;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebull;
  z ^= z >> 31;
  return z;
}
__global__ void __launch_bounds__(kRedThreads) fingerprint_kernel(const double* __restrict__ a, long long n,
                                                                  unsigned long long* out) {
  unsigned long long h0 = 0, h1 = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    const unsigned long long v = (unsigned long long)__double_as_longlong(__ldg(a + i));
    const unsigned long long k = (unsigned long long)i;
    h0 += mix64(v + k * 0x9e3779b97f4a7c15ull);
    h1 += mix64(v ^ mix64(k + 0x632be59bd9b4e019ull));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    h0 += __shfl_down_sync(0xffffffffu, h0, o);
    h1 += __shfl_down_sync(0xffffffffu, h1, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(out, h0);
    atomicAdd(out + 1, h1);
  }
}

// the 16-byte kernels apply when every vector start is 16-byte aligned (ld even)
static bool al16(const void* a, const void* b, long long ld) {
  return (((uintptr_t)a | (uintptr_t)(b ? b : a)) & 15u) == 0 && (ld & 1) == 0;
}

static unsigned red_blocks(long long n) {
  long long b = (n + 2 * kRedThreads - 1) / (2 * kRedThreads);
  if (b > kRedBlocks) b = kRedBlocks;
  if (b < 1) b = 1;
  return (unsigned)b;
}

void launch_mdot(const double* w, const double* V, long long ldv, int k, long long n, double* out, RedWs ws,
                 cudaStream_t s) {
  // k dots + ||w||^2 in chunks of <= 16 vectors; the norm rides on the last chunk
  unsigned g = red_blocks(n);
  int done = 0;
  do {
    int J = k - done;
    if (J > 16) J = 16;
    bool nrm = (done + J == k);
    const double* Vj = V + (long long)done * ldv;
    double* o = out + done;
    const bool v2 = al16(w, J > 0 ? Vj : nullptr, J > 1 ? ldv : 0);
#define MD(JJ)                                                                                 \
  case JJ:                                                                                     \
    if (v2) {                                                                                  \
      if (nrm) mdot2_kernel<JJ, true><<<g, kRedThreads, 0, s>>>(w, Vj, ldv, n, o, ws);         \
      else mdot2_kernel<JJ, false><<<g, kRedThreads, 0, s>>>(w, Vj, ldv, n, o, ws);            \
    } else {                                                                                   \
      if (nrm) mdot_kernel<JJ, true><<<g, kRedThreads, 0, s>>>(w, Vj, ldv, n, o, ws);          \
      else mdot_kernel<JJ, false><<<g, kRedThreads, 0, s>>>(w, Vj, ldv, n, o, ws);             \
    }                                                                                          \
    break;
    switch (J) {
      case 0:
        if (v2) mdot2_kernel<0, true><<<g, kRedThreads, 0, s>>>(w, Vj, ldv, n, o, ws);
        else mdot_kernel<0, true><<<g, kRedThreads, 0, s>>>(w, Vj, ldv, n, o, ws);
        break;
      MD(1) MD(2) MD(3) MD(4) MD(5) MD(6) MD(7) MD(8)
      MD(9) MD(10) MD(11) MD(12) MD(13) MD(14) MD(15) MD(16)
    }
#undef MD
    done += J;
  } while (done < k);
}

void launch_maxpy_norm(double* w, const double* V, long long ldv, int k, const double* h, const double* s2,
                       long long n, double* out, RedWs ws, cudaStream_t s) {
  maxpy_norm_kernel<<<red_blocks(n), kRedThreads, 0, s>>>(w, V, ldv, k, h, s2, n, out, ws);
}

bool launch_maxpy_dots(double* w, const double* V, long long ldv, int k, const double* h, const double* s2,
                       long long n, double* out, RedWs ws, cudaStream_t s) {
  const unsigned g = red_blocks(n);
  const bool v2 = al16(w, V, k > 1 ? ldv : 0);
#define MX(JJ)                                                                              \
  case JJ:                                                                                  \
    if (v2) maxpy_dots2_kernel<JJ><<<g, kRedThreads, 0, s>>>(w, V, ldv, h, s2, n, out, ws); \
    else maxpy_dots_kernel<JJ><<<g, kRedThreads, 0, s>>>(w, V, ldv, h, s2, n, out, ws);    \
    return true;
  switch (k) {
    MX(1) MX(2) MX(3) MX(4) MX(5) MX(6) MX(7) MX(8)
    MX(9) MX(10) MX(11) MX(12) MX(13) MX(14) MX(15) MX(16)
    default: return false;
  }
#undef MX
}

static unsigned ew_blocks(long long n) {
  long long b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  if (b < 1) b = 1;
  return (unsigned)b;
}

void launch_lincomb(double* x, const double* Z, long long ldz, int k, const double* y, long long n, cudaStream_t s) {
  if (al16(x, Z, k > 1 ? ldz : 0)) lincomb2_kernel<<<ew_blocks((n + 1) / 2), 256, 0, s>>>(x, Z, ldz, k, y, n);
  else lincomb_kernel<<<ew_blocks(n), 256, 0, s>>>(x, Z, ldz, k, y, n);
}
void launch_scale_dev(const double* w, double* v, const double* nrm2, long long n, cudaStream_t s) {
  scale_dev_kernel<<<ew_blocks(n), 256, 0, s>>>(w, v, nrm2, n);
}
void launch_scale(const double* w, double* v, double alpha, long long n, cudaStream_t s) {
  scale_kernel<<<ew_blocks(n), 256, 0, s>>>(w, v, alpha, n);
}
void launch_gm_init(double* st, int k, const double* nrm2, cudaStream_t s) { gm_init_kernel<<<1, 1, 0, s>>>(st, k, nrm2); }
void launch_gm_col(double* st, int k, int j, const double* h, const double* nrm2w, cudaStream_t s) {
  gm_col_kernel<<<1, 1, 0, s>>>(st, k, j, h, nrm2w);
}
void launch_gm_solve(double* st, int k, int mcols, cudaStream_t s) { gm_solve_kernel<<<1, 1, 0, s>>>(st, k, mcols); }
int gm_y_offset(int k) { return (k + 1) + 2 * k + k * (k + 1); }

void launch_fingerprint(const double* a, long long n, unsigned long long* out, cudaStream_t s) {
  cudaMemsetAsync(out, 0, 2 * sizeof(unsigned long long), s);
  fingerprint_kernel<<<red_blocks(n), kRedThreads, 0, s>>>(a, n, out);
}

}  // namespace st
