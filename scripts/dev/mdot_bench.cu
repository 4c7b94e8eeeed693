// Multi-dot microbenchmark (FGMRES classical Gram-Schmidt h = V^T w): the library's grid-stride
// kernel (scalar loads, 2 elements per iteration) against a contiguous-chunk kernel with 16-byte
// loads. Reports GB/s of the J + 1 vectors read; config 2 (N = 17.0M) and a config-5-sized N.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mdot_bench mdot_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int T = 256;

template <int NV>
__device__ void block_sum(double (&acc)[NV], double* partial) {
  __shared__ double sm[T / 32][NV];
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
    for (int w = 0; w < T / 32; ++w) a += sm[w][threadIdx.x];
    partial[blockIdx.x * NV + threadIdx.x] = a;
  }
}

// library form: grid stride, scalar loads, two elements per iteration
template <int J>
__global__ void __launch_bounds__(T) md_stride(const double* __restrict__ w, const double* __restrict__ V, long long ldv,
                                               long long n, double* partial) {
  double acc[J + 1] = {};
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + stride < n; i += 2 * stride) {
    double w0 = __ldg(w + i), w1 = __ldg(w + i + stride);
    double v0[J], v1[J];
#pragma unroll
    for (int j = 0; j < J; ++j) { v0[j] = __ldg(V + j * ldv + i); v1[j] = __ldg(V + j * ldv + i + stride); }
#pragma unroll
    for (int j = 0; j < J; ++j) acc[j] += v0[j] * w0 + v1[j] * w1;
    acc[J] += w0 * w0 + w1 * w1;
  }
  if (i < n) {
    double wi = w[i];
    for (int j = 0; j < J; ++j) acc[j] += V[j * ldv + i] * wi;
    acc[J] += wi * wi;
  }
  block_sum<J + 1>(acc, partial);
}

// contiguous chunk per block (block b: [b n / G, (b + 1) n / G), 16-element aligned), 16-byte loads,
// U double2 per thread per iteration
template <int J, int U>
__global__ void __launch_bounds__(T) md_chunk(const double* __restrict__ w, const double* __restrict__ V, long long ldv,
                                              long long n, double* partial) {
  double acc[J + 1] = {};
  const long long n2 = n / 2;
  const long long c0 = n2 * blockIdx.x / gridDim.x, c1 = n2 * (blockIdx.x + 1) / gridDim.x;
  const double2* w2 = reinterpret_cast<const double2*>(w);
  long long i = c0 + threadIdx.x;
  for (; i + (U - 1) * T < c1; i += U * T) {
    double2 a[U], v[U][J];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a[u] = __ldg(w2 + i + u * T);
#pragma unroll
      for (int j = 0; j < J; ++j) v[u][j] = __ldg(reinterpret_cast<const double2*>(V + j * ldv) + i + u * T);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int j = 0; j < J; ++j) acc[j] += v[u][j].x * a[u].x + v[u][j].y * a[u].y;
      acc[J] += a[u].x * a[u].x + a[u].y * a[u].y;
    }
  }
  for (; i < c1; i += T) {
    double2 a = __ldg(w2 + i);
    for (int j = 0; j < J; ++j) {
      double2 v = __ldg(reinterpret_cast<const double2*>(V + j * ldv) + i);
      acc[j] += v.x * a.x + v.y * a.y;
    }
    acc[J] += a.x * a.x + a.y * a.y;
  }
  block_sum<J + 1>(acc, partial);
}

// grid stride with 16-byte loads
template <int J>
__global__ void __launch_bounds__(T) md_stride2(const double* __restrict__ w, const double* __restrict__ V, long long ldv,
                                                long long n, double* partial) {
  double acc[J + 1] = {};
  const long long n2 = n / 2;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const double2* w2 = reinterpret_cast<const double2*>(w);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += stride) {
    double2 a = __ldg(w2 + i);
    double2 v[J];
#pragma unroll
    for (int j = 0; j < J; ++j) v[j] = __ldg(reinterpret_cast<const double2*>(V + j * ldv) + i);
#pragma unroll
    for (int j = 0; j < J; ++j) acc[j] += v[j].x * a.x + v[j].y * a.y;
    acc[J] += a.x * a.x + a.y * a.y;
  }
  block_sum<J + 1>(acc, partial);
}

template <class K>
float timeit(K launch, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

template <int J>
void run(long long n, double* w, double* V, long long ld, double* partial) {
  const double gb = (double)(J + 1) * n * 8 / 1e9;
  for (int g : {148 * 4, 148 * 6, 148 * 8, 148 * 16}) {
    float a = timeit([&] { md_stride<J><<<g, T>>>(w, V, ld, n, partial); }, 20);
    float b = timeit([&] { md_chunk<J, 1><<<g, T>>>(w, V, ld, n, partial); }, 20);
    float c = timeit([&] { md_chunk<J, 2><<<g, T>>>(w, V, ld, n, partial); }, 20);
    float d = timeit([&] { md_stride2<J><<<g, T>>>(w, V, ld, n, partial); }, 20);
    printf("J=%2d n=%lld grid=%5d  stride %6.0f  chunk1 %6.0f  chunk2 %6.0f  stride2 %6.0f GB/s\n", J, n, g, gb / a * 1e3,
           gb / b * 1e3, gb / c * 1e3, gb / d * 1e3);
  }
}

int main() {
  const long long nmax = 135005697LL + 64;
  const int JM = 12;
  double *w, *V, *partial;
  cudaMalloc(&V, sizeof(double) * nmax * JM);
  cudaMalloc(&w, sizeof(double) * nmax);
  cudaMalloc(&partial, sizeof(double) * 148 * 16 * 16);
  cudaMemset(V, 0, sizeof(double) * nmax * JM);
  cudaMemset(w, 0, sizeof(double) * nmax);
  for (long long n : {16974593LL + 1, 135005697LL + 1}) {  // even lengths (16-byte pairs)
    const long long ld = (n + 31) / 32 * 32;
    run<6>(n, w, V, ld, partial);
    run<11>(n, w, V, ld, partial);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
