// TMA smoke probe: load a 34x10 box of a padded 3D fp64 array at negative coordinates.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
template <int V>
__global__ void k(const __grid_constant__ CUtensorMap tm, double* out, int c0, int c1, int c2) {
  extern __shared__ __align__(128) double sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  double* dst = sm + 16;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(1));
    if (V >= 1) asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar)), "r"(34 * 10 * 8) : "memory");
    if (V == 2)
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n"
                   ::"r"(su32(dst)), "l"((uint64_t)&tm), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n"
                   ::"r"(su32(dst)), "l"((uint64_t)&tm), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
  }
  asm volatile("{\n .reg .pred P1;\nWAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @P1 bra DONE_%=;\n bra WAIT_%=;\nDONE_%=:\n}\n" ::"r"(su32(bar)), "r"(0) : "memory");
  for (int e = threadIdx.x; e < 340; e += blockDim.x) out[e] = dst[e];
}
int main() {
  int nn = 17, pr = 18, nt1 = 5;
  size_t P = (size_t)pr * nn, N = P * nt1;
  double* h = new double[N];
  for (size_t i = 0; i < N; ++i) h[i] = (double)i;
  double *d, *o;
  cudaMalloc(&d, N * 8); cudaMalloc(&o, 340 * 8);
  cudaMemcpy(d, h, N * 8, cudaMemcpyHostToDevice);
  void* fnp = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto fn = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)nn, (cuuint64_t)nn, (cuuint64_t)nt1};
  cuuint64_t str[2] = {(cuuint64_t)pr * 8, (cuuint64_t)P * 8};
  cuuint32_t box[3] = {34, 10, 1}, es[3] = {1, 1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  for (int v = 0; v < 3; ++v) {
    cudaMemset(o, 0xff, 340 * 8);
    cudaFuncSetAttribute(v == 0 ? k<0> : v == 1 ? k<1> : k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
    if (v == 0) k<0><<<1, 128, 8192>>>(m, o, -1, -1, 2);
    if (v == 1) k<1><<<1, 128, 8192>>>(m, o, -1, -1, 2);
    if (v == 2) k<2><<<1, 128, 8192>>>(m, o, -1, -1, 2);
    cudaError_t e = cudaDeviceSynchronize();
    double ho[340];
    cudaMemcpy(ho, o, 340 * 8, cudaMemcpyDeviceToHost);
    printf("variant %d: %s  [0]=%g [1]=%g [35]=%g expect 0 0 %g\n", v, cudaGetErrorString(e), ho[0], ho[1], (double)(2 * P + 0));
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
