// tv2d.cu — (2+1)D fine-level operator for a space-time (time-varying) design with uniform
// capacity, sm_100a, fp64 (BASELINE configs 1, 3, 5: C = 1, k = k(rho) per element and layer).
//
// Same operator and modes as op_kernel (ops.cu; plane form in DESIGN.md sec. 7) with the upwind
// capacity factor and a symmetric conduction factor (as tc2d.cu). With uniform capacity the mass
// is the same separable stencil on every layer; the stiffness of layer tau, K^(tau), comes from
// the element conductivities of that layer. Per plane q the kernel forms
//   M x_q (separable),  Kb_q = K^(q-1) x_q  (layer below),  Ka_q = K^(q) x_q  (layer above)
// and completes row q-1 = carry + t00 Ka_{q-1} + t01 Kb_q (K^T: - M x_q), carry for row q =
// M (x_q - x_{q-1}) + t01 Ka_{q-1} + t11 Kb_q (K^T: M x_q).
// Design: persistent one-wave grid over (tile, plane) work as tc2d; x and b
// tiles by TMA into a 6-slot mbarrier ring; the 33 x 9 element tile of rho for layer q by
// cp.async (zero outside the domain), converted once to k~ in shared memory (two layer buffers);
// 9 stiffness weights per node and layer rebuilt from 4 element values; 2 applies per plane.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace st {
namespace tv {

constexpr int TX = 32, TYT = 4, RY = 2, TY = TYT * RY;   // node tile 32 x 8
constexpr int HX = TX + 4, HY = TY + 2;                  // x tile 36 x 10 (col 0 unused)
constexpr int XS = 368, BS = 256;                        // slot sizes (doubles)
constexpr int EX = TX + 1, EY = TY + 1, ET = EX * EY;    // element tile 33 x 9
constexpr int CXW = TX + 2, CT = CXW * EY;               // stored-coefficient node tile 34 x 9
constexpr int RS0 = 304, RS1 = 5 * CT + 2;               // per-layer slot: rho tile / 5 K coefficient tiles
constexpr int NB = 6;
constexpr int NTH = TX * TYT;
constexpr unsigned XBYTES = HX * HY * 8, BBYTES = TX * TY * 8;

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @P1 bra DONE_%=;\n"
      " bra WAIT_%=;\n"
      "DONE_%=:\n}\n" ::"r"(su32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(
          su32(dst)),
      "l"((uint64_t)map), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ double ap9(const double (&w)[9], const double (&nb)[RY + 2][3], int r) {
  double a = w[4] * nb[r + 1][1];
  double b = w[0] * nb[r][0];
  a = fma(w[1], nb[r][1], a);
  b = fma(w[2], nb[r][2], b);
  a = fma(w[3], nb[r + 1][0], a);
  b = fma(w[5], nb[r + 1][2], b);
  a = fma(w[6], nb[r + 2][0], a);
  b = fma(w[7], nb[r + 2][1], b);
  a = fma(w[8], nb[r + 2][2], a);
  return a + b;
}

// 1/d for the per-plane Jacobi diagonal: float reciprocal + two Newton steps (full double accuracy
// for the positive, float-range diagonals; ~8 instructions instead of a double division)
__device__ __forceinline__ double rcp_d(double d) {
  double r = (double)__frcp_rn((float)d);
  r = r * fma(-d, r, 2.0);
  return r * fma(-d, r, 2.0);
}

// 9 stiffness weights of the thread's row-r node from the 4 element conductivities (x 6)
__device__ __forceinline__ void wk_from(double sw, double se, double nw, double ne, double (&w)[9]) {
  w[0] = -2.0 * sw; w[2] = -2.0 * se; w[6] = -2.0 * nw; w[8] = -2.0 * ne;
  w[1] = -(sw + se); w[7] = -(nw + ne); w[3] = -(sw + nw); w[5] = -(se + ne);
  w[4] = 4.0 * ((sw + se) + (nw + ne));
}

// SRC: 0 = fine level from rho (per-layer k~ from the element densities); 1 = stored per-layer
// stiffness of a time-varying Galerkin space level (uniform capacity: the separable mass op.msc)
// PK3: SIMP conductivity exponent p_k = 3 (every BASELINE config) evaluated as rho^3 (a runtime
// exponent costs a branch ladder and a pow call per element and layer)
template <int SRC, int MODE, bool TRANS, bool PK3>
__global__ void __launch_bounds__(NTH, SRC == 0 ? 3 : 2)
    tv2d_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmb, OpDesc op,
                const double* __restrict__ x, double* __restrict__ y, double omega, long long wtot, int kchunk, int ntx) {
  constexpr bool NX = (MODE != MODE_JAC0);
  constexpr bool NBV = (MODE != MODE_APPLY);
  constexpr bool ND = (MODE == MODE_JAC || MODE == MODE_JAC0);
  extern __shared__ __align__(128) double smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  double* xs = smem + 16;                    // [NB][XS]
  double* bs = xs + (NX ? NB * XS : 0);      // [NB][BS]
  constexpr int RS = SRC == 0 ? RS0 : RS1;
  double* rs = bs + (NBV ? NB * BS : 0);     // [NB][RS] layer tiles (layer q arrives with plane q)
  double* kk = rs + NB * RS;                 // [2][ET] k~ of the current / next layer (SRC 0)

  const Geom& g = op.g;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
  const int n = g.n, pr = g.pr;
  const long long P = g.P;
  const long long NP = g.nt + 1;
  const int xo = (ty * RY) * HX + tx + 1;
  const int bo = (ty * RY) * TX + tx;
  constexpr int TILE = SRC == 0 ? ET : 5 * CT;  // doubles copied per layer
  constexpr int RPT = (TILE + NTH - 1) / NTH;

  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < NB; ++k) mbar_init(&bar[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  const double sm = SRC == 0 ? g.dx * g.dx * (1.0 / 36.0) * op.m.Cins : op.msc;
  const double sk = SRC == 0 ? 1.0 / 6.0 : 1.0;
  const double t00 = op.Tm[0][0] * sk, t01 = op.Tm[0][1] * sk, t11 = op.Tm[1][1] * sk;
  const unsigned tx_full = (NX ? XBYTES : 0u) + (NBV ? BBYTES : 0u);

  long long w = wtot * blockIdx.x / gridDim.x;
  const long long wend = wtot * (blockIdx.x + 1) / gridDim.x;
  unsigned ring = 0u, phase = 0u;
  while (w < wend) {
    long long tile;
    int p0, p1;
    work_segment(w, wend, wtot / NP, (int)NP, kchunk, &tile, &p0, &p1);
    w += p1 - p0;
    const int x0 = (int)(tile % ntx) * TX, y0 = (int)(tile / ntx) * TY;
    const int qs = max(p0 - 1, 0), qe = min(p1, g.nt);
    const int i = x0 + tx, j0 = y0 + ty * RY;
    bool act[RY], patch[RY];
    double cy[RY];
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      const int j = j0 + r;
      act[r] = (i <= n) && (j <= n);
      patch[r] = i == 0 && j >= g.plo && j <= g.phi;
      cy[r] = (j == 0 || j == n) ? 2.0 : 4.0;
    }
    const double cx = (i == 0 || i == n) ? 2.0 : 4.0;
    // this thread's per-layer copies: SRC 0 the 33 x 9 element tile of rho from (x0-1, y0-1);
    // SRC 1 the 34 x 9 node tiles of the 5 forward stiffness coefficients from (x0-1, y0-1); zero outside
    long long roff[RPT];
    unsigned rval = 0u;
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      const int e = tid + k * NTH;
      bool v;
      if (SRC == 0) {
        const int ly = e / EX, lx = e - ly * EX;
        const int gi = x0 - 1 + lx, gj = y0 - 1 + ly;
        v = (e < ET) && gi >= 0 && gi < n && gj >= 0 && gj < n;
        roff[k] = v ? (long long)gj * n + gi : 0;
      } else {
        const int a = e / CT, loc = e - a * CT;
        const int ly = loc / CXW, lx = loc - ly * CXW;
        const int gi = x0 - 1 + lx, gj = y0 - 1 + ly;
        v = (e < 5 * CT) && gi >= 0 && gi <= n && gj >= 0 && gj <= n;
        roff[k] = v ? (long long)a * P + (long long)gj * pr + gi : 0;
      }
      if (v) rval |= 1u << k;
    }
    __syncthreads();  // barrier init / previous segment fully consumed

    // producer: x / b by TMA (elected thread), rho layer q by cp.async (all threads), one
    // commit group per plane
    auto issue_rho = [&](int q, unsigned slot) {
      if (q < g.nt) {  // layer q exists locally (the last plane has no layer above)
        double* rd = rs + slot * RS;
        const double* rq = SRC == 0 ? op.rho + (long long)q * n * n
                                    : op.st + ((long long)q * 2 + 1) * 5 * P;  // K block of layer q
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
          const int e = tid + k * NTH;
          if (e < TILE) {
            const int sz = ((rval >> k) & 1u) ? 8 : 0;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(su32(rd + e)), "l"(rq + roff[k]), "r"(sz));
          }
        }
      }
      asm volatile("cp.async.commit_group;\n" ::);
    };
    if (tid == 0) {
      for (int k = 0; k < NB - 1 && qs + k <= qe; ++k) {
        const int q = qs + k;
        const unsigned slot = (ring + k) % NB;
        const bool wb = NBV && q >= p0 && q < p1;
        mbar_expect_tx(&bar[slot], tx_full - ((NBV && !wb) ? BBYTES : 0u));
        if (NX) tma3(xs + slot * XS, &tmx, &bar[slot], x0, y0, q);
        if (wb) tma3(bs + slot * BS, &tmb, &bar[slot], x0, y0, q);
      }
    }
    for (int k = 0; k < NB - 1; ++k) {
      if (qs + k <= qe) issue_rho(qs + k, (ring + k) % NB);
      else asm volatile("cp.async.commit_group;\n" ::);
    }

    double wKc[RY][9];  // stiffness weights of layer q-1 (below plane q)
    double dCc[RY];     // their centre weights
    double Mprev[RY], Kaprev[RY], carry[RY], dcarry[RY];
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      Mprev[r] = Kaprev[r] = carry[r] = dcarry[r] = dCc[r] = 0.0;
#pragma unroll
      for (int k = 0; k < 9; ++k) wKc[r][k] = 0.0;
    }
    double* yrow = y + (long long)(qs - 1) * P + (long long)j0 * pr + i;
    unsigned cur = ring, prv = (ring + NB - 1) % NB;
    const double* xq = xs + cur * XS + xo;
    const double* xp = xs + prv * XS + xo;
    const double* bp = bs + prv * BS + bo;
    int kb = 0;  // k~ buffer of the layer above plane q
    for (int q = qs; q <= qe; ++q) {
      mbar_wait(&bar[cur], (phase >> cur) & 1u);
      phase ^= 1u << cur;
      asm volatile("cp.async.wait_group %0;\n" ::"n"(NB - 2));
      // k~ of layer q (above plane q), zero outside the domain / beyond the last layer
      if (SRC == 0) {
        double* kd = kk + kb * ET;
        const double* rd = rs + cur * RS;
        const bool has = q < g.nt;
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
          const int e = tid + k * NTH;
          if (e < ET) {
            const bool v = has && ((rval >> k) & 1u);
            const double rr = rd[e];
            kd[e] = v ? op.m.kins + op.m.dk * (PK3 ? rr * rr * rr : powp(rr, op.m.pk)) : 0.0;
          }
        }
      }
      __syncthreads();
      // weights of layer q for the thread's nodes (rows j0, j0+1): elements rows j0-1 .. j0+1
      double wKn[RY][9];
      if (SRC == 1) {
        // own forward coefficients and the neighbours' mirrored ones (zero beyond the last layer)
        const double* ct = rs + cur * RS;
        const bool has = q < g.nt;
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          const int L = (ty * RY + r + 1) * CXW + tx + 1;  // node (i, j) in the tile
          wKn[r][4] = has ? ct[0 * CT + L] : 0.0;
          wKn[r][5] = has ? ct[1 * CT + L] : 0.0;
          wKn[r][6] = has ? ct[2 * CT + L] : 0.0;
          wKn[r][7] = has ? ct[3 * CT + L] : 0.0;
          wKn[r][8] = has ? ct[4 * CT + L] : 0.0;
          wKn[r][0] = has ? ct[4 * CT + L - CXW - 1] : 0.0;  // (i-1, j-1): its (+1, +1)
          wKn[r][1] = has ? ct[3 * CT + L - CXW] : 0.0;      // (i,   j-1): its ( 0, +1)
          wKn[r][2] = has ? ct[2 * CT + L - CXW + 1] : 0.0;  // (i+1, j-1): its (-1, +1)
          wKn[r][3] = has ? ct[1 * CT + L - 1] : 0.0;        // (i-1, j  ): its (+1,  0)
        }
      } else {
        const double* kd = kk + kb * ET + (ty * RY) * EX + tx;
        double kw[RY + 1], ke[RY + 1];
#pragma unroll
        for (int s = 0; s <= RY; ++s) { kw[s] = kd[s * EX]; ke[s] = kd[s * EX + 1]; }
#pragma unroll
        for (int r = 0; r < RY; ++r) wk_from(kw[r], ke[r], kw[r + 1], ke[r + 1], wKn[r]);
      }
      double Mq[RY], Kb[RY], Ka[RY];
      if (NX && q + g.pg0 > 0) {
        double nb[RY + 2][3];
#pragma unroll
        for (int s = 0; s < RY + 2; ++s)
#pragma unroll
          for (int c = 0; c < 3; ++c) nb[s][c] = xq[s * HX + c];
        double rsum[RY + 2];
#pragma unroll
        for (int s = 0; s < RY + 2; ++s) rsum[s] = fma(cx, nb[s][1], nb[s][0] + nb[s][2]);
        if (j0 == 0) rsum[0] = 0.0;  // row j = -1 aliases the previous plane's last row
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          Mq[r] = fma(cy[r], rsum[r + 1], rsum[r] + rsum[r + 2]);
          Kb[r] = ap9(wKc[r], nb, r);
          Ka[r] = ap9(wKn[r], nb, r);
        }
      } else {
#pragma unroll
        for (int r = 0; r < RY; ++r) Mq[r] = Kb[r] = Ka[r] = 0.0;
      }
      if (q > qs && q - 1 >= p0) {  // row q-1 complete (bottom part of layer q-1)
        if (q - 1 + g.pg0 == 0) {
#pragma unroll
          for (int r = 0; r < RY; ++r) {
            if (!act[r]) continue;
            const double xc = NX ? __ldg(x + (yrow - y) + r * pr) : 0.0;
            const double bv = NBV ? bp[r * TX] : 0.0;
            double o;
            if (MODE == MODE_APPLY) o = xc;
            else if (MODE == MODE_RESID) o = bv - xc;
            else if (MODE == MODE_JAC) o = fma(omega, bv - xc, xc);
            else o = omega * bv;
            yrow[r * pr] = o;
          }
        } else {
#pragma unroll
          for (int r = 0; r < RY; ++r) {
            const double bot = fma(t00, Kaprev[r], t01 * Kb[r]);
            const double Ax = TRANS ? fma(-sm, Mq[r], carry[r] + bot) : carry[r] + bot;
            const double od = ND ? omega * rcp_d(dcarry[r] + t00 * dCc[r]) : 0.0;
            double o;
            if (MODE == MODE_APPLY) o = Ax;
            else if (MODE == MODE_RESID) o = bp[r * TX] - Ax;
            else if (MODE == MODE_JAC) o = fma(od, bp[r * TX] - Ax, xp[(r + 1) * HX + 1]);
            else o = od * bp[r * TX];
            if (act[r]) yrow[r * pr] = patch[r] ? 0.0 : o;
          }
        }
      }
#pragma unroll
      for (int r = 0; r < RY; ++r) {  // top part of layer q-1 -> row q; diagonal carried likewise
        const double cap = TRANS ? Mq[r] : Mq[r] - Mprev[r];
        const bool lay = q > qs;
        carry[r] = lay ? fma(sm, cap, fma(t01, Kaprev[r], t11 * Kb[r])) : 0.0;
        dcarry[r] = lay ? fma(sm, cx * cy[r], t11 * dCc[r]) : 0.0;
        Mprev[r] = Mq[r];
        Kaprev[r] = Ka[r];
        dCc[r] = wKn[r][4];
#pragma unroll
        for (int k = 0; k < 9; ++k) wKc[r][k] = wKn[r][k];
      }
      __syncthreads();  // planes q-1, q and the k~ buffer of layer q-1 consumed
      if (tid == 0 && q + NB - 1 <= qe) {
        const int qn = q + NB - 1;
        const bool wb = NBV && qn >= p0 && qn < p1;
        mbar_expect_tx(&bar[prv], tx_full - ((NBV && !wb) ? BBYTES : 0u));
        if (NX) tma3(xs + prv * XS, &tmx, &bar[prv], x0, y0, qn);
        if (wb) tma3(bs + prv * BS, &tmb, &bar[prv], x0, y0, qn);
      }
      if (q + NB - 1 <= qe) issue_rho(q + NB - 1, prv);
      else asm volatile("cp.async.commit_group;\n" ::);
      kb ^= 1;
      yrow += P;
      prv = cur;
      xp = xq;
      bp = bs + cur * BS + bo;
      if (++cur == NB) { cur = 0u; xq -= (NB - 1) * XS; } else { xq += XS; }
    }
    if (p1 == g.nt + 1) {  // last row: top part of layer nt-1 only
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        const double od = ND ? omega / dcarry[r] : 0.0;
        const double Ax = carry[r];
        double o;
        if (MODE == MODE_APPLY) o = Ax;
        else if (MODE == MODE_RESID) o = bp[r * TX] - Ax;
        else if (MODE == MODE_JAC) o = fma(od, bp[r * TX] - Ax, xp[(r + 1) * HX + 1]);
        else o = od * bp[r * TX];
        if (act[r]) yrow[r * pr] = patch[r] ? 0.0 : o;
      }
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
    ring = cur;
  }
}

}  // namespace tv

// ---------------------------------------------------------------------------------------
namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn_tv() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    else
      cudaGetLastError();
  }
  return fn;
}

bool map3_tv(CUtensorMap* m, const void* base, unsigned long long d0, unsigned long long d1, unsigned long long d2,
             unsigned long long s1, unsigned long long s2, unsigned b0, unsigned b1) {
  auto fn = encode_fn_tv();
  if (!fn || ((uintptr_t)base & 15u) || (s1 & 15u) || (s2 & 15u)) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1, s2};
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int SRC, int MODE, bool TRANS, bool PK3>
void ltv(const CUtensorMap& mx, const CUtensorMap& mb, const OpDesc& op, const double* x, double* y, double omega,
         cudaStream_t s) {
  using namespace tv;
  const Geom& g = op.g;
  auto kern = tv2d_kernel<SRC, MODE, TRANS, PK3>;
  constexpr bool NX = (MODE != MODE_JAC0), NBV = (MODE != MODE_APPLY);
  constexpr int RS = SRC == 0 ? RS0 : RS1;
  constexpr size_t bytes = sizeof(double) * (16 + (NX ? NB * XS : 0) + (NBV ? NB * BS : 0) + NB * RS + 2 * ET);
  static int resident = 0, nsm = 0;
  if (!resident) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, kern, NTH, bytes);
    if (resident < 1) resident = 1;
  }
  const long long ntx = (g.nn + TX - 1) / TX, nty = (g.nn + TY - 1) / TY;
  const long long wtot = ntx * nty * (g.nt + 1);
  long long grid = (long long)nsm * resident;
  // large levels: >= 4 planes per CTA (one reload plane per segment); small levels: every CTA a
  // short chain so that the TMA round trips of a level overlap (launch-latency bound there)
  const long long minw = (wtot >= 16LL * nsm * resident) ? 4 : 1;
  if (grid > wtot / minw) grid = wtot / minw;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, dim3(TX, TYT, 1), bytes, s>>>(mx, mb, op, x, y, omega, wtot, chunk_planes(g.P, g.nt + 1, g.sd), (int)ntx);
}
}  // namespace

// Masked modes of the fine level of a space-time design with uniform capacity; false if not covered.
bool launch_op_tv2d(const OpDesc& op, int mode, bool trans, bool mask, const double* x, const double* b, double* y,
                    double omega, cudaStream_t s) {
  const Geom& g = op.g;
  const bool rho_tv = op.form == FORM_RHO && !op.rho_tc && op.m.dC == 0.0;
  const bool mk_tv = op.form == FORM_MK && op.tvl && op.msep;
  const bool pk3 = op.m.pk == 3.0;
  if (g.sd != 2 || !mask || !(rho_tv || mk_tv)) return false;
  if (op.U[0][0] != 0.0 || op.U[0][1] != 0.0 || op.U[1][0] != -1.0 || op.U[1][1] != 1.0) return false;
  if (op.Tm[0][1] != op.Tm[1][0]) return false;
  CUtensorMap mx{}, mb{};
  const unsigned long long nn = g.nn, s1 = (unsigned long long)g.pr * 8, s2 = (unsigned long long)g.P * 8;
  const bool nx = (mode != MODE_JAC0), nbv = (mode != MODE_APPLY);
  if (nx && !map3_tv(&mx, x - (g.pr + 2), (unsigned long long)g.pr + 2, nn + 1, g.nt + 1, s1, s2, tv::HX, tv::HY))
    return false;
  if (nbv && !map3_tv(&mb, b, nn, nn, g.nt + 1, s1, s2, tv::TX, tv::TY)) return false;
#define C4(M)                                                                            \
  case M:                                                                                \
    if (rho_tv && pk3) { if (trans) ltv<0, M, true, true>(mx, mb, op, x, y, omega, s);   \
                         else ltv<0, M, false, true>(mx, mb, op, x, y, omega, s); }      \
    else if (rho_tv) { if (trans) ltv<0, M, true, false>(mx, mb, op, x, y, omega, s);    \
                       else ltv<0, M, false, false>(mx, mb, op, x, y, omega, s); }       \
    else { if (trans) ltv<1, M, true, true>(mx, mb, op, x, y, omega, s);                 \
           else ltv<1, M, false, true>(mx, mb, op, x, y, omega, s); }                    \
    break;
  switch (mode) {
    C4(MODE_APPLY)
    C4(MODE_RESID)
    C4(MODE_JAC)
    C4(MODE_JAC0)
  }
#undef C4
  return true;
}

}  // namespace st
