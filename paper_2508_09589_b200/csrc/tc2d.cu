// tc2d.cu — lean (2+1)D level operator for time-constant levels, sm_100a, fp64.
//
// Serves the forms that carry most of the V-cycle bytes for a time-constant (extruded,
// PAPER.md:262, 604-608) design: the matrix-free fine level (FORM_RHO, rho_tc) and the stored
// M/K stencils of every time-constant coarse level (FORM_MK, nl = 1). Same operator and modes
// as op_kernel (ops.cu; plane form in common.cuh / DESIGN.md sec. 7):
//   (K x)_p = [U (x) M + Tm (x) K] rows, with the upwind capacity factor U = [[0,0],[-1,1]]
//   (every level of this build, R-22) and a symmetric conduction factor Tm, so
//     bottom part of layer p-1 -> row p-1:  t00 K x_{p-1} + t01 K x_p
//     top    part of layer p-1 -> row p  :  M (x_p - x_{p-1}) + t01 K x_{p-1} + t11 K x_p
//   and for K^T the capacity moves to the bottom part: -M x_p (bottom), M x_p (top).
// Design:
//   * persistent one-wave grid; CTA c owns a contiguous range of the (tile, plane) list
//     (tile-major), i.e. one or two (tile, plane-range) segments;
//   * 128 threads own a 32 x 8 node tile, 1 x 2 nodes each; one elected thread streams the
//     x tile (36 x 10 with halo; zero outside the domain through the zeroed guard / pad / TMA
//     out-of-bounds fill) and the b tile (32 x 8) of every plane with cp.async.bulk.tensor
//     into a 6-slot ring of mbarrier-tracked slots (5 planes in flight);
//   * 9 stiffness weights per node in registers (from rho on the fly, or the stored symmetric
//     stencil); the mass is either the same (stored) or, for uniform capacity on the fine
//     level, the separable product of 1D masses (x_{-1} + c x_0 + x_1, c = 4 or 2 at a
//     boundary, neighbours outside the domain read as zero: columns -1 and n+1 are the zero
//     pad / guard, rows beyond n are TMA out-of-bounds; the row below j = 0 is zeroed explicitly);
//   * per plane: 12 shared loads, 2 stencil applies per node, the layer combination carried
//     in registers; no per-element masking (the t = 0 plane's layer contributions are skipped
//     by a CTA-uniform branch; sink-patch nodes hold x = 0 in every solver vector).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>

#include "common.cuh"
#include "kernels.h"

#ifndef ST_TC2D_MINB
#define ST_TC2D_MINB 4  // resident CTAs per SM for the uniform-capacity variants (register cap 128)
#endif

namespace st {
namespace tc {

constexpr int TX = 32, TYT = 4, RY = 2, TY = TYT * RY;   // node tile 32 x 8
constexpr int HX = TX + 4, HY = TY + 2;                  // x tile 36 x 10 (col 0 unused: 16-B aligned box)
constexpr int XS = 368, BS = 256;                        // slot sizes (doubles), 128-byte multiples
constexpr int NB = 6;
constexpr int NTH = TX * TYT;
constexpr unsigned XBYTES = HX * HY * 8, BBYTES = TX * TY * 8;
// prolongation fused into a Jacobi sweep (PRO): the coarse correction box of a space-coarsened
// next level, coarse nodes (x0/2 - 2 .. x0/2 + 17) x (y0/2 - 1 .. y0/2 + 4) of the same time plane
constexpr int EW = 20, EH = 6, ES = 128;
constexpr unsigned EBYTES = EW * EH * 8;

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

// 9-point apply on rows r..r+2 of the thread's window
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

// SRC: 0 = fine level from rho (time-constant design), 1 = stored MK stencils (nl = 1)
// PRO (MODE_JAC only): x + P e instead of x, e the correction of the space-coarsened next level
// (tme: its TMA map) — the V-cycle's prolongation + correction fused into the first post-sweep
template <int SRC, bool CUNI, int MODE, bool TRANS, bool PRO = false>
__global__ void __launch_bounds__(NTH, CUNI ? ST_TC2D_MINB : 3)
    tc2d_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmb,
                const __grid_constant__ CUtensorMap tme, OpDesc op, const double* __restrict__ x,
                double* __restrict__ y, double omega, long long wtot, int kchunk, int ntx) {
  static_assert(!PRO || MODE == MODE_JAC, "prolongation is fused into Jacobi sweeps only");
  constexpr bool NX = (MODE != MODE_JAC0);
  constexpr bool NBV = (MODE != MODE_APPLY);
  constexpr bool ND = (MODE == MODE_JAC || MODE == MODE_JAC0);
  extern __shared__ __align__(128) double smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  double* xs = smem + 16;                    // [NB][XS]
  double* bs = xs + (NX ? NB * XS : 0);      // [NB][BS]
  double* es = bs + (NBV ? NB * BS : 0);     // [NB][ES] (PRO)

  const Geom& g = op.g;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
  const int n = g.n, pr = g.pr;
  const long long P = g.P;
  const long long NP = g.nt + 1;
  const int xo = (ty * RY) * HX + tx + 1;   // top-left of the thread's 3 x (RY+2) window in a slot
  const int bo = (ty * RY) * TX + tx;

  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < NB; ++k) mbar_init(&bar[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  pdl_wait();  // the previous kernel's writes (x, b, stencils) are visible from here on
  // spatial scales folded into the time factors (fine level: M = C dx^2/36 [..], K = 1/6 [..])
  const double sm = (SRC == 0) ? g.dx * g.dx * (1.0 / 36.0) * (CUNI ? op.m.Cins : 1.0) : (CUNI ? op.msc : 1.0);
  const double sk = (SRC == 0) ? (1.0 / 6.0) : 1.0;
  const double t00 = op.Tm[0][0] * sk, t01 = op.Tm[0][1] * sk, t11 = op.Tm[1][1] * sk;
  const unsigned tx_full = (NX ? XBYTES : 0u) + (NBV ? BBYTES : 0u) + (PRO ? EBYTES : 0u);

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
    const int i = x0 + tx;
    const int j0 = y0 + ty * RY;
    __syncthreads();  // barrier init / previous segment fully consumed

    if (tid == 0) {
      for (int k = 0; k < NB - 1 && qs + k <= qe; ++k) {
        const int q = qs + k;
        const unsigned slot = (ring + k) % NB;
        const bool wb = NBV && q >= p0 && q < p1;
        mbar_expect_tx(&bar[slot], tx_full - ((NBV && !wb) ? BBYTES : 0u));
        if (NX) tma3(xs + slot * XS, &tmx, &bar[slot], x0, y0, q);
        if (PRO) tma3(es + slot * ES, &tme, &bar[slot], x0 >> 1, y0 >> 1, q);
        if (wb) tma3(bs + slot * BS, &tmb, &bar[slot], x0, y0, q);
      }
    }

    // ---- weights of the thread's nodes --------------------------------------------------
    bool act[RY], patch[RY];
    double wK[RY][9], wM[CUNI ? 1 : RY][9];
    double cx = 4.0, cy[RY];
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      const int j = j0 + r;
      act[r] = (i <= n) && (j <= n);
      patch[r] = i == 0 && j >= g.plo && j <= g.phi;
      cy[r] = (j == 0 || j == n) ? 2.0 : 4.0;
      if (SRC == 0) {
        double ce[4], ke[4];  // SW, SE, NW, NE (zero outside the domain)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int a = i - 1 + (e & 1), bb = j - 1 + (e >> 1);
          const bool v = act[r] && a >= 0 && a < n && bb >= 0 && bb < n;
          const double rho = v ? __ldg(op.rho + (long long)bb * n + a) : 0.0;
          ce[e] = v ? op.m.Cins + op.m.dC * powp(rho, op.m.pc) : 0.0;
          ke[e] = v ? op.m.kins + op.m.dk * powp(rho, op.m.pk) : 0.0;
        }
        const double sw = ke[0], se = ke[1], nw = ke[2], ne = ke[3];
        wK[r][0] = -2.0 * sw; wK[r][2] = -2.0 * se; wK[r][6] = -2.0 * nw; wK[r][8] = -2.0 * ne;
        wK[r][1] = -(sw + se); wK[r][7] = -(nw + ne); wK[r][3] = -(sw + nw); wK[r][5] = -(se + ne);
        wK[r][4] = 4.0 * ((sw + se) + (nw + ne));
        if (!CUNI) {
          const double a = ce[0], b = ce[1], c = ce[2], d = ce[3];
          double* m = wM[CUNI ? 0 : r];
          m[0] = a; m[2] = b; m[6] = c; m[8] = d;
          m[1] = 2.0 * (a + b); m[7] = 2.0 * (c + d); m[3] = 2.0 * (a + c); m[5] = 2.0 * (b + d);
          m[4] = 4.0 * ((a + b) + (c + d));
        }
      } else {
        // stored symmetric stencils: own forward coefficients (k >= 4), mirrored neighbours' (k < 4)
        const long long pn = act[r] ? (long long)j * pr + i : 0;
        const double* Mb = op.st;
        const double* Kb = op.st + 5 * P;
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          const int dx = (k % 3) - 1, dy = (k / 3) - 1;
          double* m = wM[CUNI ? 0 : r];
          if (k >= 4) {
            if (!CUNI) m[k] = act[r] ? __ldg(Mb + (k - 4) * P + pn) : 0.0;
            wK[r][k] = act[r] ? __ldg(Kb + (k - 4) * P + pn) : 0.0;
          } else {
            const int ni = i + dx, nj = j + dy;
            const bool v = act[r] && ni >= 0 && ni <= n && nj >= 0 && nj <= n;
            const long long q = v ? (long long)nj * pr + ni : 0;
            if (!CUNI) m[k] = v ? __ldg(Mb + (8 - k - 4) * P + q) : 0.0;
            wK[r][k] = v ? __ldg(Kb + (8 - k - 4) * P + q) : 0.0;
          }
        }
      }
    }
    if (CUNI) cx = (i == 0 || i == n) ? 2.0 : 4.0;
    // omega / D (interior rows: both layers; last row: top part only)
    double odI[RY];
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      const double mc = (CUNI ? cx * cy[r] : wM[CUNI ? 0 : r][4]) * sm;
      const double kc = wK[r][4];
      // diag = S^{tt}_{p-1} + S^{bb}_p = (mc + t11 kc) + t00 kc (the same for K^T)
      odI[r] = (ND && act[r]) ? omega / (mc + (t00 + t11) * kc) : 0.0;
    }

    double Mprev[RY], Kprev[RY], carry[RY];
#pragma unroll
    for (int r = 0; r < RY; ++r) Mprev[r] = Kprev[r] = carry[r] = 0.0;
    double* yrow = y + (long long)(qs - 1) * P + (long long)j0 * pr + i;  // row q-1 at iteration q
    // windows of the current plane (x) and of the previous plane (x, b) in their ring slots
    unsigned cur = ring, prv = (ring + NB - 1) % NB;
    const double* xq = xs + cur * XS + xo;
    const double* xp = xs + prv * XS + xo;
    const double* bp = bs + prv * BS + bo;
    for (int q = qs; q <= qe; ++q) {
      mbar_wait(&bar[cur], (phase >> cur) & 1u);
      phase ^= 1u << cur;
      if (PRO && q + g.pg0 > 0) {
        // x += P e on the tile's in-domain, unconstrained nodes (the same weights and order as
        // prolong2s_kernel); rows / columns outside the domain keep their zero or aliased values
        double* xt = xs + cur * XS;
        const double* et = es + cur * ES;
        for (int e = tid; e < HY * (TX + 2); e += NTH) {
          const int sr = e / (TX + 2), c = 1 + e % (TX + 2);
          const int ii = x0 - 2 + c, jj = y0 - 1 + sr;
          if (ii < 0 || ii > n || jj < 0 || jj > n) continue;
          if (ii == 0 && jj >= g.plo && jj <= g.phi) continue;  // sink patch
          const double* e0 = et + ((jj >> 1) - (y0 >> 1) + 1) * EW + ((ii >> 1) - (x0 >> 1) + 2);
          double v;
          if (!(ii & 1) && !(jj & 1)) v = e0[0];
          else if (!(jj & 1)) v = 0.5 * (e0[0] + e0[1]);
          else if (!(ii & 1)) v = 0.5 * (e0[0] + e0[EW]);
          else v = 0.25 * ((e0[0] + e0[1]) + (e0[EW] + e0[EW + 1]));
          xt[sr * HX + c] += v;
        }
        __syncthreads();
      }
      double Mq[RY], Kq[RY];  // Mq without the scale sm
      if (NX && q + g.pg0 > 0) {
        double nb[RY + 2][3];
#pragma unroll
        for (int s = 0; s < RY + 2; ++s)
#pragma unroll
          for (int c = 0; c < 3; ++c) nb[s][c] = xq[s * HX + c];
        if (CUNI) {
          double rs[RY + 2];
#pragma unroll
          for (int s = 0; s < RY + 2; ++s) rs[s] = fma(cx, nb[s][1], nb[s][0] + nb[s][2]);
          // the halo row j = -1 of a plane q >= 1 aliases the previous plane's last row: not zero
          if (j0 == 0) rs[0] = 0.0;
#pragma unroll
          for (int r = 0; r < RY; ++r) Mq[r] = fma(cy[r], rs[r + 1], rs[r] + rs[r + 2]);
        } else {
#pragma unroll
          for (int r = 0; r < RY; ++r) Mq[r] = ap9(wM[CUNI ? 0 : r], nb, r);
        }
#pragma unroll
        for (int r = 0; r < RY; ++r) Kq[r] = ap9(wK[r], nb, r);
      } else {  // masked t = 0 plane (JAC0: no x at all)
#pragma unroll
        for (int r = 0; r < RY; ++r) Mq[r] = Kq[r] = 0.0;
      }
      if (q > qs && q - 1 >= p0) {  // row q-1 complete (bottom part of layer q-1)
        if (q - 1 + g.pg0 == 0) {
          // t = 0 plane: identity rows of the initial condition
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
            const double bot = fma(t00, Kprev[r], t01 * Kq[r]);
            const double Ax = TRANS ? fma(-sm, Mq[r], carry[r] + bot) : carry[r] + bot;
            double o;
            if (MODE == MODE_APPLY) o = Ax;
            else if (MODE == MODE_RESID) o = bp[r * TX] - Ax;
            else if (MODE == MODE_JAC) { const double xc = xp[(r + 1) * HX + 1]; o = fma(odI[r], bp[r * TX] - Ax, xc); }
            else o = odI[r] * bp[r * TX];
            // sink-patch rows: x = b = 0 there in every solver vector, so the identity row gives 0
            if (act[r]) yrow[r * pr] = patch[r] ? 0.0 : o;
          }
        }
      }
#pragma unroll
      for (int r = 0; r < RY; ++r) {  // top part of layer q-1 -> row q (none before the first plane)
        const double cap = TRANS ? Mq[r] : Mq[r] - Mprev[r];
        carry[r] = (q > qs) ? fma(sm, cap, fma(t01, Kprev[r], t11 * Kq[r])) : 0.0;
        Mprev[r] = Mq[r];
        Kprev[r] = Kq[r];
      }
      __syncthreads();  // planes q-1, q consumed: the slot of q-1 can be refilled
      if (tid == 0 && q + NB - 1 <= qe) {
        const int qn = q + NB - 1;
        const bool wb = NBV && qn >= p0 && qn < p1;
        mbar_expect_tx(&bar[prv], tx_full - ((NBV && !wb) ? BBYTES : 0u));
        if (NX) tma3(xs + prv * XS, &tmx, &bar[prv], x0, y0, qn);
        if (PRO) tma3(es + prv * ES, &tme, &bar[prv], x0 >> 1, y0 >> 1, qn);
        if (wb) tma3(bs + prv * BS, &tmb, &bar[prv], x0, y0, qn);
      }
      yrow += P;
      prv = cur;
      xp = xq;
      bp = bs + cur * BS + bo;
      if (++cur == NB) { cur = 0u; xq -= (NB - 1) * XS; } else { xq += XS; }
    }
    if (p1 == g.nt + 1) {  // last row: top part of layer nt-1 only
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        const double mc = (CUNI ? cx * cy[r] : wM[CUNI ? 0 : r][4]) * sm;
        const double odT = omega / (mc + t11 * wK[r][4]);
        const double Ax = carry[r];
        double o;
        if (MODE == MODE_APPLY) o = Ax;
        else if (MODE == MODE_RESID) o = bp[r * TX] - Ax;
        else if (MODE == MODE_JAC) o = fma(odT, bp[r * TX] - Ax, xp[(r + 1) * HX + 1]);
        else o = odT * bp[r * TX];
        if (act[r]) yrow[r * pr] = patch[r] ? 0.0 : o;
      }
    }
    ring = cur;
  }
}

}  // namespace tc

// ---------------------------------------------------------------------------------------
namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn_tc() {
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

bool map3_tc(CUtensorMap* m, const void* base, unsigned long long d0, unsigned long long d1, unsigned long long d2,
             unsigned long long s1, unsigned long long s2, unsigned b0, unsigned b1) {
  auto fn = encode_fn_tc();
  if (!fn || ((uintptr_t)base & 15u) || (s1 & 15u) || (s2 & 15u)) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1, s2};
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int SRC, bool CUNI, int MODE, bool TRANS, bool PRO = false>
void ltc(const CUtensorMap& mx, const CUtensorMap& mb, const OpDesc& op, const double* x, double* y, double omega,
         cudaStream_t s, const CUtensorMap* me = nullptr) {
  using namespace tc;
  const Geom& g = op.g;
  auto kern = tc2d_kernel<SRC, CUNI, MODE, TRANS, PRO>;
  constexpr bool NX = (MODE != MODE_JAC0), NBV = (MODE != MODE_APPLY);
  constexpr size_t bytes = sizeof(double) * (16 + (NX ? NB * XS : 0) + (NBV ? NB * BS : 0) + (PRO ? NB * ES : 0));
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
  const long long grid = persistent_grid(op, nsm, resident, wtot);
  launch_pdl(kern, dim3((unsigned)grid), dim3(TX, TYT, 1), bytes, s, mx, mb, me ? *me : mx, op, x, y, omega, wtot,
                                                       chunk_planes(op, g.nt + 1, g.nt + 1), (int)ntx);
}

template <int SRC, bool CUNI>
void ltc_modes(const CUtensorMap& mx, const CUtensorMap& mb, const OpDesc& op, int mode, bool trans, const double* x,
               double* y, double omega, cudaStream_t s) {
#define C4(M)                                                            \
  case M:                                                                \
    if (trans) ltc<SRC, CUNI, M, true>(mx, mb, op, x, y, omega, s);      \
    else ltc<SRC, CUNI, M, false>(mx, mb, op, x, y, omega, s);           \
    break;
  switch (mode) {
    C4(MODE_APPLY)
    C4(MODE_RESID)
    C4(MODE_JAC)
    C4(MODE_JAC0)
  }
#undef C4
}
}  // namespace

// Masked (eliminated) operator only; false if the level is not covered.
bool launch_op_tc2d(const OpDesc& op, int mode, bool trans, bool mask, const double* x, const double* b, double* y,
                    double omega, cudaStream_t s) {
  if (op.g.walls) return false;  // Example 2's cold walls: the generic kernels (is_cons)
  const Geom& g = op.g;
  if (g.sd != 2 || !mask) return false;
  const bool rho_tc = (op.form == FORM_RHO && op.rho_tc), mk_tc = (op.form == FORM_MK && !op.tvl);
  if (!rho_tc && !mk_tc) return false;
  // the lean kernel hard-wires the upwind capacity factor and a symmetric conduction factor
  if (op.U[0][0] != 0.0 || op.U[0][1] != 0.0 || op.U[1][0] != -1.0 || op.U[1][1] != 1.0) return false;
  if (op.Tm[0][1] != op.Tm[1][0]) return false;
  CUtensorMap mx{}, mb{};
  const unsigned long long nn = g.nn, s1 = (unsigned long long)g.pr * 8, s2 = (unsigned long long)g.P * 8;
  const bool nx = (mode != MODE_JAC0), nbv = (mode != MODE_APPLY);
  // x: based pr + 2 entries before the data (zeroed front guard): box coordinate (x0, y0, q) is
  // node (x0 - 2, y0 - 1) of plane q; columns i = n+1 (pad) and beyond / rows beyond n read zero
  if (nx && !map3_tc(&mx, x - (g.pr + 2), (unsigned long long)g.pr + 2, nn + 1, g.nt + 1, s1, s2, tc::HX, tc::HY))
    return false;
  if (nbv && !map3_tc(&mb, b, nn, nn, g.nt + 1, s1, s2, tc::TX, tc::TY)) return false;
  if (rho_tc && op.m.dC == 0.0) ltc_modes<0, true>(mx, mb, op, mode, trans, x, y, omega, s);
  else if (rho_tc) ltc_modes<0, false>(mx, mb, op, mode, trans, x, y, omega, s);
  else if (op.msep) ltc_modes<1, true>(mx, mb, op, mode, trans, x, y, omega, s);
  else ltc_modes<1, false>(mx, mb, op, mode, trans, x, y, omega, s);
  return true;
}

// Damped-Jacobi sweep from x + P e (the V-cycle's prolongation + correction fused into the first
// post-smoothing sweep): e is the correction of the next level gc, a space coarsening of this one
// (same time planes, one GPU). false if not covered (then: prolongation kernel + plain sweep).
bool launch_op_tc2d_pro(const OpDesc& op, const Geom& gc, bool trans, const double* x, const double* e,
                        const double* b, double* y, double omega, cudaStream_t s) {
  if (op.g.walls) return false;  // Example 2's cold walls: the generic kernels (is_cons)
  const Geom& g = op.g;
  if (g.sd != 2 || gc.nt != g.nt || gc.nn != g.n / 2 + 1 || g.pg0 != 0 || gc.pg0 != 0) return false;
  const bool rho_tc = (op.form == FORM_RHO && op.rho_tc), mk_tc = (op.form == FORM_MK && !op.tvl);
  if (!rho_tc && !mk_tc) return false;
  if (op.U[0][0] != 0.0 || op.U[0][1] != 0.0 || op.U[1][0] != -1.0 || op.U[1][1] != 1.0) return false;
  if (op.Tm[0][1] != op.Tm[1][0]) return false;
  CUtensorMap mx{}, mb{}, me{};
  const unsigned long long nn = g.nn, s1 = (unsigned long long)g.pr * 8, s2 = (unsigned long long)g.P * 8;
  if (!map3_tc(&mx, x - (g.pr + 2), (unsigned long long)g.pr + 2, nn + 1, g.nt + 1, s1, s2, tc::HX, tc::HY)) return false;
  if (!map3_tc(&mb, b, nn, nn, g.nt + 1, s1, s2, tc::TX, tc::TY)) return false;
  // e: based like x (guarded internal vector): coordinate (X, Y, q) is coarse node (X - 2, Y - 1)
  if (!map3_tc(&me, e - (gc.pr + 2), (unsigned long long)gc.pr + 2, (unsigned long long)gc.nn + 1, gc.nt + 1,
               (unsigned long long)gc.pr * 8, (unsigned long long)gc.P * 8, tc::EW, tc::EH))
    return false;
#define PR(SRC, CU)                                                                          \
  if (trans) ltc<SRC, CU, MODE_JAC, true, true>(mx, mb, op, x, y, omega, s, &me);            \
  else ltc<SRC, CU, MODE_JAC, false, true>(mx, mb, op, x, y, omega, s, &me);
  if (rho_tc && op.m.dC == 0.0) { PR(0, true) }
  else if (rho_tc) { PR(0, false) }
  else if (op.msep) { PR(1, true) }
  else { PR(1, false) }
#undef PR
  return true;
}

}  // namespace st
