// tc3d.cu — (3+1)D level operator for time-constant levels, sm_100a, fp64.
//
// The (3+1)D analogue of tc2d.cu (the 16-node tensor-product space-time element, SURVEY.md 2.7
// B4): the fine level from a time-constant rho (FORM_RHO) and the stored M/K stencils of
// time-constant coarse levels (FORM_MK), all masked modes. Plane form as in tc2d.cu
// (upwind capacity factor U = [[0,0],[-1,1]], symmetric conduction factor Tm):
//   bottom part of layer p-1 -> row p-1:  t00 K x_{p-1} + t01 K x_p          (K^T: - M x_p)
//   top    part of layer p-1 -> row p  :  M (x_p - x_{p-1}) + t01 K x_{p-1} + t11 K x_p  (K^T: M x_p)
// with 27-point spatial stencils M (mass, weighted by C_e) and K (stiffness, weighted by k~_e;
// its 6 face-neighbour weights vanish for the trilinear element).
// Design:
//   * persistent one-wave grid over the (tile, plane) list, as tc2d;
//   * CTA = 256 threads = one 16 x 8 x 2 node tile, one node per thread (16-wide x rows waste
//     less than 32-wide ones on the 2^k + 1 node lines of the hierarchy); one elected thread
//     streams the x tile (20 x 10 x 4 with halo) and the b tile (16 x 8 x 2) of every plane with
//     4-D cp.async.bulk.tensor into a 5-slot mbarrier ring (4 planes in flight);
//   * 27 + 21 weights per node in registers (fine level; a Galerkin coarse stiffness has 27),
//     built once per segment (from rho, or from the stored forward coefficients and the
//     neighbours' mirrored ones); per plane 27 shared loads and 48 (54) FMA per node; ghost /
//     outside entries carry zero weight, so the halo needs no mask.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace st {
namespace t3 {

constexpr int TX = 16, TY = 8, TZ = 2;                    // node tile 16 x 8 x 2 (a warp: 16 x 2)
constexpr int HX = TX + 4, HY = TY + 2, HZ = TZ + 2;      // x tile 20 x 10 x 4 (col 0 unused)
constexpr int XS = HX * HY * HZ;                          // 800 doubles (6400 B, 128-B multiple)
constexpr int BS = TX * TY * TZ;                          // 256 doubles
constexpr int NB = 5;
constexpr int NTH = TX * TY * TZ;
constexpr unsigned XBYTES = XS * 8, BBYTES = BS * 8;

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
__device__ __forceinline__ void tma4(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];\n" ::"r"(
          su32(dst)),
      "l"((uint64_t)map), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// K weight slot of stencil offset k (0..26). The trilinear fine-level stiffness vanishes on the 6
// face neighbours (21 weights, FACE0 = true); a Galerkin coarse stiffness P^T K P does not (27).
template <bool FACE0> __host__ __device__ constexpr int kslot(int k) {
  return !FACE0 ? k
                : ((k == 4 || k == 10 || k == 12 || k == 14 || k == 16 || k == 22) ? -1
                   : (k - (k > 4) - (k > 10) - (k > 12) - (k > 14) - (k > 16) - (k > 22)));
}

// SRC: 0 = fine level from rho (time-constant design), 1 = stored MK stencils (nl = 1)
#ifndef ST_TC3D_MINB
#define ST_TC3D_MINB 2  // resident CTAs per SM of the fine-level variants (register cap 128); 1 CTA
                        // (184 registers) with the 27 window loads batched ahead of the FMAs
                        // measured slower: 634 vs ~580 us per config-4 sweep
#endif
template <int SRC, int MODE, bool TRANS>
#ifndef ST_TC3D_MINB1
#define ST_TC3D_MINB1 1  // resident CTAs per SM of the stored-stencil variants (54 weights per node)
#endif
__global__ void __launch_bounds__(NTH, SRC == 0 ? ST_TC3D_MINB : ST_TC3D_MINB1)
    tc3d_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmb, OpDesc op,
                const double* __restrict__ x, double* __restrict__ y, double omega, long long wtot, int kchunk, int ntx,
                int nty) {
  constexpr bool NX = (MODE != MODE_JAC0);
  constexpr bool NBV = (MODE != MODE_APPLY);
  constexpr bool ND = (MODE == MODE_JAC || MODE == MODE_JAC0);
  constexpr bool F0 = (SRC == 0);          // fine level: zero face stiffness
  constexpr int NK = F0 ? 21 : 27;
  extern __shared__ __align__(128) double smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  double* xs = smem + 16;                    // [NB][XS]
  double* bs = xs + (NX ? NB * XS : 0);      // [NB][BS]

  const Geom& g = op.g;
  const int tx = threadIdx.x, ty = threadIdx.y, tz = threadIdx.z;
  const int tid = (tz * TY + ty) * TX + tx;
  const int n = g.n, nn = g.nn, pr = g.pr;
  const long long P = g.P, RS = (long long)pr * nn;  // slice stride (x3)
  const long long NP = g.nt + 1;
  const int xo = (tz * HY + ty) * HX + tx + 1;        // (-1,-1,-1) corner of the thread's 3x3x3 window
  const int bo = tid;

  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < NB; ++k) mbar_init(&bar[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  const double sm = (SRC == 0) ? g.dx * g.dx * g.dx * (1.0 / 216.0) : 1.0;
  const double sk = (SRC == 0) ? g.dx * (1.0 / 12.0) : 1.0;
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
    const int tyx = (int)(tile % ((long long)ntx * nty));
    const int x0 = (tyx % ntx) * TX, y0 = (tyx / ntx) * TY, z0 = (int)(tile / ((long long)ntx * nty)) * TZ;
    const int qs = max(p0 - 1, 0), qe = min(p1, g.nt);
    const int i = x0 + tx, j = y0 + ty, kz = z0 + tz;
    const bool act = (i <= n) && (j <= n) && (kz <= n);
    const bool patch = i == 0 && j >= g.plo && j <= g.phi && kz >= g.plo && kz <= g.phi;
    __syncthreads();  // barrier init / previous segment fully consumed

    if (tid == 0) {
      for (int k = 0; k < NB - 1 && qs + k <= qe; ++k) {
        const int q = qs + k;
        const unsigned slot = (ring + k) % NB;
        const bool wb = NBV && q >= p0 && q < p1;
        mbar_expect_tx(&bar[slot], tx_full - ((NBV && !wb) ? BBYTES : 0u));
        if (NX) tma4(xs + slot * XS, &tmx, &bar[slot], x0, y0, z0, q);
        if (wb) tma4(bs + slot * BS, &tmb, &bar[slot], x0, y0, z0, q);
      }
    }

    // ---- weights of the thread's node: 27 mass, 21 stiffness (face weights vanish) --------
    double wM[27], wK[NK];
    if (SRC == 0) {
      double ce[8], ke[8];  // element (e0, e1, e2) in {-1, 0}^3 at bit e: node - 1 + bit
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int a = i - 1 + (e & 1), bb = j - 1 + ((e >> 1) & 1), cc = kz - 1 + (e >> 2);
        const bool v = act && a >= 0 && a < n && bb >= 0 && bb < n && cc >= 0 && cc < n;
        const double rho = v ? __ldg(op.rho + ((long long)cc * n + bb) * n + a) : 0.0;
        ce[e] = v ? op.m.Cins + op.m.dC * powp(rho, op.m.pc) : 0.0;
        ke[e] = v ? op.m.kins + op.m.dk * powp(rho, op.m.pk) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < 27; ++k) {
        const int d0 = (k % 3) - 1, d1 = ((k / 3) % 3) - 1, d2 = (k / 9) - 1;
        const int h = (d0 != 0) + (d1 != 0) + (d2 != 0);
        double sc = 0.0, skk = 0.0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int b0 = e & 1, b1 = (e >> 1) & 1, b2 = e >> 2;  // element side: 0 -> below, 1 -> above
          const bool in = (d0 == 0 || (d0 == 1) == (b0 == 1)) && (d1 == 0 || (d1 == 1) == (b1 == 1)) &&
                          (d2 == 0 || (d2 == 1) == (b2 == 1));
          if (in) { sc += ce[e]; skk += ke[e]; }
        }
        wM[k] = sc * (h == 0 ? 8.0 : (h == 1 ? 4.0 : (h == 2 ? 2.0 : 1.0)));
        if (kslot<F0>(k) >= 0) wK[kslot<F0>(k)] = skk * (h == 0 ? 4.0 : -1.0);
      }
    } else {
      const double* Mb = op.st;
      const double* Kb = op.st + 14 * P;
      const long long pn = act ? (long long)kz * RS + (long long)j * pr + i : 0;
#pragma unroll
      for (int k = 0; k < 27; ++k) {
        const int d0 = (k % 3) - 1, d1 = ((k / 3) % 3) - 1, d2 = (k / 9) - 1;
        double mv = 0.0, kv = 0.0;
        if (k >= 13) {  // own forward coefficient
          if (act) {
            mv = __ldg(Mb + (k - 13) * P + pn);
            kv = __ldg(Kb + (k - 13) * P + pn);
          }
        } else {  // mirrored: the neighbour's coefficient of the opposite offset
          const int ni = i + d0, nj = j + d1, nk = kz + d2;
          const bool v = act && ni >= 0 && ni <= n && nj >= 0 && nj <= n && nk >= 0 && nk <= n;
          const long long q = v ? (long long)nk * RS + (long long)nj * pr + ni : 0;
          if (v) {
            mv = __ldg(Mb + (26 - k - 13) * P + q);
            kv = __ldg(Kb + (26 - k - 13) * P + q);
          }
        }
        wM[k] = mv;
        if (kslot<F0>(k) >= 0) wK[kslot<F0>(k)] = kv;
      }
    }
    const double mc = wM[13] * sm, kc = wK[kslot<F0>(13)];
    const double odI = (ND && act) ? omega / (mc + (t00 + t11) * kc) : 0.0;

    double Mprev = 0.0, Kprev = 0.0, carry = 0.0;
    double* yrow = y + (long long)(qs - 1) * P + (long long)kz * RS + (long long)j * pr + i;
    unsigned cur = ring, prv = (ring + NB - 1) % NB;
    const double* xq = xs + cur * XS + xo;
    const double* xp = xs + prv * XS + xo;
    const double* bp = bs + prv * BS + bo;
    for (int q = qs; q <= qe; ++q) {
      mbar_wait(&bar[cur], (phase >> cur) & 1u);
      phase ^= 1u << cur;
      double Mq = 0.0, Kq = 0.0;  // Mq without the scale sm
      if (NX && q + g.pg0 > 0) {
        double ma = 0.0, mb = 0.0, ka = 0.0, kb = 0.0;
#pragma unroll
        for (int k = 0; k < 27; ++k) {
          const int d0 = (k % 3), d1 = ((k / 3) % 3), d2 = (k / 9);
          const double v = xq[(d2 * HY + d1) * HX + d0];
          if (k & 1) ma = fma(wM[k], v, ma); else mb = fma(wM[k], v, mb);
          if (kslot<F0>(k) >= 0) {
            if (k & 1) ka = fma(wK[kslot<F0>(k)], v, ka); else kb = fma(wK[kslot<F0>(k)], v, kb);
          }
        }
        Mq = ma + mb;
        Kq = ka + kb;
      }
      if (q > qs && q - 1 >= p0) {  // row q-1 complete
        if (q - 1 + g.pg0 == 0) {   // t = 0 plane: identity rows of the initial condition
          if (act) {
            const double xc = NX ? __ldg(x + (yrow - y)) : 0.0;
            const double bv = NBV ? bp[0] : 0.0;
            double o;
            if (MODE == MODE_APPLY) o = xc;
            else if (MODE == MODE_RESID) o = bv - xc;
            else if (MODE == MODE_JAC) o = fma(omega, bv - xc, xc);
            else o = omega * bv;
            *yrow = o;
          }
        } else {
          const double bot = fma(t00, Kprev, t01 * Kq);
          const double Ax = TRANS ? fma(-sm, Mq, carry + bot) : carry + bot;
          double o;
          if (MODE == MODE_APPLY) o = Ax;
          else if (MODE == MODE_RESID) o = bp[0] - Ax;
          else if (MODE == MODE_JAC) o = fma(odI, bp[0] - Ax, xp[(HY + 1) * HX + 1]);
          else o = odI * bp[0];
          // sink-patch rows: x = b = 0 there in every solver vector
          if (act) *yrow = patch ? 0.0 : o;
        }
      }
      {
        const double cap = TRANS ? Mq : Mq - Mprev;
        carry = (q > qs) ? fma(sm, cap, fma(t01, Kprev, t11 * Kq)) : 0.0;
        Mprev = Mq;
        Kprev = Kq;
      }
      __syncthreads();  // planes q-1, q consumed: the slot of q-1 can be refilled
      if (tid == 0 && q + NB - 1 <= qe) {
        const int qn = q + NB - 1;
        const bool wb = NBV && qn >= p0 && qn < p1;
        mbar_expect_tx(&bar[prv], tx_full - ((NBV && !wb) ? BBYTES : 0u));
        if (NX) tma4(xs + prv * XS, &tmx, &bar[prv], x0, y0, z0, qn);
        if (wb) tma4(bs + prv * BS, &tmb, &bar[prv], x0, y0, z0, qn);
      }
      yrow += P;
      prv = cur;
      xp = xq;
      bp = bs + cur * BS + bo;
      if (++cur == NB) { cur = 0u; xq -= (NB - 1) * XS; } else { xq += XS; }
    }
    if (p1 == g.nt + 1) {  // last row: top part of layer nt-1 only
      const double odT = omega / (mc + t11 * kc);
      const double Ax = carry;
      double o;
      if (MODE == MODE_APPLY) o = Ax;
      else if (MODE == MODE_RESID) o = bp[0] - Ax;
      else if (MODE == MODE_JAC) o = fma(odT, bp[0] - Ax, xp[(HY + 1) * HX + 1]);
      else o = odT * bp[0];
      if (act) *yrow = patch ? 0.0 : o;
    }
    ring = cur;
  }
}

}  // namespace t3

// ---------------------------------------------------------------------------------------
namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn_t3() {
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

bool map4(CUtensorMap* m, const void* base, const unsigned long long (&dims)[4], const unsigned long long (&str)[3],
          const unsigned (&box)[4]) {
  auto fn = encode_fn_t3();
  if (!fn || ((uintptr_t)base & 15u)) return false;
  for (int d = 0; d < 3; ++d)
    if (str[d] & 15u) return false;
  cuuint64_t dd[4] = {dims[0], dims[1], dims[2], dims[3]};
  cuuint64_t ss[3] = {str[0], str[1], str[2]};
  cuuint32_t bb[4] = {box[0], box[1], box[2], box[3]};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void*>(base), dd, ss, bb, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int SRC, int MODE, bool TRANS>
void lt3(const CUtensorMap& mx, const CUtensorMap& mb, const OpDesc& op, const double* x, double* y, double omega,
         cudaStream_t s) {
  using namespace t3;
  const Geom& g = op.g;
  auto kern = tc3d_kernel<SRC, MODE, TRANS>;
  constexpr bool NX = (MODE != MODE_JAC0), NBV = (MODE != MODE_APPLY);
  constexpr size_t bytes = sizeof(double) * (16 + (NX ? NB * XS : 0) + (NBV ? NB * BS : 0));
  static int resident = 0, nsm = 0;
  if (!resident) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, kern, NTH, bytes);
    if (resident < 1) resident = 1;
  }
  const long long ntx = (g.nn + TX - 1) / TX, nty = (g.nn + TY - 1) / TY, ntz = (g.nn + TZ - 1) / TZ;
  const long long wtot = ntx * nty * ntz * (g.nt + 1);
  const long long grid = persistent_grid(op, nsm, resident, wtot);
  kern<<<(unsigned)grid, dim3(TX, TY, TZ), bytes, s>>>(mx, mb, op, x, y, omega, wtot, chunk_planes(op, g.nt + 1, g.nt + 1), (int)ntx, (int)nty);
}

template <int SRC>
void lt3_modes(const CUtensorMap& mx, const CUtensorMap& mb, const OpDesc& op, int mode, bool trans, const double* x,
               double* y, double omega, cudaStream_t s) {
#define C4(M)                                                     \
  case M:                                                         \
    if (trans) lt3<SRC, M, true>(mx, mb, op, x, y, omega, s);     \
    else lt3<SRC, M, false>(mx, mb, op, x, y, omega, s);          \
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

// Masked (eliminated) operator on a (3+1)D time-constant level; false if not covered.
bool launch_op_tc3d(const OpDesc& op, int mode, bool trans, bool mask, const double* x, const double* b, double* y,
                    double omega, cudaStream_t s) {
  if (op.g.walls) return false;  // Example 2's cold walls: the generic kernels (is_cons)
  const Geom& g = op.g;
  if (g.sd != 3 || !mask) return false;
  const bool rho_tc = (op.form == FORM_RHO && op.rho_tc), mk_tc = (op.form == FORM_MK && !op.tvl);
  if (!rho_tc && !mk_tc) return false;
  if (op.U[0][0] != 0.0 || op.U[0][1] != 0.0 || op.U[1][0] != -1.0 || op.U[1][1] != 1.0) return false;
  if (op.Tm[0][1] != op.Tm[1][0]) return false;
  CUtensorMap mx{}, mb{};
  const unsigned long long nn = g.nn, pr = g.pr;
  const unsigned long long str[3] = {pr * 8, pr * nn * 8, (unsigned long long)g.P * 8};
  const bool nx = (mode != MODE_JAC0), nbv = (mode != MODE_APPLY);
  // x: based one slice + one row + 2 entries before the data (zeroed front guard), so the box
  // coordinate (x0, y0, z0, q) is node (x0 - 2, y0 - 1, z0 - 1) of plane q
  const long long shift = (long long)pr * nn + pr + 2;
  if (nx) {
    const unsigned long long dims[4] = {pr + 2, nn + 1, nn + 1, (unsigned long long)g.nt + 1};
    const unsigned box[4] = {t3::HX, t3::HY, t3::HZ, 1};
    if (!map4(&mx, x - shift, dims, str, box)) return false;
  }
  if (nbv) {
    const unsigned long long dims[4] = {nn, nn, nn, (unsigned long long)g.nt + 1};
    const unsigned box[4] = {t3::TX, t3::TY, t3::TZ, 1};
    if (!map4(&mb, b, dims, str, box)) return false;
  }
  if (rho_tc) lt3_modes<0>(mx, mb, op, mode, trans, x, y, omega, s);
  else lt3_modes<1>(mx, mb, op, mode, trans, x, y, omega, s);
  return true;
}

}  // namespace st
