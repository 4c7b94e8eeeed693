// tma2d.cu — (2+1)D level operator with TMA plane streaming, sm_100a, fp64.
//
// Same operator and modes as op_kernel (ops.cu; algebra in common.cuh). Covers the forms that
// carry the V-cycle bytes: the fine level (FORM_RHO, time-constant or space-time design) and
// the stored MK stencils of time-constant coarse levels:
//   * CTA = 128 threads owns a 32 x 8 node tile and marches through a chunk of time planes;
//     each thread owns 1 x 2 nodes;
//   * one elected thread streams the x plane tile (36 x 10 with halo) and the b tile (32 x 8)
//     with cp.async.bulk.tensor into a 6-slot shared-memory ring tracked by mbarriers (5 planes
//     in flight), so the loop has no per-element copy code; for a space-time design the rho
//     tile of the layer (33 x 9) follows with cp.async;
//   * preconditions (true for every vector of the solver; the ABI test hooks mask first):
//     x = 0 at the sink-patch nodes; the t = 0 plane is treated as zero (MASK) and its rows
//     are identity rows;
//   * time-constant levels keep their 9-point stiffness (and, for non-uniform capacity, mass)
//     weights in registers: 2 stencil applies per plane, the layer combination is carried;
//     uniform capacity applies the mass separably (My (x) Mx, 1D patterns [1,4,1]/[0,2,1]/[1,2,0]).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace st {
namespace t2 {

constexpr int TX = 32, TYT = 4, RY = 2, TY = TYT * RY;   // node tile 32 x 8
// x tile: columns x0-2 .. x0+33 (36, the first is unused: keeps the TMA base 16-byte aligned),
// rows y0-1 .. y0+8; the map is based pr + 2 entries before the data (zeroed front guard), so
// box coordinates (x0, y0, q) are never negative
constexpr int HX = TX + 4, HY = TY + 2;                  // 36 x 10
constexpr int RYE = TY + 1;                              // element rows of the rho tile
constexpr int XS = 368, BS = 256, RS = 320;              // slot sizes (doubles), 128-byte multiples
constexpr int EX = TX + 1, ET = EX * RYE;                // element tile 33 x 9
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

__device__ __forceinline__ double ap9(const double* w, const double (&nb)[RY + 2][3], int r) {
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

// integer-scaled 9-point weights from the 4 element coefficients (SW, SE, NW, NE)
__device__ __forceinline__ void wM_from(double sw, double se, double nw, double ne, double* w) {
  w[0] = sw; w[2] = se; w[6] = nw; w[8] = ne;
  w[1] = 2.0 * (sw + se); w[7] = 2.0 * (nw + ne);
  w[3] = 2.0 * (sw + nw); w[5] = 2.0 * (se + ne);
  w[4] = 4.0 * ((sw + se) + (nw + ne));
}
__device__ __forceinline__ void wK_from(double sw, double se, double nw, double ne, double* w) {
  w[0] = -2.0 * sw; w[2] = -2.0 * se; w[6] = -2.0 * nw; w[8] = -2.0 * ne;
  w[1] = -(sw + se); w[7] = -(nw + ne);
  w[3] = -(sw + nw); w[5] = -(se + ne);
  w[4] = 4.0 * ((sw + se) + (nw + ne));
}

// SRC: 0 = RHO (fine level), 1 = MK stored (time-constant coarse level).
// Persistent, balanced schedule: the work is the list of (tile, plane) pairs in tile-major order;
// CTA c takes the contiguous range [c W / G, (c+1) W / G) of it (W = tiles x (nt+1), G = grid) and
// processes it as one or two (tile, plane-range) segments. The grid is one wave (SMs x resident
// CTAs), so there is no partial last wave whatever the tile count.
template <bool TC, int SRC, bool CUNI, int MODE, bool TRANS, bool MASK>
__global__ void __launch_bounds__(NTH, (TC && CUNI) ? 4 : 3)
    tma2d_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmb, OpDesc op,
                 const double* __restrict__ x, double* __restrict__ y, double omega, long long wtot, int kchunk, int ntx) {
  constexpr bool TVR = (!TC) && SRC == 0;
  constexpr bool NX = (MODE != MODE_JAC0);
  constexpr bool NBV = (MODE != MODE_APPLY);
  constexpr bool ND = (MODE == MODE_JAC || MODE == MODE_JAC0);
  extern __shared__ __align__(128) double smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);                 // NB "full" mbarriers
  double* xs = smem + 16;                                            // [NB][XS]
  double* bs = xs + (NX ? NB * XS : 0);                              // [NB][BS]
  double* rs = bs + (NBV ? NB * BS : 0);                             // [NB][RS]
  double* cC = rs + (TVR ? NB * RS : 0);                             // [ET]
  double* cK = cC + (TVR ? ET : 0);

  const Geom& g = op.g;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
  const int n = g.n, pr = g.pr;
  const long long P = g.P;
  const long long NP = g.nt + 1;
  // per-thread shared offsets (doubles, within one slot)
  const int xo = (ty * RY) * HX + tx + 1;     // top-left of the thread's 3 x (RY+2) window
  const int bo = (ty * RY) * TX + tx;         // b of the thread's first row

  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < NB; ++k) mbar_init(&bar[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }

  // time factors with the spatial scale folded in (block transpose: (a,b) -> (b,a))
  const double sm = (SRC == 0) ? g.dx * g.dx * (1.0 / 36.0) * (CUNI ? op.m.Cins : 1.0) : 1.0;
  const double sk = (SRC == 0) ? (1.0 / 6.0) : 1.0;
  const double u00 = op.U[0][0] * sm, u11 = op.U[1][1] * sm;
  const double u01 = (TRANS ? op.U[1][0] : op.U[0][1]) * sm, u10 = (TRANS ? op.U[0][1] : op.U[1][0]) * sm;
  const double t00 = op.Tm[0][0] * sk, t11 = op.Tm[1][1] * sk;
  const double t01 = (TRANS ? op.Tm[1][0] : op.Tm[0][1]) * sk, t10 = (TRANS ? op.Tm[0][1] : op.Tm[1][0]) * sk;
  const unsigned tx_full = (NX ? XBYTES : 0u) + (NBV ? BBYTES : 0u);

  long long w = wtot * blockIdx.x / gridDim.x;
  const long long wend = wtot * (blockIdx.x + 1) / gridDim.x;
  unsigned ring = 0u;   // slot of the first plane of the next segment
  unsigned phase = 0u;  // mbarrier parity bit per slot
  while (w < wend) {
    long long tile;
    int p0, p1;
    work_segment(w, wend, wtot / NP, (int)NP, kchunk, &tile, &p0, &p1);
    w += p1 - p0;
    const int x0 = (int)(tile % ntx) * TX, y0 = (int)(tile / ntx) * TY;
    const int qs = max(p0 - 1, 0), qe = min(p1, g.nt);
    const int i = x0 + tx;
    int jr[RY];
    bool act[RY], patch[RY];
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      jr[r] = y0 + ty * RY + r;
      act[r] = (i <= n) && (jr[r] <= n);
      patch[r] = MASK && i == 0 && jr[r] >= g.plo && jr[r] <= g.phi;
    }
    __syncthreads();  // barrier init (first segment) / every slot of the previous segment consumed

    // ---- producer: one elected thread, NB-1 planes in flight ------------------------------
    auto issue = [&](int q, unsigned slot) {
      unsigned bytes = tx_full;
      const bool wb = NBV && q >= p0 && q < p1;
      if (NBV && !wb) bytes -= BBYTES;
      mbar_expect_tx(&bar[slot], bytes);
      if (NX) tma3(xs + slot * XS, &tmx, &bar[slot], x0, y0, q);
      if (wb) tma3(bs + slot * BS, &tmb, &bar[slot], x0, y0, q);
    };
    // space-time design: rho tile of layer q-1 (33 x 9 elements from (x0-1, y0-1)) by cp.async
    constexpr int RPT = (ET + NTH - 1) / NTH;
    int roff[RPT];
    unsigned rval = 0u;
    if (TVR) {
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        const int e = tid + k * NTH;
        const int ly = e / EX, lx = e - ly * EX;
        const int gi = x0 - 1 + lx, gj = y0 - 1 + ly;
        const bool v = (e < ET) && gi >= 0 && gi < n && gj >= 0 && gj < n;
        roff[k] = v ? gj * n + gi : 0;
        if (v) rval |= 1u << k;
      }
    }
    auto issue_rho = [&](int q, unsigned slot) {  // all threads; one commit group per plane
      if (TVR && q - 1 >= qs && q <= qe) {
        double* rd = rs + slot * RS;
        const double* rq = op.rho + (long long)(q - 1) * n * n;
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
          const int e = tid + k * NTH;
          if (e < ET) {
            const int sz = ((rval >> k) & 1u) ? 8 : 0;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(su32(rd + e)), "l"(rq + roff[k]), "r"(sz));
          }
        }
      }
      if (TVR) asm volatile("cp.async.commit_group;\n" ::);
    };
    if (tid == 0) {
#pragma unroll
      for (int k = 0; k < NB - 1; ++k)
        if (qs + k <= qe) issue(qs + k, (ring + k) % NB);
    }
#pragma unroll
    for (int k = 0; k < NB - 1; ++k) issue_rho(qs + k, (ring + k) % NB);

    // ---- time-constant weights of the thread's nodes (registers) ---------------------------
    double wM[(TC && !CUNI) ? RY : 1][9], wK[TC ? RY : 1][9];
    double wx[3], wy[RY][3];
    if (CUNI) {
      wx[0] = (i == 0) ? 0.0 : 1.0; wx[1] = (i == 0 || i == n) ? 2.0 : 4.0; wx[2] = (i >= n) ? 0.0 : 1.0;
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        const int j = jr[r];
        wy[r][0] = (j == 0) ? 0.0 : 1.0; wy[r][1] = (j == 0 || j == n) ? 2.0 : 4.0; wy[r][2] = (j >= n) ? 0.0 : 1.0;
      }
    }
    if (TC) {
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        if (SRC == 0) {
          double ce[4], ke[4];  // SW, SE, NW, NE
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int a = i - 1 + (e & 1), bb = jr[r] - 1 + (e >> 1);
            const bool v = act[r] && a >= 0 && a < n && bb >= 0 && bb < n;
            const double rho = v ? __ldg(op.rho + (long long)bb * n + a) : 0.0;
            ce[e] = v ? op.m.Cins + op.m.dC * powp(rho, op.m.pc) : 0.0;
            ke[e] = v ? op.m.kins + op.m.dk * powp(rho, op.m.pk) : 0.0;
          }
          if (!CUNI) wM_from(ce[0], ce[1], ce[2], ce[3], wM[CUNI ? 0 : r]);
          wK_from(ke[0], ke[1], ke[2], ke[3], wK[r]);
        } else {
          const long long pn = act[r] ? (long long)jr[r] * pr + i : 0;
          const double* Mb = op.st;
          const double* Kb = op.st + 5 * P;
#pragma unroll
          for (int k = 0; k < 9; ++k) {
            const int dx = (k % 3) - 1, dy = (k / 3) - 1;
            if (k >= 4) {
              wM[CUNI ? 0 : r][k] = act[r] ? __ldg(Mb + (k - 4) * P + pn) : 0.0;
              wK[r][k] = act[r] ? __ldg(Kb + (k - 4) * P + pn) : 0.0;
            } else {
              const int ni = i + dx, nj = jr[r] + dy;
              const bool v = act[r] && ni >= 0 && ni <= n && nj >= 0 && nj <= n;
              const long long q = v ? (long long)nj * pr + ni : 0;
              wM[CUNI ? 0 : r][k] = v ? __ldg(Mb + (8 - k - 4) * P + q) : 0.0;
              wK[r][k] = v ? __ldg(Kb + (8 - k - 4) * P + q) : 0.0;
            }
          }
        }
      }
    }
    double odI[RY], odT[RY];  // omega / D: interior rows, last row
    if (TC && ND) {
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        const double mc = CUNI ? wx[1] * wy[r][1] : wM[CUNI ? 0 : r][4];
        const double db = u00 * mc + t00 * wK[r][4], dt = u11 * mc + t11 * wK[r][4];
        odI[r] = act[r] ? omega / (db + dt) : 0.0;
        odT[r] = act[r] ? omega / dt : 0.0;
      }
    }

    double Mprev[RY], Kprev[RY], carry[RY], dcarry[RY];
#pragma unroll
    for (int r = 0; r < RY; ++r) Mprev[r] = Kprev[r] = carry[r] = dcarry[r] = 0.0;
    const long long nodeoff = (long long)jr[0] * pr + i;
    double* yrow = y + (long long)(qs - 1) * P + nodeoff;  // row q-1 of iteration q

    // output of row p (slot = ring slot of plane p); Ax = A x at the row, od = omega / D
    auto out_rows = [&](int p, unsigned slot, const double* Ax, const double* od) {
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        if (!act[r]) continue;
        const bool cons = MASK && (p + g.pg0 == 0 || patch[r]);
        const double bv = NBV ? bs[slot * BS + bo + r * TX] : 0.0;
        double xc = 0.0;
        if (NX) xc = (MASK && p + g.pg0 == 0) ? __ldg(yrow - y + x + r * pr) : xs[slot * XS + xo + (r + 1) * HX + 1];
        double o;
        if (MODE == MODE_APPLY) o = cons ? xc : Ax[r];
        else if (MODE == MODE_RESID) o = bv - (cons ? xc : Ax[r]);
        else if (MODE == MODE_JAC) o = cons ? fma(omega, bv - xc, xc) : fma(od[r], bv - Ax[r], xc);
        else o = (cons ? omega : od[r]) * bv;
        yrow[r * pr] = o;
      }
    };

    unsigned cur = ring, prv = (ring + NB - 1) % NB;
    for (int q = qs; q <= qe; ++q) {
      mbar_wait(&bar[cur], (phase >> cur) & 1u);
      phase ^= 1u << cur;
      if (TVR) {
        asm volatile("cp.async.wait_group %0;\n" ::"n"(NB - 2));
        if (q > qs) {
          // C, k~ of the layer q-1 rho tile this thread copied (zero outside the domain)
#pragma unroll
          for (int k = 0; k < RPT; ++k) {
            const int e = tid + k * NTH;
            if (e < ET) {
              const bool v = (rval >> k) & 1u;
              const double rho = rs[cur * RS + e];
              cC[e] = v ? op.m.Cins + op.m.dC * powp(rho, op.m.pc) : 0.0;
              cK[e] = v ? op.m.kins + op.m.dk * powp(rho, op.m.pk) : 0.0;
            }
          }
        }
        if (MASK && NX && q + g.pg0 == 0) {  // masked t = 0 plane: zero its x slot (raw values via __ldg)
          for (int e = tid; e < HX * HY; e += NTH) xs[cur * XS + e] = 0.0;
        }
        __syncthreads();
      }
      const bool outp = (q > qs) && (q - 1 >= p0);  // row q-1 is this segment's
      if (TC) {
        double Mq[RY], Kq[RY];
        if (NX && !(MASK && q + g.pg0 == 0)) {
          double nb[RY + 2][3];
          const double* t = xs + cur * XS + xo;
#pragma unroll
          for (int s = 0; s < RY + 2; ++s)
#pragma unroll
            for (int c = 0; c < 3; ++c) nb[s][c] = t[s * HX + c];
          double rsum[RY + 2];
          if (CUNI) {
#pragma unroll
            for (int s = 0; s < RY + 2; ++s) rsum[s] = fma(wx[0], nb[s][0], fma(wx[1], nb[s][1], wx[2] * nb[s][2]));
          }
#pragma unroll
          for (int r = 0; r < RY; ++r) {
            Mq[r] = CUNI ? fma(wy[r][0], rsum[r], fma(wy[r][1], rsum[r + 1], wy[r][2] * rsum[r + 2]))
                         : ap9(wM[CUNI ? 0 : r], nb, r);
            Kq[r] = ap9(wK[r], nb, r);
          }
        } else {
#pragma unroll
          for (int r = 0; r < RY; ++r) Mq[r] = Kq[r] = 0.0;
        }
        if (outp) {
          double Ax[RY];
#pragma unroll
          for (int r = 0; r < RY; ++r)
            Ax[r] = carry[r] + fma(u00, Mprev[r], fma(u01, Mq[r], fma(t00, Kprev[r], t01 * Kq[r])));
          out_rows(q - 1, prv, Ax, odI);
        }
#pragma unroll
        for (int r = 0; r < RY; ++r) {  // top part of layer q-1 -> row q (none before the first plane)
          carry[r] = (q > qs) ? fma(u10, Mprev[r], fma(u11, Mq[r], fma(t10, Kprev[r], t11 * Kq[r]))) : 0.0;
          Mprev[r] = Mq[r];
          Kprev[r] = Kq[r];
        }
      } else if (q > qs) {
        double nbp[RY + 2][3], nbq[RY + 2][3];
        if (NX) {
          const double* tp = xs + prv * XS + xo;
          const double* tq = xs + cur * XS + xo;
#pragma unroll
          for (int s = 0; s < RY + 2; ++s)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              nbp[s][c] = tp[s * HX + c];
              nbq[s][c] = tq[s * HX + c];
            }
        }
        double cw[RY + 1], ckw[RY + 1], ce_[RY + 1], cke[RY + 1];
#pragma unroll
        for (int s = 0; s <= RY; ++s) {
          const int e = (ty * RY + s) * EX + tx;
          cw[s] = cC[e]; ce_[s] = cC[e + 1];
          ckw[s] = cK[e]; cke[s] = cK[e + 1];
        }
        double Ax[RY], od[RY];
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          double w1[9], w2[9];
          wM_from(cw[r], ce_[r], cw[r + 1], ce_[r + 1], w1);
          wK_from(ckw[r], cke[r], ckw[r + 1], cke[r + 1], w2);
          double bot = 0.0, top = 0.0;
          if (NX) {
            const double Mb = ap9(w1, nbp, r), Mt = ap9(w1, nbq, r);
            const double Kb = ap9(w2, nbp, r), Kt = ap9(w2, nbq, r);
            bot = fma(u00, Mb, fma(u01, Mt, fma(t00, Kb, t01 * Kt)));
            top = fma(u10, Mb, fma(u11, Mt, fma(t10, Kb, t11 * Kt)));
          }
          const double db = u00 * w1[4] + t00 * w2[4];
          const double dt = u11 * w1[4] + t11 * w2[4];
          od[r] = (ND && act[r]) ? omega / (dcarry[r] + db) : 0.0;
          Ax[r] = carry[r] + bot;
          carry[r] = top;
          dcarry[r] = dt;
        }
        if (outp) out_rows(q - 1, prv, Ax, od);
      }
      __syncthreads();  // everyone is done with planes q-1, q: the slot of q-1 can be refilled
      if (tid == 0 && q + NB - 1 <= qe) issue(q + NB - 1, prv);
      issue_rho(q + NB - 1, prv);
      yrow += P;
      prv = cur;
      cur = (cur + 1 == NB) ? 0u : cur + 1;
    }
    if (p1 == g.nt + 1) {  // last row: top part of layer nt-1 only
      double od[RY];
#pragma unroll
      for (int r = 0; r < RY; ++r) od[r] = ND ? (TC ? odT[r] : (act[r] ? omega / dcarry[r] : 0.0)) : 0.0;
      out_rows(g.nt, prv, carry, od);
    }
    ring = cur;
  }
  if (TVR) asm volatile("cp.async.wait_group 0;\n" ::);
}

}  // namespace t2

// ---------------------------------------------------------------------------------------
namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

bool map3(CUtensorMap* m, const void* base, unsigned long long d0, unsigned long long d1, unsigned long long d2,
          unsigned long long s1, unsigned long long s2, unsigned b0, unsigned b1) {
  auto fn = encode_fn();
  if (!fn || ((uintptr_t)base & 15u) || (s1 & 15u) || (s2 & 15u)) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1, s2};
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool TC, int SRC, bool CUNI, int MODE, bool TRANS, bool MASK>
void lt2(const CUtensorMap& mx, const CUtensorMap& mb, const OpDesc& op, const double* x, double* y, double omega,
         cudaStream_t s) {
  using namespace t2;
  const Geom& g = op.g;
  auto kern = tma2d_kernel<TC, SRC, CUNI, MODE, TRANS, MASK>;
  constexpr bool NX = (MODE != MODE_JAC0), NBV = (MODE != MODE_APPLY), TVR = (!TC) && SRC == 0;
  constexpr size_t bytes = sizeof(double) * (16 + (NX ? NB * XS : 0) + (NBV ? NB * BS : 0) + (TVR ? NB * RS + 2 * ET : 0));
  static int resident = 0;  // CTAs per SM (occupancy), once per instantiation
  static int nsm = 0;
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
  kern<<<(unsigned)grid, dim3(TX, TYT, 1), bytes, s>>>(mx, mb, op, x, y, omega, wtot, chunk_planes(op, g.nt + 1, g.nt + 1), (int)ntx);
}

template <bool TC, int SRC, bool CUNI>
void lt2_modes(const CUtensorMap& mx, const CUtensorMap& mb, const OpDesc& op, int mode, bool trans, bool mask,
               const double* x, double* y, double omega, cudaStream_t s) {
  if (!mask) {
    if (trans) lt2<TC, SRC, CUNI, MODE_APPLY, true, false>(mx, mb, op, x, y, omega, s);
    else lt2<TC, SRC, CUNI, MODE_APPLY, false, false>(mx, mb, op, x, y, omega, s);
    return;
  }
#define C4(M)                                                                        \
  case M:                                                                            \
    if (trans) lt2<TC, SRC, CUNI, M, true, true>(mx, mb, op, x, y, omega, s);    \
    else lt2<TC, SRC, CUNI, M, false, true>(mx, mb, op, x, y, omega, s);         \
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

bool launch_op_tma2d(const OpDesc& op, int mode, bool trans, bool mask, const double* x, const double* b, double* y,
                     double omega, cudaStream_t s) {
  if (op.g.walls) return false;  // Example 2's cold walls: the generic kernels (is_cons)
  const Geom& g = op.g;
  if (g.sd != 2) return false;
  const bool rho_tc = (op.form == FORM_RHO && op.rho_tc), rho_tv = (op.form == FORM_RHO && !op.rho_tc);
  const bool mk_tc = (op.form == FORM_MK && !op.tvl);
  if (!rho_tc && !rho_tv && !mk_tc) return false;
  CUtensorMap mx{}, mb{};
  const unsigned long long nn = g.nn, s1 = (unsigned long long)g.pr * 8, s2 = (unsigned long long)g.P * 8;
  const bool nx = (mode != MODE_JAC0), nbv = (mode != MODE_APPLY);
  // x: based pr + 2 entries before the data (front guard), dims (pr + 2, nn + 1, nt + 1): box
  // coordinate (x0, y0, q) is node (x0 - 2, y0 - 1) of plane q
  if (nx && !map3(&mx, x - (g.pr + 2), (unsigned long long)g.pr + 2, nn + 1, g.nt + 1, s1, s2, t2::HX, t2::HY))
    return false;
  if (nbv && !map3(&mb, b, nn, nn, g.nt + 1, s1, s2, t2::TX, t2::TY)) return false;
  if (rho_tc && op.m.dC == 0.0) lt2_modes<true, 0, true>(mx, mb, op, mode, trans, mask, x, y, omega, s);
  else if (rho_tc) lt2_modes<true, 0, false>(mx, mb, op, mode, trans, mask, x, y, omega, s);
  else if (rho_tv) lt2_modes<false, 0, false>(mx, mb, op, mode, trans, mask, x, y, omega, s);
  else lt2_modes<true, 1, false>(mx, mb, op, mode, trans, mask, x, y, omega, s);
  return true;
}

}  // namespace st
