// tc3r.cu — (3+1)D fine-level operator for a time-constant design (BASELINE config 4), sm_100a, fp64.
//
// Same operator, modes and plane form as tc3d.cu: per node plane q the kernel needs
// the spatial mass and stiffness products M x_q and K x_q of the 16-node space-time element
// and completes
//   row q-1 += t00 K x_{q-1} + t01 K x_q            (K^T: - M x_q)
//   row q    = M (x_q - x_{q-1}) + t01 K x_{q-1} + t11 K x_q   (K^T: M x_q).
// tc3d evaluates both products as 27-point stencils with 48 per-node weights in registers: one node
// per thread, 27 shared-memory loads per node and plane — the kernel is bound by the shared-memory
// crossbar (27 x 8 B per node and plane; ~300 us per config-4 sweep at 128 B/clk/SM) and by its
// 16 x 8 x 2 tiles on the 65-node lines of a 64^3 grid (70 % of the threads active).
//
// This kernel evaluates the products ELEMENT-wise, layer by layer, with the trilinear element matrices
// written as tensor products of the 1D factors m = (2, 1) (mass) and k = (1, -1) (stiffness):
//   M_e = (dx^3/216) m(x)m(x)m,   K_e = (dx/36) (k(x)m(x)m + m(x)k(x)m + m(x)m(x)k)
// (the 3D Q1 matrices, entries (dx^3/216)[8,4,2,1] and (dx/12)[4,0,-1,-1] by Hamming distance; the
// decomposition is exact). A thread owns a column of R nodes in x3 (z) at one (x1, x2) position and
// walks the R + 2 node slices z0-1 .. z0+R of its column: per slice it forms, for each of the 4 element
// quadrants q = (sx, sy) of the (x1, x2) plane, the 2D quadrant products
//   Bm_q = sum m(cx) m(cy) x(sx cx, sy cy),   Bk_q = sum (k(cx) m(cy) + m(cx) k(cy)) x(sx cx, sy cy)
// (9 shared loads per slice), and per element layer between slices s-1 and s (element coefficients
// c_q, k_q of the layer in registers, evaluated from rho once per segment)
//   bottom node (slice s-1):  M += sum c_q (2 Bm_q(s-1) + Bm_q(s)),
//                             K += sum k_q (2 Bk_q(s-1) + Bk_q(s) + Bm_q(s-1) - Bm_q(s))
//   top node    (slice s):    M += sum c_q (Bm_q(s-1) + 2 Bm_q(s)),
//                             K += sum k_q (Bk_q(s-1) + 2 Bk_q(s) - Bm_q(s-1) + Bm_q(s)).
// Shared loads per node: 9 (R + 2) / R (13.5 at R = 4, against 27), no per-node weights (4 (R + 1)
// element coefficients per thread), ~75 fp64 operations per node and plane.
// Tiles are FULL x1 rows: a CTA of RY nn threads (RY rows of the nn = n + 1 nodes, nn <= 176) owns an
// RY x R block of node columns, so a 64^3 grid runs at 83 % active threads (tc3d: 70 %). One elected
// thread streams, per plane, the x box (W x (RY+2) x (R+2): nodes -2 .. nn of the rows y0-1 .. y0+RY,
// slices z0-1 .. z0+R) and the b box with 4-D cp.async.bulk.tensor into an mbarrier ring, walking the
// CTA's (segment, plane) sequence NB-1 planes ahead across segment boundaries. Schedule: the strided
// tile groups of tv2d (common.cuh sched_next); a config-4 fine level has 17 x 17 tiles for 296 CTA slots,
// so the grid is trimmed to one CTA per tile column and every CTA marches its tile through all planes in
// step with its neighbours (halo boxes hit L2). Entries outside the domain carry zero element
// coefficients (the box reads there are finite: zero guard, zero pads, TMA zero fill, or a neighbouring
// row / slice / plane).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace st {
namespace t3r {

#ifndef ST_TC3R_R
#define ST_TC3R_R 5  // nodes per thread along x3 (R = 2: three CTAs per SM at <= 96 registers; R = 4, 5:
                     // two CTAs per SM at <= 144 registers)
#endif
constexpr int MAXT = 224;  // threads per CTA (7 warps)
constexpr int MAXREG = ST_TC3R_R <= 2 ? 96 : 128;  // three (R = 2) / two (R >= 3) CTAs per SM: at most
                                                   // 4 warps x 32 x 128 registers on an SMSP (16384)
template <int R> struct Cfg {
  static constexpr int NB = R <= 2 ? 4 : 3;  // ring depth (planes)
};

struct Lay {
  int RY;        // node rows (x2) per tile
  int W, Wb;     // x / b box widths (doubles, even)
  int XSZ, BSZ;  // ring slot sizes (doubles, multiples of 16)
  int CSZ;       // coefficient table (doubles, multiple of 16)
  int nty;       // tiles along x2
};

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

template <int R, int MODE, bool TRANS>
__global__ void __maxnreg__(MAXREG)
    tc3r_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmb, OpDesc op,
                double* __restrict__ y, double omega, long long wtot, int kchunk, Lay L) {
  constexpr bool NX = (MODE != MODE_JAC0);
  constexpr bool NBV = (MODE != MODE_APPLY);
  constexpr bool ND = (MODE == MODE_JAC || MODE == MODE_JAC0);
  constexpr int NB = Cfg<R>::NB;
  extern __shared__ __align__(128) double smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  double* xs = smem + 16;                      // [NB][XSZ]: [R+2 slices][RY+2 rows][W]
  double* bs = xs + (NX ? NB * L.XSZ : 0);     // [NB][BSZ]: [R slices][RY rows][Wb]
  // element coefficients (C_e, k~_e) of the tile's R+1 element layers z0-1 .. z0+R-1, rows y0-1 ..
  // y0+RY-1 and columns -1 .. nn-1 (zero outside the domain), filled once per segment: quadrant
  // qd = qx + 2 qy of the thread's column is entry [l][yr + qy][xi + qx]
  double2* ct = reinterpret_cast<double2*>(bs + (NBV ? NB * L.BSZ : 0));

  const Geom& g = op.g;
  const int t = threadIdx.x;
  const int n = g.n, nn = g.nn, pr = g.pr;
  const long long P = g.P, SS = (long long)pr * nn;  // plane / slice strides
  const int NP = g.nt + 1;
  const int W = L.W, SL = (L.RY + 2) * W, BSL = L.RY * L.Wb;
  const bool tin = t < L.RY * nn;  // threads of the last warp beyond the tile: idle (read row 0)
  const int xi = tin ? t % nn : 0, yr = tin ? t / nn : 0;
  const int xo = yr * W + xi + 1;  // (x-1, y-1) corner of the thread's window in slice 0
  const int bo = yr * L.Wb + xi;
  const unsigned xbytes = (unsigned)(W * (L.RY + 2) * (R + 2)) * 8u;
  const unsigned bbytes = (unsigned)(L.Wb * L.RY * R) * 8u;

  if (t == 0) {
#pragma unroll
    for (int k = 0; k < NB; ++k) mbar_init(&bar[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  pdl_wait();  // the previous kernel's writes are visible from here on

  const double sm = g.dx * g.dx * g.dx * (1.0 / 216.0);
  const double sk = g.dx * (1.0 / 36.0);
  const double t00 = op.Tm[0][0] * sk, t01 = op.Tm[0][1] * sk, t11 = op.Tm[1][1] * sk;
  const long long tiles = wtot / NP;

  // producer (thread 0): this CTA's (segment, plane) sequence, NB-1 planes ahead of the consumer.
  // The schedule state of producer and consumer lives in shared memory (only thread 0 advances it),
  // so it costs no registers in the plane loop.
  __shared__ Sched psc, csc;
  __shared__ long long ptile, ctile;
  __shared__ int pst[4], cst[3];  // producer: p0, p1, next plane, last plane; consumer: p0, p1, valid
  __shared__ bool pv;
  auto pnext = [&]() {
    long long tl;
    int a, b;
    pv = sched_next(psc, tl, a, b);
    ptile = tl;
    pst[0] = a;
    pst[1] = b;
    pst[2] = max(a - 1, 0);
    pst[3] = min(b, g.nt);
  };
  auto issue_next = [&](unsigned slot) {
    if (!pv) return;
    const int q = pst[2];
    const bool wb = NBV && q >= pst[0] && q < pst[1];
    mbar_expect_tx(&bar[slot], (NX ? xbytes : 0u) + (wb ? bbytes : 0u));
    const int cy = (int)(ptile % L.nty) * L.RY, cz = (int)(ptile / L.nty) * R;
    if (NX) tma4(xs + slot * L.XSZ, &tmx, &bar[slot], 0, cy, cz, q);
    if (wb) tma4(bs + slot * L.BSZ, &tmb, &bar[slot], 0, cy, cz, q);
    if ((pst[2] = q + 1) > pst[3]) pnext();
  };
  if (t == 0) {
    sched_init(psc, tiles, NP, kchunk);
    sched_init(csc, tiles, NP, kchunk);
    pnext();
    for (int k = 0; k < NB - 1; ++k) issue_next((unsigned)k);
  }

  unsigned cur = 0u, prv = NB - 1, phase = 0u;
  for (;;) {
    if (t == 0) {
      long long tl;
      int a, b;
      cst[2] = sched_next(csc, tl, a, b);
      ctile = tl;
      cst[0] = a;
      cst[1] = b;
    }
    __syncthreads();  // consumer segment published (and the previous segment's tail row done)
    if (!cst[2]) break;
    const long long tile = ctile;
    const int p0 = cst[0], p1 = cst[1];
    __syncthreads();  // every thread has read the segment before thread 0 advances it again
    const int qs = max(p0 - 1, 0), qe = min(p1, g.nt);
    const int y0 = (int)(tile % L.nty) * L.RY, z0 = (int)(tile / L.nty) * R;
    const int j = y0 + yr;

    {  // coefficient table of the segment's tile (the previous segment is done: barrier above)
      const int CW = nn + 1, CR = L.RY + 1;
      const int cnt = (R + 1) * CR * CW;
      for (int e = t; e < cnt; e += blockDim.x) {
        const int l = e / (CR * CW), rem = e - l * CR * CW;
        const int ex = rem % CW - 1, ey = y0 - 1 + rem / CW, ez = z0 - 1 + l;
        const bool v = ex >= 0 && ex < n && ey >= 0 && ey < n && ez >= 0 && ez < n;
        const double r = v ? __ldg(op.rho + ((long long)ez * n + ey) * n + ex) : 0.0;
        ct[e] = v ? make_double2(op.m.Cins + op.m.dC * powp(r, op.m.pc), op.m.kins + op.m.dk * powp(r, op.m.pk))
                  : make_double2(0.0, 0.0);
      }
    }
    __syncthreads();
    const double2* cth = ct + yr * (nn + 1) + xi;  // quadrant (0, 0) of layer 0
    const int CLS = (L.RY + 1) * (nn + 1);         // layer stride
    auto cload = [&](int l, double2 (&e)[4]) {
#pragma unroll
      for (int qd = 0; qd < 4; ++qd) e[qd] = cth[l * CLS + (qd >> 1) * (nn + 1) + (qd & 1)];
    };
    unsigned actm = 0u, patm = 0u;  // bit r: node r active / sink-patch node
    double odI[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int kz = z0 + r;
      const bool act = tin && j <= n && kz <= n;
      if (act) actm |= 1u << r;
      if (xi == 0 && j >= g.plo && j <= g.phi && kz >= g.plo && kz <= g.phi) patm |= 1u << r;
      double cs = 0.0, ks = 0.0;
      double2 e0[4], e1[4];
      cload(r, e0);
      cload(r + 1, e1);
#pragma unroll
      for (int qd = 0; qd < 4; ++qd) {
        cs += e0[qd].x + e1[qd].x;
        ks += e0[qd].y + e1[qd].y;
      }
      const double mc = 8.0 * sm * cs, kc = 12.0 * ks;  // diagonal: mass centre, stiffness centre (x sk in t..)
      odI[r] = (ND && act) ? omega / (mc + (t00 + t11) * kc) : 0.0;
    }

    double rowp[R], pend[R];
    double* yrow = y + (long long)(qs - 1) * P + (long long)z0 * SS + (long long)j * pr + xi;

    auto plane = [&](int q, auto first_tag) -> bool {
      constexpr bool FIRST = decltype(first_tag)::value;
      mbar_wait(&bar[cur], (phase >> cur) & 1u);
      phase ^= 1u << cur;
      double Mq[R], Kq[R];
#pragma unroll
      for (int r = 0; r < R; ++r) Mq[r] = Kq[r] = 0.0;
      if (NX && q + g.pg0 > 0) {
        const double* v0 = xs + cur * L.XSZ + xo;
        double2 eb[4], ea[4];  // coefficients of the layer below / above the current slice
#pragma unroll
        for (int s = 0; s < R + 2; ++s) {
#pragma unroll
          for (int qd = 0; qd < 4; ++qd) eb[qd] = ea[qd];
          if (s <= R) cload(s, ea);
          // keep the 9 loads of a slice next to their use: hoisting the loads of all R + 2 slices ahead
          // (ptxas' default) needs ~54 more registers and spills at the two-CTA register budget
          asm volatile("" ::: "memory");
          const double* a = v0 + s * SL;
          const double* b = a + W;
          const double* c = b + W;
          const double vmm = a[0], v0m = a[1], vpm = a[2];
          const double vm0 = b[0], v00 = b[1], vp0 = b[2];
          const double vmp = c[0], v0p = c[1], vpp = c[2];
          // 1D mass along x1 toward sx, rows dy = -1, 0, +1
          const double Amm = fma(2.0, v0m, vmm), Apm = fma(2.0, v0m, vpm);
          const double Am0 = fma(2.0, v00, vm0), Ap0 = fma(2.0, v00, vp0);
          const double Amp = fma(2.0, v0p, vmp), App = fma(2.0, v0p, vpp);
          double Bm[4], Bk[4];
          Bm[0] = fma(2.0, Am0, Amm);
          Bm[1] = fma(2.0, Ap0, Apm);
          Bm[2] = fma(2.0, Am0, Amp);
          Bm[3] = fma(2.0, Ap0, App);
          const double c4 = 4.0 * v00;
          const double em = c4 - vm0, ep = c4 - vp0;
          Bk[0] = fma(-2.0, vmm, em - v0m);
          Bk[1] = fma(-2.0, vpm, ep - v0m);
          Bk[2] = fma(-2.0, vmp, em - v0p);
          Bk[3] = fma(-2.0, vpp, ep - v0p);
          // slice s is the top slice of layer s-1 (nodes s-2 below, s-1 = this slice) and the bottom
          // slice of layer s (nodes s-1 = this slice, s above); node r sits on slice r + 1
          if (s >= 1) {
            double S = eb[0].x * Bm[0], G = eb[0].y * Bk[0], H = eb[0].y * Bm[0];
#pragma unroll
            for (int qd = 1; qd < 4; ++qd) {
              S = fma(eb[qd].x, Bm[qd], S);
              G = fma(eb[qd].y, Bk[qd], G);
              H = fma(eb[qd].y, Bm[qd], H);
            }
            if (s - 2 >= 0) {  // node below: M += S1, K += G1 - H1
              Mq[s - 2] += S;
              Kq[s - 2] += G - H;
            }
            if (s - 1 < R) {  // node on this slice: M += 2 S1, K += 2 G1 + H1
              Mq[s - 1] = fma(2.0, S, Mq[s - 1]);
              Kq[s - 1] += fma(2.0, G, H);
            }
          }
          if (s <= R) {
            double S = ea[0].x * Bm[0], G = ea[0].y * Bk[0], H = ea[0].y * Bm[0];
#pragma unroll
            for (int qd = 1; qd < 4; ++qd) {
              S = fma(ea[qd].x, Bm[qd], S);
              G = fma(ea[qd].y, Bk[qd], G);
              H = fma(ea[qd].y, Bm[qd], H);
            }
            if (s - 1 >= 0) {  // node on this slice: M += 2 S0, K += 2 G0 + H0
              Mq[s - 1] = fma(2.0, S, Mq[s - 1]);
              Kq[s - 1] += fma(2.0, G, H);
            }
            if (s < R) {  // node above: M += S0, K += G0 - H0
              Mq[s] += S;
              Kq[s] += G - H;
            }
          }
        }
      }
      if (!FIRST && q - 1 >= p0) {  // row q-1 complete
        const double* bp = bs + prv * L.BSZ + bo;
        const double* xp = xs + prv * L.XSZ + xo + SL + W + 1;  // centre of node r = 0, plane q-1
        if (q - 1 + g.pg0 == 0) {  // t = 0 plane: identity rows of the initial condition
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (!((actm >> r) & 1u)) continue;
            const double xc = NX ? xp[r * SL] : 0.0;
            const double bv = NBV ? bp[r * BSL] : 0.0;
            double o;
            if (MODE == MODE_APPLY) o = xc;
            else if (MODE == MODE_RESID) o = bv - xc;
            else if (MODE == MODE_JAC) o = fma(omega, bv - xc, xc);
            else o = omega * bv;
            yrow[r * SS] = o;
          }
        } else {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const double Ax = TRANS ? fma(-sm, Mq[r], fma(t01, Kq[r], rowp[r])) : fma(t01, Kq[r], rowp[r]);
            double o;
            if (MODE == MODE_APPLY) o = Ax;
            else if (MODE == MODE_RESID) o = bp[r * BSL] - Ax;
            else if (MODE == MODE_JAC) o = fma(odI[r], bp[r * BSL] - Ax, xp[r * SL]);
            else o = odI[r] * bp[r * BSL];
            if ((actm >> r) & 1u) yrow[r * SS] = ((patm >> r) & 1u) ? 0.0 : o;  // sink-patch rows: x = b = 0 there
          }
        }
      }
      // row q so far: pend (plane q-1's share: - M x_{q-1} (not for K^T) + t01 K x_{q-1}) + M x_q +
      // (t00 + t11) K x_q (the last plane has no layer above: t11 only); the segment's first row gets
      // the bottom part of layer q only (it is a reloaded row of the previous segment, or the t = 0 row)
      const double tk = q < g.nt ? t00 + t11 : t11;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        rowp[r] = FIRST ? t00 * Kq[r] : fma(sm, Mq[r], fma(tk, Kq[r], pend[r]));
        pend[r] = TRANS ? t01 * Kq[r] : fma(-sm, Mq[r], t01 * Kq[r]);
      }
      __syncthreads();  // slot of plane q-1 consumed by every thread
      if (t == 0) issue_next(prv);
      yrow += P;
      prv = cur;
      if (++cur == NB) cur = 0u;
      return q < qe;  // plane qe's slot (now prv) stays until the next plane's barrier: tail row
    };
    if (plane(qs, std::true_type{}))
      for (int q = qs + 1; plane(q, std::false_type{}); ++q) {
      }
    if (p1 == g.nt + 1) {  // last row: top part of layer nt-1 only
      const double* bp = bs + prv * L.BSZ + bo;
      const double* xp = xs + prv * L.XSZ + xo + SL + W + 1;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double cs = 0.0, ks = 0.0;  // last plane: no layer above it
        double2 e0[4], e1[4];
        cload(r, e0);
        cload(r + 1, e1);
#pragma unroll
        for (int qd = 0; qd < 4; ++qd) {
          cs += e0[qd].x + e1[qd].x;
          ks += e0[qd].y + e1[qd].y;
        }
        const double odT = (ND && ((actm >> r) & 1u)) ? omega / (8.0 * sm * cs + t11 * 12.0 * ks) : 0.0;
        const double Ax = rowp[r];
        double o;
        if (MODE == MODE_APPLY) o = Ax;
        else if (MODE == MODE_RESID) o = bp[r * BSL] - Ax;
        else if (MODE == MODE_JAC) o = fma(odT, bp[r * BSL] - Ax, xp[r * SL]);
        else o = odT * bp[r * BSL];
        if ((actm >> r) & 1u) yrow[r * SS] = ((patm >> r) & 1u) ? 0.0 : o;
      }
    }
  }
}

}  // namespace t3r

// ---------------------------------------------------------------------------------------
namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn_t3r() {
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

bool map4r(CUtensorMap* m, const void* base, const unsigned long long (&dims)[4], const unsigned long long (&str)[3],
           const unsigned (&box)[4]) {
  auto fn = encode_fn_t3r();
  if (!fn || ((uintptr_t)base & 15u)) return false;
  for (int d = 0; d < 3; ++d)
    if (str[d] & 15u) return false;
  for (int d = 0; d < 4; ++d)
    if (box[d] < 1 || box[d] > 256) return false;
  cuuint64_t dd[4] = {dims[0], dims[1], dims[2], dims[3]};
  cuuint64_t ss[3] = {str[0], str[1], str[2]};
  cuuint32_t bb[4] = {box[0], box[1], box[2], box[3]};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void*>(base), dd, ss, bb, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

constexpr int kR = ST_TC3R_R;

inline int round16(long long v) { return (int)((v + 15) / 16 * 16); }

// rows per tile: minimise the busiest SM's thread rows per plane, ceil(tiles / nsm) x threads per CTA
// (config 4, nn = 65: RY = 4, 17 x 17 tiles of 288 threads, two per SM)
int choose_ry(const Geom& g, int nsm) {
  const int ntz = (g.nn + kR - 1) / kR;
  int best = 0;
  long long bestc = 0;
  for (int RY = 1; RY <= g.nn && RY * g.nn <= t3r::MAXT; ++RY) {
    const long long nth = (RY * g.nn + 31) / 32 * 32;
    const long long tl = (long long)((g.nn + RY - 1) / RY) * ntz;
    const long long cost = (tl + nsm - 1) / nsm * nth;
    if (!best || cost < bestc) {
      best = RY;
      bestc = cost;
    }
  }
  return best;
}

t3r::Lay make_lay(const Geom& g, int RY) {
  t3r::Lay L{};
  L.RY = RY;
  L.W = (g.nn + 3 + 1) & ~1;  // nodes -2 .. nn (nn + 3 entries), even
  L.Wb = (g.nn + 1) & ~1;
  L.XSZ = round16((long long)L.W * (RY + 2) * (kR + 2));
  L.BSZ = round16((long long)L.Wb * RY * kR);
  L.CSZ = round16(2LL * (kR + 1) * (RY + 1) * (g.nn + 1));
  L.nty = (g.nn + RY - 1) / RY;
  return L;
}

template <int MODE, bool TRANS>
void lt3r(const CUtensorMap& mx, const CUtensorMap& mb, const OpDesc& op, const t3r::Lay& L, int nsm, double* y,
          double omega, cudaStream_t s) {
  using namespace t3r;
  const Geom& g = op.g;
  auto kern = tc3r_kernel<kR, MODE, TRANS>;
  constexpr bool NX = (MODE != MODE_JAC0), NBV = (MODE != MODE_APPLY);
  constexpr int NB = Cfg<kR>::NB;
  static bool attr = false;
  if (!attr) {
    attr = true;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    // two ~107 KB CTAs per SM need the largest shared-memory carve-out
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  }
  const int ntz = (g.nn + kR - 1) / kR;
  const int nth = (L.RY * g.nn + 31) / 32 * 32;
  const size_t bytes = sizeof(double) * (16 + (size_t)NB * ((NX ? L.XSZ : 0) + (NBV ? L.BSZ : 0)) + L.CSZ);
  // occupancy of this (block, smem) shape: cached for the last shape queried
  static int last_nth = -1, last_res = 1;
  static size_t last_bytes = 0;
  if (nth != last_nth || bytes != last_bytes) {
    int res = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res, kern, nth, bytes);
    last_nth = nth;
    last_bytes = bytes;
    last_res = res < 1 ? 1 : res;
  }
  const long long tiles = (long long)L.nty * ntz;
  const int NPl = g.nt + 1;
  const long long wtot = tiles * NPl;
  long long grid = persistent_grid(op, nsm, last_res, wtot);
  // one CTA per tile column when the tiles nearly fill the wave (config 4: 289 tiles, 296 slots):
  // every CTA marches its column through all planes in step with its neighbours; a large partial
  // group is trimmed to equal full groups as in tv2d
  if (tiles * 2 >= grid) {
    const long long part = tiles % grid;
    if (tiles <= grid || op.max_ctas < 0 || (op.max_ctas == 0 && part * 5 >= grid * 2)) {
      const long long groups = (tiles + grid - 1) / grid;
      grid = (tiles + groups - 1) / groups;
    }
  }
  const int kch = chunk_planes(op, NPl, NPl);
  launch_pdl(kern, dim3((unsigned)grid), dim3(nth), bytes, s, mx, mb, op, y, omega, wtot, kch, L);
}
}  // namespace

// Masked (eliminated) operator on the (3+1)D fine level of a time-constant design; false if not
// covered (the tc3d kernels then run).
bool launch_op_tc3r(const OpDesc& op, int mode, bool trans, bool mask, const double* x, const double* b, double* y,
                    double omega, cudaStream_t s) {
#ifdef ST_TC3R_OFF
  return false;  // A/B builds: the tc3d stencil kernel on the fine level
#endif
  if (op.g.walls) return false;  // Example 2's cold walls: the generic kernels (is_cons)
  const Geom& g = op.g;
  if (g.sd != 3 || !mask || !(op.form == FORM_RHO && op.rho_tc)) return false;
  if (g.nn * 2 > t3r::MAXT || g.nt < 1) return false;
  if (op.U[0][0] != 0.0 || op.U[0][1] != 0.0 || op.U[1][0] != -1.0 || op.U[1][1] != 1.0) return false;
  if (op.Tm[0][1] != op.Tm[1][0]) return false;
  CUtensorMap mx{}, mb{};
  const unsigned long long nn = g.nn, pr = g.pr;
  const unsigned long long str[3] = {pr * 8, pr * nn * 8, (unsigned long long)g.P * 8};
  const bool nx = (mode != MODE_JAC0), nbv = (mode != MODE_APPLY);
  // rows per tile as the launcher chooses them (the box shapes depend on it)
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm < 1) nsm = 148;
  }
  const t3r::Lay L = make_lay(g, choose_ry(g, nsm));
  // x: based one slice + one row + 2 entries before the data (zeroed front guard): box coordinate
  // (0, y0, z0, q) is node (-2, y0 - 1, z0 - 1) of plane q
  const long long shift = (long long)pr * nn + pr + 2;
  if (nx) {
    const unsigned long long dims[4] = {pr + 2, nn + 1, nn + 1, (unsigned long long)g.nt + 1};
    const unsigned box[4] = {(unsigned)L.W, (unsigned)L.RY + 2, (unsigned)kR + 2, 1};
    if (!map4r(&mx, x - shift, dims, str, box)) return false;
  }
  if (nbv) {
    const unsigned long long dims[4] = {nn, nn, nn, (unsigned long long)g.nt + 1};
    const unsigned box[4] = {(unsigned)L.Wb, (unsigned)L.RY, (unsigned)kR, 1};
    if (!map4r(&mb, b, dims, str, box)) return false;
  }
#define C4(M)                                              \
  case M:                                                  \
    if (trans) lt3r<M, true>(mx, mb, op, L, nsm, y, omega, s);     \
    else lt3r<M, false>(mx, mb, op, L, nsm, y, omega, s);          \
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
