// fast2d.cu — bandwidth-oriented (2+1)D level operator for sm_100a.
//
// Same operator and modes as op_kernel in ops.cu (see the algebra there), specialised for
// the forms that dominate the V-cycle bytes:
//   * RHO (fine level, matrix-free from rho), time-constant (TC) or space-time (TV) design;
//   * MK stored stencils of time-constant levels (nl = 1).
// Design:
//   * CTA = 128 threads owns a 32 x 8 node tile and marches through a chunk of time planes;
//     each thread owns 1 x RY(=2) nodes.
//   * x planes stream through a 5-slot shared-memory ring filled with cp.async (8-byte,
//     zero-fill for the halo outside the domain and for Dirichlet nodes: the mask costs no
//     instruction in the inner loop); 3 planes in flight.
//   * TC: the 9-point M and K weights of the thread's nodes are built once into registers;
//     every plane costs 2 stencil applies (M x_q, K x_q) and the layer combination uses the
//     previous plane's results (carry). TV: the rho tile of the layer streams through its
//     own ring; C, k~ are evaluated once per element in shared memory, 4 applies per plane.
#include "common.cuh"
#include "kernels.h"

namespace st {
#ifndef ST_CUNI_MINB
#define ST_CUNI_MINB 3
#endif
namespace f2 {

constexpr int TX = 32, TYT = 4, RY = 2, TY = TYT * RY;   // node tile 32 x 8
constexpr int HX = TX + 2, HY = TY + 2, PT = HX * HY;    // plane tile with halo: 34 x 10
constexpr int EX = TX + 1, EY = TY + 1, ET = EX * EY;    // element tile: 33 x 9
constexpr int NB = 6;                                     // ring slots (NB-2 planes in flight)
constexpr int NTH = TX * TYT;
constexpr int BT = TX * TY;                               // interior (b) tile

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// apply 9-point weights w to the 3x3 neighbourhood (rows s0..s0+2, cols 0..2) of nb
__device__ __forceinline__ double ap9(const double* w, const double (&nb)[RY + 2][3], int r) {
  double a = w[4] * nb[r + 1][1];
  a = fma(w[0], nb[r][0], a);
  a = fma(w[1], nb[r][1], a);
  a = fma(w[2], nb[r][2], a);
  a = fma(w[3], nb[r + 1][0], a);
  a = fma(w[5], nb[r + 1][2], a);
  a = fma(w[6], nb[r + 2][0], a);
  a = fma(w[7], nb[r + 2][1], a);
  a = fma(w[8], nb[r + 2][2], a);
  return a;
}

// integer-scaled 9-point weights from the 4 element coefficients around a node
// (SW, SE, NW, NE); M: [1,2,1;2,4,2;1,2,1]-pattern sums, K: 6x the Q1 stiffness weights
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

struct Fac {  // layer time factors with the spatial scale folded in
  double u00, u01, u10, u11, t00, t01, t10, t11;
};

template <bool TRANS> __device__ __forceinline__ Fac make_fac(const OpDesc& op, double sm, double sk) {
  Fac f;
  if (!TRANS) {
    f.u00 = op.U[0][0] * sm; f.u01 = op.U[0][1] * sm; f.u10 = op.U[1][0] * sm; f.u11 = op.U[1][1] * sm;
    f.t00 = op.Tm[0][0] * sk; f.t01 = op.Tm[0][1] * sk; f.t10 = op.Tm[1][0] * sk; f.t11 = op.Tm[1][1] * sk;
  } else {  // block transpose: (a,b) -> (b,a)
    f.u00 = op.U[0][0] * sm; f.u01 = op.U[1][0] * sm; f.u10 = op.U[0][1] * sm; f.u11 = op.U[1][1] * sm;
    f.t00 = op.Tm[0][0] * sk; f.t01 = op.Tm[1][0] * sk; f.t10 = op.Tm[0][1] * sk; f.t11 = op.Tm[1][1] * sk;
  }
  return f;
}

// SRC: 0 = RHO, 1 = MK stored (TC only). CUNI: uniform capacity (C_ins = C_con) on the RHO
// time-constant level: the spatial mass is the tensor product of the 1D assembled masses,
// M = C dx^2/36 (My (x) Mx) with 1D patterns [1,4,1] (interior), [0,2,1] / [1,2,0] (ends), applied
// separably; only the 9 stiffness weights are held in registers.
template <bool TC, int SRC, bool CUNI, int MODE, bool TRANS, bool MASK>
__global__ void __launch_bounds__(NTH, CUNI ? ST_CUNI_MINB : 3) op2d_kernel(OpDesc op, const double* __restrict__ x,
                                                      const double* __restrict__ b, double* __restrict__ y,
                                                      double omega, int chunk) {
  constexpr bool TVR = (!TC) && SRC == 0;
  constexpr bool NX = (MODE != MODE_JAC0);   // reads x
  constexpr bool NBV = (MODE != MODE_APPLY); // reads b
  __shared__ __align__(16) double xs[NX ? NB : 1][NX ? PT : 1];
  __shared__ __align__(16) double bs[NBV ? NB : 1][NBV ? BT : 1];
  __shared__ __align__(16) double rs[TVR ? NB : 1][TVR ? ET : 1];
  __shared__ double cC[TVR ? ET : 1], cK[TVR ? ET : 1];

  const Geom& g = op.g;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int p0 = blockIdx.z * chunk;
  if (p0 > g.nt) return;
  const int p1 = min(p0 + chunk, g.nt + 1);
  const int qs = max(p0 - 1, 0), qe = min(p1, g.nt);
  const int i = x0 + tx;
  const int n = g.n, nn = g.nn, pr = g.pr;
  const long long P = g.P;
  const double sm = (SRC == 0) ? g.dx * g.dx * (1.0 / 36.0) * (CUNI ? op.m.Cins : 1.0) : 1.0;
  const double sk = (SRC == 0) ? (1.0 / 6.0) : 1.0;
  const Fac F = make_fac<TRANS>(op, sm, sk);
  int jr[RY];
  bool act[RY];
#pragma unroll
  for (int r = 0; r < RY; ++r) {
    jr[r] = y0 + ty * RY + r;
    act[r] = (i <= n) && (jr[r] <= n);
  }

  // --- per-thread copy descriptors (computed once; every plane only bumps a pointer) ---
  constexpr int XPT = (PT + NTH - 1) / NTH;   // x elements per thread (3)
  constexpr int BPT = (BT + NTH - 1) / NTH;   // b elements per thread (2)
  constexpr int RPT = (ET + NTH - 1) / NTH;   // rho elements per thread (3)
  int xoff[XPT], xsm[XPT];
  unsigned xval = 0u, xpatch = 0u;
#pragma unroll
  for (int k = 0; k < XPT; ++k) {
    int e = tid + k * NTH;
    int ly = e / HX, lx = e - ly * HX;
    int gi = x0 - 1 + lx, gj = y0 - 1 + ly;
    bool v = (e < PT) && (gi >= 0 && gi <= n && gj >= 0 && gj <= n);
    xoff[k] = v ? gj * pr + gi : 0;
    xsm[k] = e < PT ? e : 0;
    if (v) xval |= 1u << k;
    if (v && gi == 0 && gj >= g.plo && gj <= g.phi) xpatch |= 1u << k;
  }
  int boff[BPT];
  unsigned bval = 0u;
#pragma unroll
  for (int k = 0; k < BPT; ++k) {
    int e = tid + k * NTH;
    int ly = e / TX, lx = e - ly * TX;
    int gi = x0 + lx, gj = y0 + ly;
    bool v = (e < BT) && gi <= n && gj <= n;
    boff[k] = v ? gj * pr + gi : 0;
    if (v) bval |= 1u << k;
  }
  int roff[RPT];
  unsigned rval = 0u;
  if (TVR) {
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      int e = tid + k * NTH;
      int ly = e / EX, lx = e - ly * EX;
      int gi = x0 - 1 + lx, gj = y0 - 1 + ly;
      bool v = (e < ET) && gi >= 0 && gi < n && gj >= 0 && gj < n;
      roff[k] = v ? gj * n + gi : 0;
      if (v) rval |= 1u << k;
    }
  }

  // --- plane / layer loaders -------------------------------------------------------
  auto issue_plane = [&](int q, int slot, const double* xq, const double* bq) {
    if (NX) {
      double* dst = xs[slot];
      const double* src = xq;
      unsigned vm = xval & (MASK ? (q + g.pg0 == 0 ? 0u : ~xpatch) : ~0u);
#pragma unroll
      for (int k = 0; k < XPT; ++k)
        if (k < XPT - 1 || tid + k * NTH < PT) cp_async8(&dst[xsm[k]], src + xoff[k], (vm >> k) & 1u);
    }
    if (NBV && q >= p0 && q < p1) {  // b of row q (interior tile)
      double* dst = bs[slot];
      const double* src = bq;
#pragma unroll
      for (int k = 0; k < BPT; ++k) cp_async8(&dst[tid + k * NTH], src + boff[k], (bval >> k) & 1u);
    }
    if (TVR) {
      int tau = q - 1;  // layer needed when plane q arrives
      if (tau >= qs) {
        double* rd = rs[slot];
        const double* rsrc = op.rho + (long long)tau * n * n;
#pragma unroll
        for (int k = 0; k < RPT; ++k)
          if (k < RPT - 1 || tid + k * NTH < ET) cp_async8(&rd[tid + k * NTH], rsrc + roff[k], (rval >> k) & 1u);
      }
    }
  };

  // --- time-constant weights in registers ------------------------------------------
  double wM[CUNI ? 1 : RY][9], wK[RY][9];
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
          int a = i - 1 + (e & 1), bb = jr[r] - 1 + (e >> 1);
          bool v = act[r] && a >= 0 && a < n && bb >= 0 && bb < n;
          double rho = v ? __ldg(op.rho + (long long)bb * n + a) : 0.0;
          ce[e] = v ? op.m.Cins + op.m.dC * powp(rho, op.m.pc) : 0.0;
          ke[e] = v ? op.m.kins + op.m.dk * powp(rho, op.m.pk) : 0.0;
        }
        if (!CUNI) wM_from(ce[0], ce[1], ce[2], ce[3], wM[r]);
        wK_from(ke[0], ke[1], ke[2], ke[3], wK[r]);
      } else {
        // stored symmetric stencils: own forward coefs (k >= 4) + neighbours' mirrored ones
        const long long pn = act[r] ? (long long)jr[r] * pr + i : 0;
        const double* Mb = op.st;
        const double* Kb = op.st + 5 * P;
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          int dx = (k % 3) - 1, dy = (k / 3) - 1;
          if (k >= 4) {
            wM[r][k] = act[r] ? __ldg(Mb + (k - 4) * P + pn) : 0.0;
            wK[r][k] = act[r] ? __ldg(Kb + (k - 4) * P + pn) : 0.0;
          } else {
            int ni = i + dx, nj = jr[r] + dy;
            bool v = act[r] && ni >= 0 && ni <= n && nj >= 0 && nj <= n;
            long long q = v ? (long long)nj * pr + ni : 0;
            wM[r][k] = v ? __ldg(Mb + (8 - k - 4) * P + q) : 0.0;
            wK[r][k] = v ? __ldg(Kb + (8 - k - 4) * P + q) : 0.0;
          }
        }
      }
    }
  }

  // diagonal parts (TC: loop invariant)
  double odI[RY], odT[RY];  // omega / D for interior rows and for the last row (top part only)
  if (TC && (MODE == MODE_JAC || MODE == MODE_JAC0)) {
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      const double mc = CUNI ? wx[1] * wy[r][1] : wM[CUNI ? 0 : r][4];
      double db = F.u00 * mc + F.t00 * wK[r][4];
      double dt = F.u11 * mc + F.t11 * wK[r][4];
      odI[r] = act[r] ? omega / (db + dt) : 0.0;
      odT[r] = act[r] ? omega / dt : 0.0;
    }
  }

  // --- prologue: NB-2 planes in flight -----------------------------------------------
#pragma unroll
  for (int k = 0; k < NB - 2; ++k) {
    int q = qs + k;
    if (q <= qe) issue_plane(q, q % NB, x + (long long)q * P, b + (long long)q * P);
    cp_commit();
  }
  // running plane pointers of the next plane to issue (qs + NB - 2)
  const double* xnext = x + (long long)(qs + NB - 2) * P;
  const double* bnext = b + (long long)(qs + NB - 2) * P;
  // ring slots: cur = slot of plane q, prv = slot of plane q-1, nxt = slot of plane q+NB-2
  int cur = qs % NB;
  int prv = (cur + NB - 1) % NB;
  int nxt = (cur + NB - 2) % NB;
  const int nodeoff0 = jr[0] * pr + i;
  double* yrow = y + (long long)(qs - 1) * P + nodeoff0;   // row q-1 of the current iteration

  double Mprev[RY], Kprev[RY], carry[RY], dcarry[RY];
#pragma unroll
  for (int r = 0; r < RY; ++r) { Mprev[r] = Kprev[r] = carry[r] = dcarry[r] = 0.0; }

  // out_row: od = omega / D (JAC, JAC0); slot = ring slot of plane p
  const bool patchr[RY] = {MASK && i == 0 && jr[0] >= g.plo && jr[0] <= g.phi,
                           MASK && i == 0 && jr[1] >= g.plo && jr[1] <= g.phi};
  auto out_row = [&](int p, int slot, int r, double Ax, double od) {
    if (p < p0 || p >= p1 || !act[r]) return;
    const long long gi = (long long)p * P + nodeoff0 + r * pr;
    const bool cons = MASK && (p + g.pg0 == 0 || patchr[r]);
    double* yo = yrow + r * pr;
    const double bv = NBV ? bs[slot][(ty * RY + r) * TX + tx] : 0.0;
    double o;
    if (MODE == MODE_APPLY) {
      o = cons ? __ldg(x + gi) : Ax;
    } else if (MODE == MODE_RESID) {
      o = bv - (cons ? __ldg(x + gi) : Ax);
    } else if (MODE == MODE_JAC) {
      double xc = xs[slot][(ty * RY + r + 1) * HX + tx + 1];
      if (cons) { xc = __ldg(x + gi); Ax = xc; od = omega; }
      o = fma(od, bv - Ax, xc);
    } else {  // JAC0
      o = (cons ? omega : od) * bv;
    }
    *yo = o;
  };

  for (int q = qs; q <= qe; ++q) {
    cp_wait<NB - 3>();
    if (TVR) {
      // convert the layer (q-1) rho tile this thread copied into C, k~ (zero outside)
      __syncthreads();  // previous iteration finished reading cC / cK
      int tau = q - 1;
      if (tau >= qs) {
        const double* rd = rs[cur];
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
          const int e = tid + k * NTH;
          if (k < RPT - 1 || e < ET) {
            const bool v = (rval >> k) & 1u;
            const double rho = rd[e];
            cC[e] = v ? op.m.Cins + op.m.dC * powp(rho, op.m.pc) : 0.0;
            cK[e] = v ? op.m.kins + op.m.dk * powp(rho, op.m.pk) : 0.0;
          }
        }
      }
    }
    __syncthreads();
    // refill: plane q + NB - 2 into the slot of plane q - 2
    {
      int qn = q + NB - 2;
      if (qn <= qe) issue_plane(qn, nxt, xnext, bnext);
      cp_commit();
      xnext += P;
      bnext += P;
    }
    const int prow = q - 1;  // row completed in this iteration
    // gather 3 x (RY+2) neighbourhood of plane q
    double nbq[RY + 2][3];
    if (NX) {
      const double* t = xs[cur] + (ty * RY) * HX + tx;
#pragma unroll
      for (int s = 0; s < RY + 2; ++s)
#pragma unroll
        for (int c = 0; c < 3; ++c) nbq[s][c] = t[s * HX + c];
    }
    if (TC) {
      double rsum[RY + 2];
      if (CUNI && NX) {
#pragma unroll
        for (int s2 = 0; s2 < RY + 2; ++s2) rsum[s2] = fma(wx[0], nbq[s2][0], fma(wx[1], nbq[s2][1], wx[2] * nbq[s2][2]));
      }
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        if (!NX) {
          if (q > qs) out_row(prow, prv, r, 0.0, odI[r]);
          continue;
        }
        double Mq = CUNI ? fma(wy[r][0], rsum[r], fma(wy[r][1], rsum[r + 1], wy[r][2] * rsum[r + 2]))
                         : ap9(wM[CUNI ? 0 : r], nbq, r);
        double Kq = ap9(wK[r], nbq, r);
        if (q > qs) {  // layer tau = q-1: planes q-1 (prev) and q
          double bot = F.u00 * Mprev[r] + F.u01 * Mq + F.t00 * Kprev[r] + F.t01 * Kq;
          double top = F.u10 * Mprev[r] + F.u11 * Mq + F.t10 * Kprev[r] + F.t11 * Kq;
          out_row(prow, prv, r, carry[r] + bot, odI[r]);
          carry[r] = top;
        }
        Mprev[r] = Mq;
        Kprev[r] = Kq;
      }
    } else {
      if (q > qs) {
        double nbp[RY + 2][3];
        if (NX) {
          const double* t = xs[prv] + (ty * RY) * HX + tx;
#pragma unroll
          for (int s = 0; s < RY + 2; ++s)
#pragma unroll
            for (int c = 0; c < 3; ++c) nbp[s][c] = t[s * HX + c];
        }
        // element coefficients of the thread's column: rows s = 0..RY, cols W (tx), E (tx+1)
        double cw[RY + 1], ckw[RY + 1], ce_[RY + 1], cke[RY + 1];
#pragma unroll
        for (int s = 0; s <= RY; ++s) {
          int e = (ty * RY + s) * EX + tx;
          cw[s] = cC[e]; ce_[s] = cC[e + 1];
          ckw[s] = cK[e]; cke[s] = cK[e + 1];
        }
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          double w1[9], w2[9];
          wM_from(cw[r], ce_[r], cw[r + 1], ce_[r + 1], w1);
          wK_from(ckw[r], cke[r], ckw[r + 1], cke[r + 1], w2);
          double bot = 0.0, top = 0.0;
          if (NX) {
            double Mb = ap9(w1, nbp, r), Mt = ap9(w1, nbq, r);
            double Kb = ap9(w2, nbp, r), Kt = ap9(w2, nbq, r);
            bot = F.u00 * Mb + F.u01 * Mt + F.t00 * Kb + F.t01 * Kt;
            top = F.u10 * Mb + F.u11 * Mt + F.t10 * Kb + F.t11 * Kt;
          }
          double db = F.u00 * w1[4] + F.t00 * w2[4];
          double dt = F.u11 * w1[4] + F.t11 * w2[4];
          double od = (MODE == MODE_JAC || MODE == MODE_JAC0) && act[r] ? omega / (dcarry[r] + db) : 0.0;
          out_row(prow, prv, r, carry[r] + bot, od);
          carry[r] = top;
          dcarry[r] = dt;
        }
      }
    }
    // ROTATE
    yrow += P;
    prv = cur;
    cur = (cur + 1 == NB) ? 0 : cur + 1;
    nxt = (nxt + 1 == NB) ? 0 : nxt + 1;
  }
  // (ring slots rotate at the end of every iteration, see ROTATE)
  // last row nt: only the top part of layer nt-1
  if (p1 == g.nt + 1) {
    const int p = g.nt;
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      double od = 0.0;
      if (MODE == MODE_JAC || MODE == MODE_JAC0) od = TC ? odT[r] : (act[r] ? omega / dcarry[r] : 0.0);
      out_row(p, prv, r, carry[r], od);
    }
  }
  cp_wait<0>();
}

}  // namespace f2

static int choose_chunk2(const Geom& g, long long tiles) {
  // ~4 waves of CTAs over 148 SMs x 3 resident CTAs; small levels: short chunks so that all
  // planes proceed in parallel (latency), large levels: long chunks (1 extra plane per chunk)
  long long target = 148LL * 3 * 4;
  long long chunks = (target + tiles - 1) / tiles;
  if (chunks > g.nt + 1) chunks = g.nt + 1;
  if (chunks < 1) chunks = 1;
  return (int)((g.nt + 1 + chunks - 1) / chunks);
}

template <bool TC, int SRC, bool CUNI, int MODE, bool TRANS, bool MASK>
static void l2d(const OpDesc& op, const double* x, const double* b, double* y, double omega, cudaStream_t s) {
  const Geom& g = op.g;
  dim3 blk(f2::TX, f2::TYT, 1);
  long long tx = (g.nn + f2::TX - 1) / f2::TX, ty = (g.nn + f2::TY - 1) / f2::TY;
  int chunk = choose_chunk2(g, tx * ty);
  dim3 grd((unsigned)tx, (unsigned)ty, (unsigned)((g.nt + 1 + chunk - 1) / chunk));
  f2::op2d_kernel<TC, SRC, CUNI, MODE, TRANS, MASK><<<grd, blk, 0, s>>>(op, x, b, y, omega, chunk);
}

template <bool TC, int SRC, bool CUNI>
static void l2d_modes(const OpDesc& op, int mode, bool trans, bool mask, const double* x, const double* b, double* y,
                      double omega, cudaStream_t s) {
  if (!mask) {
    if (trans) l2d<TC, SRC, CUNI, MODE_APPLY, true, false>(op, x, b, y, omega, s);
    else l2d<TC, SRC, CUNI, MODE_APPLY, false, false>(op, x, b, y, omega, s);
    return;
  }
#define C2(M)                                                             \
  case M:                                                                 \
    if (trans) l2d<TC, SRC, CUNI, M, true, true>(op, x, b, y, omega, s);  \
    else l2d<TC, SRC, CUNI, M, false, true>(op, x, b, y, omega, s);       \
    break;
  switch (mode) {
    C2(MODE_APPLY)
    C2(MODE_RESID)
    C2(MODE_JAC)
    C2(MODE_JAC0)
  }
#undef C2
}

// returns false when the fast path does not cover the operator
bool launch_op_fast2d(const OpDesc& op, int mode, bool trans, bool mask, const double* x, const double* b, double* y,
                      double omega, cudaStream_t s) {
  if (op.g.walls) return false;  // Example 2's cold walls: the generic kernels (is_cons)
  if (op.g.sd != 2) return false;
  if (mode == MODE_JAC0 && !mask) return false;
  if (op.form == FORM_RHO) {
    const bool cuni = (op.m.dC == 0.0);
    if (op.rho_tc && cuni) l2d_modes<true, 0, true>(op, mode, trans, mask, x, b, y, omega, s);
    else if (op.rho_tc) l2d_modes<true, 0, false>(op, mode, trans, mask, x, b, y, omega, s);
    else l2d_modes<false, 0, false>(op, mode, trans, mask, x, b, y, omega, s);
    return true;
  }
  if (op.form == FORM_MK && !op.tvl) {
    l2d_modes<true, 1, false>(op, mode, trans, mask, x, b, y, omega, s);
    return true;
  }
  return false;
}

}  // namespace st
