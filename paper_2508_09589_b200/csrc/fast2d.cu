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
namespace f2 {

constexpr int TX = 32, TYT = 4, RY = 2, TY = TYT * RY;   // node tile 32 x 8
constexpr int HX = TX + 2, HY = TY + 2, PT = HX * HY;    // plane tile with halo: 34 x 10
constexpr int EX = TX + 1, EY = TY + 1, ET = EX * EY;    // element tile: 33 x 9
constexpr int NB = 5;                                     // ring slots
constexpr int NTH = TX * TYT;

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

// SRC: 0 = RHO, 1 = MK stored (TC only)
template <bool TC, int SRC, int MODE, bool TRANS, bool MASK>
__global__ void __launch_bounds__(NTH, 3) op2d_kernel(OpDesc op, const double* __restrict__ x,
                                                      const double* __restrict__ b, double* __restrict__ y,
                                                      double omega, int chunk) {
  constexpr bool TVR = (!TC) && SRC == 0;
  __shared__ __align__(16) double xs[NB][PT];
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
  const int n = g.n, nn = g.nn;
  const long long P = g.P;
  const double sm = (SRC == 0) ? g.dx * g.dx * (1.0 / 36.0) : 1.0;
  const double sk = (SRC == 0) ? (1.0 / 6.0) : 1.0;
  const Fac F = make_fac<TRANS>(op, sm, sk);
  int jr[RY];
  bool act[RY];
#pragma unroll
  for (int r = 0; r < RY; ++r) {
    jr[r] = y0 + ty * RY + r;
    act[r] = (i <= n) && (jr[r] <= n);
  }

  // --- plane / layer loaders -------------------------------------------------------
  auto issue_plane = [&](int q) {
    double* dst = xs[q % NB];
    const double* src = x + (long long)q * P;
    for (int e = tid; e < PT; e += NTH) {
      int ly = e / HX, lx = e - ly * HX;
      int gi = x0 - 1 + lx, gj = y0 - 1 + ly;
      bool v = (gi >= 0 && gi <= n && gj >= 0 && gj <= n);
      if (MASK && v && (q == 0 || (gi == 0 && gj >= g.plo && gj <= g.phi))) v = false;
      const double* s = v ? src + (long long)gj * nn + gi : x;
      cp_async8(&dst[e], s, v);
    }
    if (TVR) {
      int tau = q - 1;  // layer needed when plane q arrives
      if (tau >= qs) {
        double* rd = rs[q % NB];
        const double* rsrc = op.rho + (long long)tau * n * n;
        for (int e = tid; e < ET; e += NTH) {
          int ly = e / EX, lx = e - ly * EX;
          int gi = x0 - 1 + lx, gj = y0 - 1 + ly;
          bool v = (gi >= 0 && gi < n && gj >= 0 && gj < n);
          const double* s = v ? rsrc + (long long)gj * n + gi : op.rho;
          cp_async8(&rd[e], s, v);
        }
      }
    }
  };

  // --- time-constant weights in registers ------------------------------------------
  double wM[RY][9], wK[RY][9];
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
        wM_from(ce[0], ce[1], ce[2], ce[3], wM[r]);
        wK_from(ke[0], ke[1], ke[2], ke[3], wK[r]);
      } else {
        // stored symmetric stencils: own forward coefs (k >= 4) + neighbours' mirrored ones
        const long long pn = act[r] ? (long long)jr[r] * nn + i : 0;
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
            long long q = v ? (long long)nj * nn + ni : 0;
            wM[r][k] = v ? __ldg(Mb + (8 - k - 4) * P + q) : 0.0;
            wK[r][k] = v ? __ldg(Kb + (8 - k - 4) * P + q) : 0.0;
          }
        }
      }
    }
  }

  // diagonal parts (TC: loop invariant)
  double dbotC[RY], dtopC[RY];
  if (TC) {
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      dbotC[r] = F.u00 * wM[r][4] + F.t00 * wK[r][4];
      dtopC[r] = F.u11 * wM[r][4] + F.t11 * wK[r][4];
    }
  }

  // --- prologue: NB-2 planes in flight -----------------------------------------------
#pragma unroll
  for (int k = 0; k < NB - 2; ++k) {
    int q = qs + k;
    if (q <= qe) issue_plane(q);
    cp_commit();
  }

  double Mprev[RY], Kprev[RY], carry[RY], dcarry[RY], bnext[RY];
#pragma unroll
  for (int r = 0; r < RY; ++r) { Mprev[r] = Kprev[r] = carry[r] = dcarry[r] = 0.0; bnext[r] = 0.0; }

  auto out_row = [&](int p, int r, double Ax, double D) {
    if (p < p0 || p >= p1 || !act[r]) return;
    const long long gi = (long long)p * P + (long long)jr[r] * nn + i;
    const bool cons = MASK && (p == 0 || (i == 0 && jr[r] >= g.plo && jr[r] <= g.phi));
    double o;
    if (MODE == MODE_APPLY) {
      o = cons ? __ldg(x + gi) : Ax;
    } else if (MODE == MODE_RESID) {
      o = bnext[r] - (cons ? __ldg(x + gi) : Ax);
    } else {  // JAC
      double xc = xs[p % NB][(ty * RY + r + 1) * HX + tx + 1];
      if (cons) { xc = __ldg(x + gi); Ax = xc; D = 1.0; }
      o = xc + omega * (bnext[r] - Ax) / D;
    }
    y[gi] = o;
  };

  for (int q = qs; q <= qe; ++q) {
    cp_wait<NB - 3>();
    if (TVR) {
      // convert the layer (q-1) rho tile this thread copied into C, k~ (zero outside)
      __syncthreads();  // previous iteration finished reading cC / cK
      int tau = q - 1;
      if (tau >= qs) {
        const double* rd = rs[q % NB];
        for (int e = tid; e < ET; e += NTH) {
          int ly = e / EX, lx = e - ly * EX;
          int gi = x0 - 1 + lx, gj = y0 - 1 + ly;
          bool v = (gi >= 0 && gi < n && gj >= 0 && gj < n);
          double rho = rd[e];
          cC[e] = v ? op.m.Cins + op.m.dC * powp(rho, op.m.pc) : 0.0;
          cK[e] = v ? op.m.kins + op.m.dk * powp(rho, op.m.pk) : 0.0;
        }
      }
    }
    __syncthreads();
    // refill: plane q + NB - 2 into the slot of plane q - 2
    {
      int qn = q + NB - 2;
      if (qn <= qe) issue_plane(qn);
      cp_commit();
    }
    // b for the row output in this iteration (row q-1) — RESID/JAC
    const int prow = q - 1;
    if (MODE == MODE_RESID || MODE == MODE_JAC) {
#pragma unroll
      for (int r = 0; r < RY; ++r)
        bnext[r] = (act[r] && prow >= p0 && prow < p1) ? __ldg(b + (long long)prow * P + (long long)jr[r] * nn + i) : 0.0;
    }
    // gather 3 x (RY+2) neighbourhood of plane q
    double nbq[RY + 2][3];
    {
      const double* t = xs[q % NB] + (ty * RY) * HX + tx;
#pragma unroll
      for (int s = 0; s < RY + 2; ++s)
#pragma unroll
        for (int c = 0; c < 3; ++c) nbq[s][c] = t[s * HX + c];
    }
    if (TC) {
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        double Mq = ap9(wM[r], nbq, r), Kq = ap9(wK[r], nbq, r);
        if (q > qs) {  // layer tau = q-1: planes q-1 (prev) and q
          double bot = F.u00 * Mprev[r] + F.u01 * Mq + F.t00 * Kprev[r] + F.t01 * Kq;
          double top = F.u10 * Mprev[r] + F.u11 * Mq + F.t10 * Kprev[r] + F.t11 * Kq;
          double D = (prow >= 1 ? dtopC[r] : 0.0) + dbotC[r];
          out_row(prow, r, carry[r] + bot, D);
          carry[r] = top;
        }
        Mprev[r] = Mq;
        Kprev[r] = Kq;
      }
    } else {
      if (q > qs) {
        double nbp[RY + 2][3];
        const double* t = xs[(q - 1) % NB] + (ty * RY) * HX + tx;
#pragma unroll
        for (int s = 0; s < RY + 2; ++s)
#pragma unroll
          for (int c = 0; c < 3; ++c) nbp[s][c] = t[s * HX + c];
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
          double Mb = ap9(w1, nbp, r), Mt = ap9(w1, nbq, r);
          double Kb = ap9(w2, nbp, r), Kt = ap9(w2, nbq, r);
          double bot = F.u00 * Mb + F.u01 * Mt + F.t00 * Kb + F.t01 * Kt;
          double top = F.u10 * Mb + F.u11 * Mt + F.t10 * Kb + F.t11 * Kt;
          double db = F.u00 * w1[4] + F.t00 * w2[4];
          double dt = F.u11 * w1[4] + F.t11 * w2[4];
          out_row(prow, r, carry[r] + bot, dcarry[r] + db);
          carry[r] = top;
          dcarry[r] = dt;
        }
      }
    }
  }
  // last row nt: only the top part of layer nt-1
  if (p1 == g.nt + 1) {
    const int p = g.nt;
    if (MODE == MODE_RESID || MODE == MODE_JAC) {
#pragma unroll
      for (int r = 0; r < RY; ++r)
        bnext[r] = act[r] ? __ldg(b + (long long)p * P + (long long)jr[r] * nn + i) : 0.0;
    }
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      double D = TC ? dtopC[r] : dcarry[r];
      out_row(p, r, carry[r], D);
    }
  }
  cp_wait<0>();
}

// JAC0 (first sweep from zero): y = omega b / D, D = diag of the masked operator
template <bool TC, int SRC>
__global__ void jac0_2d_kernel(OpDesc op, const double* __restrict__ b, double* __restrict__ y, double omega) {
  const Geom& g = op.g;
  long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= g.N) return;
  const int p = (int)(idx / g.P);
  const long long pn = idx - (long long)p * g.P;
  const int i = (int)(pn % g.nn), j = (int)(pn / g.nn);
  const bool cons = (p == 0 || (i == 0 && j >= g.plo && j <= g.phi));
  double D = 1.0;
  if (!cons) {
    const int n = g.n;
    double Dd = 0.0;
    const double sm = (SRC == 0) ? g.dx * g.dx * (1.0 / 36.0) : 1.0;
    const double sk = (SRC == 0) ? (1.0 / 6.0) : 1.0;
    for (int side = 0; side < 2; ++side) {
      int tau = side == 0 ? p - 1 : p;  // top of layer p-1, bottom of layer p
      if (tau < 0 || tau >= g.nt) continue;
      double Mc, Kc;
      if (SRC == 0) {
        double sc = 0.0, sk2 = 0.0;
        for (int e = 0; e < 4; ++e) {
          int a = i - 1 + (e & 1), bb = j - 1 + (e >> 1);
          if (a < 0 || a >= n || bb < 0 || bb >= n) continue;
          long long ri = (long long)bb * n + a + (TC ? 0 : (long long)tau * n * n);
          double rho = __ldg(op.rho + ri);
          sc += op.m.Cins + op.m.dC * powp(rho, op.m.pc);
          sk2 += op.m.kins + op.m.dk * powp(rho, op.m.pk);
        }
        Mc = 4.0 * sc * sm;
        Kc = 4.0 * sk2 * sk;
      } else {
        Mc = __ldg(op.st + pn);
        Kc = __ldg(op.st + 5 * g.P + pn);
      }
      Dd += side == 0 ? (op.U[1][1] * Mc + op.Tm[1][1] * Kc) : (op.U[0][0] * Mc + op.Tm[0][0] * Kc);
    }
    D = Dd;
  }
  y[idx] = omega * __ldg(b + idx) / D;
}

}  // namespace f2

static int choose_chunk2(const Geom& g, long long tiles) {
  // aim for ~4 waves of CTAs over 148 SMs x 3 resident CTAs, chunks >= 8 planes
  long long target = 148LL * 3 * 4;
  long long chunks = (target + tiles - 1) / tiles;
  long long maxch = (g.nt + 1 + 7) / 8;
  if (chunks > maxch) chunks = maxch;
  if (chunks < 1) chunks = 1;
  return (int)((g.nt + 1 + chunks - 1) / chunks);
}

template <bool TC, int SRC, int MODE, bool TRANS, bool MASK>
static void l2d(const OpDesc& op, const double* x, const double* b, double* y, double omega, cudaStream_t s) {
  const Geom& g = op.g;
  dim3 blk(f2::TX, f2::TYT, 1);
  long long tx = (g.nn + f2::TX - 1) / f2::TX, ty = (g.nn + f2::TY - 1) / f2::TY;
  int chunk = choose_chunk2(g, tx * ty);
  dim3 grd((unsigned)tx, (unsigned)ty, (unsigned)((g.nt + 1 + chunk - 1) / chunk));
  f2::op2d_kernel<TC, SRC, MODE, TRANS, MASK><<<grd, blk, 0, s>>>(op, x, b, y, omega, chunk);
}

template <bool TC, int SRC>
static void l2d_modes(const OpDesc& op, int mode, bool trans, bool mask, const double* x, const double* b, double* y,
                      double omega, cudaStream_t s) {
  if (mode == MODE_JAC0) {
    unsigned grd = (unsigned)((op.g.N + 255) / 256);
    f2::jac0_2d_kernel<TC, SRC><<<grd, 256, 0, s>>>(op, b, y, omega);
    return;
  }
  if (!mask) {
    if (trans) l2d<TC, SRC, MODE_APPLY, true, false>(op, x, b, y, omega, s);
    else l2d<TC, SRC, MODE_APPLY, false, false>(op, x, b, y, omega, s);
    return;
  }
#define C2(M)                                                             \
  case M:                                                                 \
    if (trans) l2d<TC, SRC, M, true, true>(op, x, b, y, omega, s);        \
    else l2d<TC, SRC, M, false, true>(op, x, b, y, omega, s);             \
    break;
  switch (mode) {
    C2(MODE_APPLY)
    C2(MODE_RESID)
    C2(MODE_JAC)
  }
#undef C2
}

// returns false when the fast path does not cover the operator
bool launch_op_fast2d(const OpDesc& op, int mode, bool trans, bool mask, const double* x, const double* b, double* y,
                      double omega, cudaStream_t s) {
  if (op.g.sd != 2) return false;
  if (mode == MODE_JAC0 && !mask) return false;
  if (op.form == FORM_RHO) {
    if (op.rho_tc) l2d_modes<true, 0>(op, mode, trans, mask, x, b, y, omega, s);
    else l2d_modes<false, 0>(op, mode, trans, mask, x, b, y, omega, s);
    return true;
  }
  if (op.form == FORM_MK && op.nl == 1) {
    l2d_modes<true, 1>(op, mode, trans, mask, x, b, y, omega, s);
    return true;
  }
  return false;
}

}  // namespace st
