// opcore.cuh — per-node level-operator algebra of the generic kernels (ops.cu).
// Algebra: common.cuh / DESIGN.md sec. 7.
#pragma once
#include "common.cuh"

namespace st {

// ---------------------------------------------------------------------------------------
// element coefficients around a node (layer tau)
template <int SD>
__device__ __forceinline__ void elem_ck(const OpDesc& op, const int* c, int tau, double* ce, double* ke) {
  const Geom& g = op.g;
#pragma unroll
  for (int e = 0; e < SG<SD>::NE; ++e) {
    bool valid = (tau >= 0 && tau < g.nt);
    long long eidx = 0, mul = 1;
#pragma unroll
    for (int d = 0; d < SD; ++d) {
      int a = c[d] + ((e >> d) & 1) - 1;
      valid = valid && (a >= 0 && a < g.n);
      eidx += (long long)a * mul;
      mul *= g.n;
    }
    if (valid) {
      long long ri = op.rho_tc ? eidx : (long long)tau * mul + eidx;
      double r = __ldg(op.rho + ri);
      ce[e] = op.m.Cins + op.m.dC * powp(r, op.m.pc);
      ke[e] = op.m.kins + op.m.dk * powp(r, op.m.pk);
    } else {
      ce[e] = 0.0;
      ke[e] = 0.0;
    }
  }
}

// normalised spatial tables: M = sM * mh[h], K = sK * kh[h]
template <int SD> __device__ __forceinline__ double mh(int h) {
  return SD == 2 ? (h == 0 ? 4.0 : (h == 1 ? 2.0 : 1.0)) : (h == 0 ? 8.0 : (h == 1 ? 4.0 : (h == 2 ? 2.0 : 1.0)));
}
template <int SD> __device__ __forceinline__ double kh(int h) {
  return SD == 2 ? (h == 0 ? 4.0 : (h == 1 ? -1.0 : -2.0)) : (h == 0 ? 4.0 : (h == 1 ? 0.0 : -1.0));
}
template <int SD> __device__ __forceinline__ double sM(double dx) {
  return SD == 2 ? dx * dx / 36.0 : dx * dx * dx / 216.0;
}
template <int SD> __device__ __forceinline__ double sK(double dx) {
  return SD == 2 ? 1.0 / 6.0 : dx / 12.0;
}

// weighted mass / stiffness applied at the node: sum_e coef_e * (element row . x)
template <int SD>
__device__ __forceinline__ void rho_MK(const double* ce, const double* ke, const double* xs, double dx,
                                       double& Mx, double& Kx) {
  double m = 0.0, k = 0.0;
#pragma unroll
  for (int e = 0; e < SG<SD>::NE; ++e) {
    double pm = 0.0, pk = 0.0;
#pragma unroll
    for (int b = 0; b < SG<SD>::NE; ++b) {
      int kk = 0, h = 0, mul = 1;
#pragma unroll
      for (int d = 0; d < SD; ++d) {
        int bit = (e >> d) & 1, be = (b >> d) & 1;
        int o = bit - 1 + be;
        kk += (o + 1) * mul;
        mul *= 3;
        h += (be != 1 - bit) ? 1 : 0;
      }
      pm += mh<SD>(h) * xs[kk];
      if (kh<SD>(h) != 0.0) pk += kh<SD>(h) * xs[kk];
    }
    m += ce[e] * pm;
    k += ke[e] * pk;
  }
  Mx = m * sM<SD>(dx);
  Kx = k * sK<SD>(dx);
}

// full stencil weight of offset k for the RHO form (s = 0: M, 1: K)
template <int SD>
__device__ __forceinline__ double rho_weight(const double* ce, const double* ke, int k, int s, double dx) {
  double w = 0.0;
  int h = 0;
#pragma unroll
  for (int d = 0; d < SD; ++d) h += SG<SD>::od(k, d) != 0;
#pragma unroll
  for (int e = 0; e < SG<SD>::NE; ++e) {
    bool in = true;
#pragma unroll
    for (int d = 0; d < SD; ++d) {
      int o = SG<SD>::od(k, d), bit = (e >> d) & 1;
      if (o == 1 && bit != 1) in = false;
      if (o == -1 && bit != 0) in = false;
    }
    if (in) w += (s == 0 ? ce[e] : ke[e]);
  }
  return s == 0 ? w * mh<SD>(h) * sM<SD>(dx) : w * kh<SD>(h) * sK<SD>(dx);
}

// stored symmetric stencil: weight of offset k at node c (base = layer/stencil origin)
template <int SD>
__device__ __forceinline__ double st_weight(const Geom& g, const double* __restrict__ base, const int* c,
                                            long long pn, int k) {
  constexpr int CEN = SG<SD>::CEN, NOFF = SG<SD>::NOFF;
  if (k >= CEN) return __ldg(base + (long long)(k - CEN) * g.P + pn);
  // mirrored offset: the neighbour's forward coefficient. Branch-free (an outside neighbour reads the
  // node's own entry and is masked), so the loads of a stencil issue back to back (latency-bound levels)
  int nb[3] = {0, 0, 0};
  bool ok = true;
#pragma unroll
  for (int d = 0; d < SD; ++d) {
    nb[d] = c[d] + SG<SD>::od(k, d);
    ok = ok && nb[d] >= 0 && nb[d] < g.nn;
  }
  const double v = __ldg(base + (long long)(NOFF - 1 - k - CEN) * g.P + (ok ? pidx<SD>(g, nb) : pn));
  return ok ? v : 0.0;
}

template <int SD>
__device__ __forceinline__ double st_apply(const Geom& g, const double* __restrict__ base, const int* c,
                                           long long pn, const double* xs) {
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < SG<SD>::NOFF; ++k) acc += st_weight<SD>(g, base, c, pn, k) * xs[k];
  return acc;
}

template <bool TRANS>
__device__ __forceinline__ void combine_mk(const OpDesc& op, double Mb, double Mt, double Kb, double Kt,
                                           double& bot, double& top) {
  if (!TRANS) {
    bot = op.U[0][0] * Mb + op.U[0][1] * Mt + op.Tm[0][0] * Kb + op.Tm[0][1] * Kt;
    top = op.U[1][0] * Mb + op.U[1][1] * Mt + op.Tm[1][0] * Kb + op.Tm[1][1] * Kt;
  } else {
    bot = op.U[0][0] * Mb + op.U[1][0] * Mt + op.Tm[0][0] * Kb + op.Tm[1][0] * Kt;
    top = op.U[0][1] * Mb + op.U[1][1] * Mt + op.Tm[0][1] * Kb + op.Tm[1][1] * Kt;
  }
}

// evaluate layer tau at node c: contributions to row tau (bot) and row tau+1 (top), plus
// the diagonal parts S^{bb}_center (dbot) and S^{tt}_center (dtop)
template <int SD, int FORM, bool TRANS, bool NEEDX, bool NEEDD>
__device__ __forceinline__ void layer_eval(const OpDesc& op, const int* c, long long pn, int tau,
                                           const double* xb, const double* xt, double& bot, double& top,
                                           double& dbot, double& dtop) {
  constexpr int NC = SG<SD>::NC, CEN = SG<SD>::CEN;
  const Geom& g = op.g;
  bot = top = dbot = dtop = 0.0;
  if (FORM == FORM_RHO) {
    double ce[SG<SD>::NE], ke[SG<SD>::NE];
    elem_ck<SD>(op, c, tau, ce, ke);
    if (NEEDX) {
      double Mb, Kb, Mt, Kt;
      rho_MK<SD>(ce, ke, xb, g.dx, Mb, Kb);
      rho_MK<SD>(ce, ke, xt, g.dx, Mt, Kt);
      combine_mk<TRANS>(op, Mb, Mt, Kb, Kt, bot, top);
    }
    if (NEEDD) {
      double Mc = rho_weight<SD>(ce, ke, CEN, 0, g.dx), Kc = rho_weight<SD>(ce, ke, CEN, 1, g.dx);
      dbot = op.U[0][0] * Mc + op.Tm[0][0] * Kc;
      dtop = op.U[1][1] * Mc + op.Tm[1][1] * Kc;
    }
  } else if (FORM == FORM_MK) {
    const double* Mbase = op.st + (long long)(op.tvl ? tau : 0) * 2 * NC * g.P;
    const double* Kbase = Mbase + (long long)NC * g.P;
    if (NEEDX) {
      double Mb = st_apply<SD>(g, Mbase, c, pn, xb), Mt = st_apply<SD>(g, Mbase, c, pn, xt);
      double Kb = st_apply<SD>(g, Kbase, c, pn, xb), Kt = st_apply<SD>(g, Kbase, c, pn, xt);
      combine_mk<TRANS>(op, Mb, Mt, Kb, Kt, bot, top);
    }
    if (NEEDD) {
      double Mc = __ldg(Mbase + pn), Kc = __ldg(Kbase + pn);
      dbot = op.U[0][0] * Mc + op.Tm[0][0] * Kc;
      dtop = op.U[1][1] * Mc + op.Tm[1][1] * Kc;
    }
  } else {  // FORM_B4: [M, Kbb, Kbt, Ktb, Ktt], S^{ab} = U[a][b] M + K^{ab}
    const double* base = op.st + (long long)(op.tvl ? tau : 0) * 5 * NC * g.P;
    const double* Mst = base;
    const double* Kbb = base + (long long)NC * g.P;
    const double* Kbt = base + 2LL * NC * g.P;
    const double* Ktb = base + 3LL * NC * g.P;
    const double* Ktt = base + 4LL * NC * g.P;
    if (NEEDX) {
      double Mb = st_apply<SD>(g, Mst, c, pn, xb), Mt = st_apply<SD>(g, Mst, c, pn, xt);
      if (!TRANS) {
        bot = op.U[0][0] * Mb + op.U[0][1] * Mt + st_apply<SD>(g, Kbb, c, pn, xb) + st_apply<SD>(g, Kbt, c, pn, xt);
        top = op.U[1][0] * Mb + op.U[1][1] * Mt + st_apply<SD>(g, Ktb, c, pn, xb) + st_apply<SD>(g, Ktt, c, pn, xt);
      } else {
        bot = op.U[0][0] * Mb + op.U[1][0] * Mt + st_apply<SD>(g, Kbb, c, pn, xb) + st_apply<SD>(g, Ktb, c, pn, xt);
        top = op.U[0][1] * Mb + op.U[1][1] * Mt + st_apply<SD>(g, Kbt, c, pn, xb) + st_apply<SD>(g, Ktt, c, pn, xt);
      }
    }
    if (NEEDD) {
      double Mc = __ldg(Mst + pn);
      dbot = op.U[0][0] * Mc + __ldg(Kbb + pn);
      dtop = op.U[1][1] * Mc + __ldg(Ktt + pn);
    }
  }
}

template <int SD, bool MASK>
__device__ __forceinline__ void load_nb(const Geom& g, const double* __restrict__ x, const int* c, int q,
                                        double* xs) {
  const double* xp = x + (long long)q * g.P;
#pragma unroll
  for (int k = 0; k < SG<SD>::NOFF; ++k) {
    int nb[3] = {0, 0, 0};
    bool valid = true;
#pragma unroll
    for (int d = 0; d < SD; ++d) {
      nb[d] = c[d] + SG<SD>::od(k, d);
      valid = valid && nb[d] >= 0 && nb[d] < g.nn;
    }
    double v = 0.0;
    if (valid) {
      v = __ldg(xp + pidx<SD>(g, nb));
      if (MASK && is_cons<SD>(g, nb, q)) v = 0.0;
    }
    xs[k] = v;
  }
}



// Rows [p0, p1) of the (masked) level operator at spatial node (i0, row r) (r = x2 in 2D, x2 + nn x3 in
// 3D), marching in time: each element layer is evaluated once, its top part carried to the next row.
// Modes: APPLY y = A x; RESID y = b - A x; JAC y = x + w D^-1 (b - A x); JAC0 y = w D^-1 b. Used by
// the generic kernels (op_kernel, ops.cu).
template <int SD, int FORM, int MODE, bool TRANS, bool MASK>
__device__ __forceinline__ void op_rows(const OpDesc& op, const double* __restrict__ x, const double* __restrict__ b,
                                        double* __restrict__ y, double omega, int i0, int r, int p0, int p1) {
  constexpr int NOFF = SG<SD>::NOFF;
  constexpr bool NEEDX = (MODE != MODE_JAC0);
  constexpr bool NEEDD = (MODE == MODE_JAC || MODE == MODE_JAC0);
  const Geom& g = op.g;
  int c[3];
  c[0] = i0;
  c[1] = (SD == 2) ? r : r % g.nn;
  c[2] = (SD == 2) ? 0 : r / g.nn;
  const long long pn = i0 + (long long)g.pr * r;
  const bool patch = MASK && is_patch<SD>(g, c);

  double xb[NOFF], xt[NOFF];
  double carry = 0.0, dcarry = 0.0;
  if (NEEDX) {
    if (p0 >= 1) {
      load_nb<SD, MASK>(g, x, c, p0 - 1, xb);
      load_nb<SD, MASK>(g, x, c, p0, xt);
    } else {
      load_nb<SD, MASK>(g, x, c, p0, xt);
    }
  }
  if (p0 >= 1) {
    double bt, tp, db, dt;
    layer_eval<SD, FORM, TRANS, NEEDX, NEEDD>(op, c, pn, p0 - 1, xb, xt, bt, tp, db, dt);
    carry = tp;
    dcarry = dt;
  }
  for (int p = p0; p < p1; ++p) {
    if (NEEDX) {
#pragma unroll
      for (int k = 0; k < NOFF; ++k) xb[k] = xt[k];
    }
    double bot = 0.0, top = 0.0, dbot = 0.0, dtop = 0.0;
    if (p < g.nt) {
      if (NEEDX) load_nb<SD, MASK>(g, x, c, p + 1, xt);
      layer_eval<SD, FORM, TRANS, NEEDX, NEEDD>(op, c, pn, p, xb, xt, bot, top, dbot, dtop);
    }
    const long long gi = (long long)p * g.P + pn;
    const bool cons = MASK && (p + g.pg0 == 0 || patch);
    double Ax = carry + bot;
    double D = dcarry + dbot;
    if (cons) {
      Ax = NEEDX ? __ldg(x + gi) : 0.0;
      D = 1.0;
    }
    double out;
    if (MODE == MODE_APPLY) out = Ax;
    else if (MODE == MODE_RESID) out = __ldg(b + gi) - Ax;
    else if (MODE == MODE_JAC) out = __ldg(x + gi) + omega * (__ldg(b + gi) - Ax) / D;
    else out = omega * __ldg(b + gi) / D;
    y[gi] = out;
    carry = top;
    dcarry = dtop;
  }
}

}  // namespace st
