// ops.cu — level operators of the space-time system (2D+t and 3D+t), fp64, sm_100a.
//
// One kernel family evaluates, for every node of a level, the row of the (masked) operator
//   (K x)_p = S^{tb}_{p-1} x_{p-1} + S^{tt}_{p-1} x_p + S^{bb}_p x_p + S^{bt}_p x_{p+1}
// (transpose: swap S^{bt} <-> S^{tb}; spatial stencils are symmetric), marching in time so
// that each element layer is evaluated once per node: the layer-p evaluation yields the
// bottom part of row p and the top part of row p+1 (carried in a register).
// Modes: APPLY y = A x; RESID y = b - A x; JAC y = x + w D^-1 (b - A x); JAC0 y = w D^-1 b.
// Dirichlet elimination (R-1): A = m_f K m_f + m_c.
// Fine level (FORM_RHO) is matrix-free: C_e, k~_e from rho by SIMP on the
// fly, element matrices C (U (x) M_sp) + k~ (Tm (x) K_sp) (F1).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "opcore.cuh"

namespace st {

template <int SD, int FORM, int MODE, bool TRANS, bool MASK>
__global__ void __launch_bounds__(128) op_kernel(OpDesc op, const double* __restrict__ x,
                                                 const double* __restrict__ b, double* __restrict__ y,
                                                 double omega, int chunk) {
  pdl_wait();
  const Geom& g = op.g;
  const int i0 = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y * blockDim.y + threadIdx.y;
  const int rows = (SD == 2) ? g.nn : g.nn * g.nn;
  if (i0 >= g.nn || r >= rows) return;
  const int p0 = blockIdx.z * chunk;
  if (p0 > g.nt) return;
  op_rows<SD, FORM, MODE, TRANS, MASK>(op, x, b, y, omega, i0, r, p0, min(p0 + chunk, g.nt + 1));
}

// ---------------------------------------------------------------------------------------
static int choose_chunk(const Geom& g) {
  long long per_plane = g.P;
  long long target = 148LL * 2048 * 2;
  long long chunks = (target + per_plane - 1) / per_plane;
  if (chunks < 1) chunks = 1;
  if (chunks > g.nt + 1) chunks = g.nt + 1;
  return (int)((g.nt + 1 + chunks - 1) / chunks);
}

template <int SD, int FORM, int MODE, bool TRANS, bool MASK>
static void launch_t(const OpDesc& op, const double* x, const double* b, double* y, double omega, cudaStream_t s) {
  const Geom& g = op.g;
  dim3 blk(32, 4, 1);
  int rows = SD == 2 ? g.nn : g.nn * g.nn;
  int chunk = op.chunk > 0 ? std::min(op.chunk, g.nt + 1) : choose_chunk(g);
  dim3 grd((g.nn + 31) / 32, (rows + 3) / 4, (g.nt + 1 + chunk - 1) / chunk);
  launch_pdl(op_kernel<SD, FORM, MODE, TRANS, MASK>, grd, blk, 0, s, op, x, b, y, omega, chunk);
}

template <int SD, int FORM>
static void launch_f(const OpDesc& op, int mode, bool trans, bool mask, const double* x, const double* b,
                     double* y, double omega, cudaStream_t s) {
  if (!mask) {
    if (trans) launch_t<SD, FORM, MODE_APPLY, true, false>(op, x, b, y, omega, s);
    else launch_t<SD, FORM, MODE_APPLY, false, false>(op, x, b, y, omega, s);
    return;
  }
#define ST_CASE(M)                                                              \
  case M:                                                                       \
    if (trans) launch_t<SD, FORM, M, true, true>(op, x, b, y, omega, s);        \
    else launch_t<SD, FORM, M, false, true>(op, x, b, y, omega, s);             \
    break;
  switch (mode) {
    ST_CASE(MODE_APPLY)
    ST_CASE(MODE_RESID)
    ST_CASE(MODE_JAC)
    ST_CASE(MODE_JAC0)
  }
#undef ST_CASE
}

void launch_op(const OpDesc& op, int mode, bool trans, bool mask, const double* x, const double* b, double* y,
               double omega, cudaStream_t s) {
  // kernel family (st_options_t kernel_family): the specialised TMA kernels where they apply, the
  // general TMA kernel (tma2d), the cp.async-ring kernels (fast2d), then the generic kernels
  const int f = op.family;
  if (f == 0 && launch_op_tc2d(op, mode, trans, mask, x, b, y, omega, s)) return;
  if (f == 0 && launch_op_tc3r(op, mode, trans, mask, x, b, y, omega, s)) return;
  if (f == 0 && launch_op_tc3d(op, mode, trans, mask, x, b, y, omega, s)) return;
  if (f == 0 && launch_op_tv2d(op, mode, trans, mask, x, b, y, omega, s)) return;
  if ((f == 0 || f == 3) && launch_op_tma2d(op, mode, trans, mask, x, b, y, omega, s)) return;
  if (f != 2 && launch_op_fast2d(op, mode, trans, mask, x, b, y, omega, s)) return;
  if (op.g.sd == 2) {
    if (op.form == FORM_RHO) launch_f<2, FORM_RHO>(op, mode, trans, mask, x, b, y, omega, s);
    else if (op.form == FORM_MK) launch_f<2, FORM_MK>(op, mode, trans, mask, x, b, y, omega, s);
    else launch_f<2, FORM_B4>(op, mode, trans, mask, x, b, y, omega, s);
  } else {
    if (op.form == FORM_RHO) launch_f<3, FORM_RHO>(op, mode, trans, mask, x, b, y, omega, s);
    else if (op.form == FORM_MK) launch_f<3, FORM_MK>(op, mode, trans, mask, x, b, y, omega, s);
    else launch_f<3, FORM_B4>(op, mode, trans, mask, x, b, y, omega, s);
  }
}

// ---------------------------------------------------------------------------------------
// Weight accessors used by the Galerkin and dense-assembly kernels (full weight of offset k
// at node c, layer tau): capacity part M (time factor op.U) and conduction blocks K^{ab}.
template <int SD, int FORM>
__device__ double mpart_weight(const OpDesc& op, const int* c, long long pn, int tau, int k) {
  constexpr int NC = SG<SD>::NC;
  const Geom& g = op.g;
  if (FORM == FORM_RHO) {
    double ce[SG<SD>::NE], ke[SG<SD>::NE];
    elem_ck<SD>(op, c, tau, ce, ke);
    return rho_weight<SD>(ce, ke, k, 0, g.dx);
  } else if (FORM == FORM_MK) {
    return st_weight<SD>(g, op.st + (long long)(op.tvl ? tau : 0) * 2 * NC * g.P, c, pn, k);
  } else {
    return st_weight<SD>(g, op.st + (long long)(op.tvl ? tau : 0) * 5 * NC * g.P, c, pn, k);
  }
}

template <int SD, int FORM>
__device__ double kblock_weight(const OpDesc& op, const int* c, long long pn, int tau, int a, int bb, int k) {
  constexpr int NC = SG<SD>::NC;
  const Geom& g = op.g;
  if (FORM == FORM_RHO) {
    double ce[SG<SD>::NE], ke[SG<SD>::NE];
    elem_ck<SD>(op, c, tau, ce, ke);
    return op.Tm[a][bb] * rho_weight<SD>(ce, ke, k, 1, g.dx);
  } else if (FORM == FORM_MK) {
    const double* Kb = op.st + (long long)(op.tvl ? tau : 0) * 2 * NC * g.P + (long long)NC * g.P;
    return op.Tm[a][bb] * st_weight<SD>(g, Kb, c, pn, k);
  } else {
    const double* Kb = op.st + (long long)(op.tvl ? tau : 0) * 5 * NC * g.P + (long long)(1 + 2 * a + bb) * NC * g.P;
    return st_weight<SD>(g, Kb, c, pn, k);
  }
}

template <int SD, int FORM>
__device__ double block_weight(const OpDesc& op, const int* c, long long pn, int tau, int a, int bb, int k) {
  return op.U[a][bb] * mpart_weight<SD, FORM>(op, c, pn, tau, k) + kblock_weight<SD, FORM>(op, c, pn, tau, a, bb, k);
}

// MK weight of stencil s (0 = M, 1 = K) — only for RHO / MK forms
template <int SD, int FORM>
__device__ double mk_weight(const OpDesc& op, const int* c, long long pn, int tau, int s, int k) {
  constexpr int NC = SG<SD>::NC;
  const Geom& g = op.g;
  if (FORM == FORM_RHO) {
    double ce[SG<SD>::NE], ke[SG<SD>::NE];
    elem_ck<SD>(op, c, tau, ce, ke);
    return rho_weight<SD>(ce, ke, k, s, g.dx);
  } else {
    const double* base = op.st + (long long)(op.tvl ? tau : 0) * 2 * NC * g.P + (long long)s * NC * g.P;
    return st_weight<SD>(g, base, c, pn, k);
  }
}

// ---------------------------------------------------------------------------------------
// Galerkin coarse operators, structured.
// Spatial coarsening: every stored stencil of the coarse level is P_x^T S P_x with the
// bilinear/trilinear interpolation P_x (weights 1, 1/2 per direction), per layer.
// NS stencils: MK -> 2 (M, K), B4 -> 5 (M, K^{bb}, K^{bt}, K^{tb}, K^{tt}).
template <int SD, int FFORM, int NS>
__global__ void rap_space_kernel(OpDesc fop, Geom gc, int nl, double* __restrict__ out) {
  constexpr int NOFF = SG<SD>::NOFF, NC = SG<SD>::NC, CEN = SG<SD>::CEN;
  const Geom& gf = fop.g;
  long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long total = gc.P * nl * NS;
  if (idx >= total) return;
  long long pc = idx % gc.P;
  int s = (int)((idx / gc.P) % NS);
  int tau = (int)(idx / (gc.P * NS));
  int C[3] = {0, 0, 0};
  if (!pdecode<SD>(gc, pc, C)) return;
  double acc[NC];
#pragma unroll
  for (int q = 0; q < NC; ++q) acc[q] = 0.0;
  // loop over fine nodes f in supp(C)
  for (int fa = 0; fa < NOFF; ++fa) {
    int f[3] = {0, 0, 0};
    bool ok = true;
    double wf = 1.0;
    for (int d = 0; d < SD; ++d) {
      int o = SG<SD>::od(fa, d);
      f[d] = 2 * C[d] + o;
      ok = ok && f[d] >= 0 && f[d] < gf.nn;
      wf *= (o == 0) ? 1.0 : 0.5;
    }
    if (!ok) continue;
    long long pf = pidx<SD>(gf, f);
    for (int k = 0; k < NOFF; ++k) {
      int gg[3] = {0, 0, 0};
      bool okg = true;
      for (int d = 0; d < SD; ++d) {
        gg[d] = f[d] + SG<SD>::od(k, d);
        okg = okg && gg[d] >= 0 && gg[d] < gf.nn;
      }
      if (!okg) continue;
      double w;
      if (NS == 2) w = mk_weight<SD, FFORM>(fop, f, pf, tau, s, k);
      else if (s == 0) w = mpart_weight<SD, FFORM>(fop, f, pf, tau, k);
      else w = kblock_weight<SD, FFORM>(fop, f, pf, tau, (s - 1) >> 1, (s - 1) & 1, k);
      if (w == 0.0) continue;
      // interpolation weight of g from coarse node C + off(q), q >= CEN
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        int kq = q + CEN;
        double wg = 1.0;
        for (int d = 0; d < SD; ++d) {
          int diff = gg[d] - 2 * (C[d] + SG<SD>::od(kq, d));
          if (diff < -1 || diff > 1) { wg = 0.0; break; }
          wg *= (diff == 0) ? 1.0 : 0.5;
        }
        acc[q] += wf * w * wg;
      }
    }
  }
  double* o = out + ((long long)tau * NS + s) * NC * gc.P;
#pragma unroll
  for (int q = 0; q < NC; ++q) o[(long long)q * gc.P + pc] = acc[q];
}

// Spatial coarsening of the fine (rho) level, M and K per layer. The Galerkin weight P^T S P of
// coarse node C and forward offset q is linear in the element coefficients of the 4^SD fine
// elements around 2C: S_q = sum_e Tab[s][q][e] coef_e (coef = C~ for s = 0, k~ for s = 1, then the
// spatial scale sM / sK). Tab (dyadic rationals, exact) is built on the host by the same loops as
// rap_space_kernel (fine nodes f of supp C, stencil offsets k, elements adjacent to f and f + k,
// interpolation weights); each thread evaluates its 4^SD element coefficients once instead of
// once per (f, k) weight.
__constant__ double c_rap2[2 * 5 * 16];
__constant__ double c_rap3[2 * 14 * 64];

template <int SD>
void rap_rho_table(double* T) {
  constexpr int NOFF = SG<SD>::NOFF, NC = SG<SD>::NC, CEN = SG<SD>::CEN, NBK = 1 << (2 * SD);
  const double mhv[4] = {SD == 2 ? 4.0 : 8.0, SD == 2 ? 2.0 : 4.0, SD == 2 ? 1.0 : 2.0, 1.0};
  const double khv[4] = {4.0, SD == 2 ? -1.0 : 0.0, SD == 2 ? -2.0 : -1.0, -1.0};
  for (int i = 0; i < 2 * NC * NBK; ++i) T[i] = 0.0;
  for (int e = 0; e < NBK; ++e)
    for (int fa = 0; fa < NOFF; ++fa)
      for (int k = 0; k < NOFF; ++k) {
        bool in = true;
        double wf = 1.0;
        int h = 0;
        for (int d = 0; d < SD; ++d) {
          const int bc = (e >> (2 * d)) & 3, o = SG<SD>::od(fa, d), kd = SG<SD>::od(k, d), gr = o + kd;
          in = in && (o == bc - 2 || o == bc - 1) && (gr == bc - 2 || gr == bc - 1);
          wf *= (o == 0) ? 1.0 : 0.5;
          h += kd != 0;
        }
        if (!in) continue;
        for (int q = 0; q < NC; ++q) {
          double wg = 1.0;
          for (int d = 0; d < SD; ++d) {
            const int diff = SG<SD>::od(fa, d) + SG<SD>::od(k, d) - 2 * SG<SD>::od(q + CEN, d);
            wg *= (diff == 0) ? 1.0 : ((diff == 1 || diff == -1) ? 0.5 : 0.0);
          }
          T[(0 * NC + q) * NBK + e] += wf * wg * mhv[h];
          T[(1 * NC + q) * NBK + e] += wf * wg * khv[h];
        }
      }
}

template <int SD>
__global__ void rap_space_rho_kernel(OpDesc fop, Geom gc, int nl, double* __restrict__ out) {
  constexpr int NC = SG<SD>::NC, NBK = 1 << (2 * SD);
  const Geom& gf = fop.g;
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= gc.P * nl) return;
  const long long pc = idx % gc.P;
  const int tau = (int)(idx / gc.P);
  int C[3] = {0, 0, 0};
  if (!pdecode<SD>(gc, pc, C)) return;
  const double* tab = SD == 2 ? c_rap2 : c_rap3;
  long long per = 1;
  for (int d = 0; d < SD; ++d) per *= gf.n;
  const double* rl = fop.rho + (fop.rho_tc ? 0LL : (long long)tau * per);
  double ce[NBK], ke[NBK];
#pragma unroll
  for (int e = 0; e < NBK; ++e) {
    bool v = tau < gf.nt;
    long long ei = 0, m = 1;
#pragma unroll
    for (int d = 0; d < SD; ++d) {
      const int a = 2 * C[d] - 2 + ((e >> (2 * d)) & 3);
      v = v && a >= 0 && a < gf.n;
      ei += (long long)a * m;
      m *= gf.n;
    }
    const double r = v ? __ldg(rl + ei) : 0.0;
    ce[e] = v ? fop.m.Cins + fop.m.dC * powp(r, fop.m.pc) : 0.0;
    ke[e] = v ? fop.m.kins + fop.m.dk * powp(r, fop.m.pk) : 0.0;
  }
  const double smf = sM<SD>(gf.dx), skf = sK<SD>(gf.dx);
  double* o = out + (long long)tau * 2 * NC * gc.P + pc;
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    double am = 0.0, ak = 0.0;
#pragma unroll
    for (int e = 0; e < NBK; ++e) {
      am = fma(tab[q * NBK + e], ce[e], am);
      ak = fma(tab[(NC + q) * NBK + e], ke[e], ak);
    }
    o[(long long)q * gc.P] = am * smf;
    o[(long long)(NC + q) * gc.P] = ak * skf;
  }
}

// Time coarsening: coarse layer T from fine layers 2T, 2T+1:
// conduction blocks by Galerkin with the linear-in-time interpolation (fine plane 2T+1 =
// (coarse T + coarse T+1)/2): K'^{AB} = sum_f sum_{a,b} W_f[a][A] W_f[b][B] K_f^{ab},
// W_0 = [[1,0],[.5,.5]], W_1 = [[.5,.5],[0,1]]; capacity part re-stabilised (rediscretised
// upwind time factor, coefficient = mean of the two layers): M' = (M_{2T} + M_{2T+1}) / 2.
template <int SD, int FFORM>
__global__ void rap_time_kernel(OpDesc fop, int nlc, double* __restrict__ out) {
  constexpr int NC = SG<SD>::NC, CEN = SG<SD>::CEN;
  const Geom& g = fop.g;
  long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long total = g.P * nlc;
  if (idx >= total) return;
  long long pn = idx % g.P;
  int T = (int)(idx / g.P);
  int c[3] = {0, 0, 0};
  if (!pdecode<SD>(g, pn, c)) return;
  const double W[2][2][2] = {{{1.0, 0.0}, {0.5, 0.5}}, {{0.5, 0.5}, {0.0, 1.0}}};
  double* o = out + (long long)T * 5 * NC * g.P;
  // FORM_RHO: element coefficients of the two fine layers once (not per weight)
  double ce[2][SG<SD>::NE], ke[2][SG<SD>::NE];
  if (FFORM == FORM_RHO)
    for (int f = 0; f < 2; ++f) elem_ck<SD>(fop, c, fop.rho_tc ? 0 : 2 * T + f, ce[f], ke[f]);
  for (int q = 0; q < NC; ++q) {
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    double macc = 0.0;
    for (int f = 0; f < 2; ++f) {
      int tau = 2 * T + f;
      if ((FFORM == FORM_RHO && fop.rho_tc) || (FFORM != FORM_RHO && !fop.tvl)) tau = 0;
      double s[2][2];
      if (FFORM == FORM_RHO) {
        macc += 0.5 * rho_weight<SD>(ce[f], ke[f], q + CEN, 0, g.dx);
        const double kw = rho_weight<SD>(ce[f], ke[f], q + CEN, 1, g.dx);
        for (int a = 0; a < 2; ++a)
          for (int b = 0; b < 2; ++b) s[a][b] = fop.Tm[a][b] * kw;
      } else {
        macc += 0.5 * mpart_weight<SD, FFORM>(fop, c, pn, tau, q + CEN);
        for (int a = 0; a < 2; ++a)
          for (int b = 0; b < 2; ++b) s[a][b] = kblock_weight<SD, FFORM>(fop, c, pn, tau, a, b, q + CEN);
      }
      for (int A = 0; A < 2; ++A)
        for (int B = 0; B < 2; ++B) {
          double v = 0.0;
          for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b) v += W[f][a][A] * W[f][b][B] * s[a][b];
          acc[A][B] += v;
        }
    }
    o[(long long)q * g.P + pn] = macc;
    for (int A = 0; A < 2; ++A)
      for (int B = 0; B < 2; ++B) o[(long long)(1 + 2 * A + B) * NC * g.P + (long long)q * g.P + pn] = acc[A][B];
  }
}

// Materialise the M, K stencils of the fine RHO operator for one layer (time-constant
// design): out[2][NC][P].
template <int SD>
__global__ void rho_to_mk_kernel(OpDesc fop, int tau, double* __restrict__ out) {
  constexpr int NC = SG<SD>::NC, CEN = SG<SD>::CEN;
  const Geom& g = fop.g;
  long long pn = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (pn >= g.P) return;
  int c[3] = {0, 0, 0};
  if (!pdecode<SD>(g, pn, c)) return;
  double ce[SG<SD>::NE], ke[SG<SD>::NE];
  elem_ck<SD>(fop, c, tau, ce, ke);
  for (int q = 0; q < NC; ++q) {
    out[(long long)q * g.P + pn] = rho_weight<SD>(ce, ke, q + CEN, 0, g.dx);
    out[(long long)(NC + q) * g.P + pn] = rho_weight<SD>(ce, ke, q + CEN, 1, g.dx);
  }
}

void launch_rap_space(const OpDesc& fop, const Geom& gc, int nl, int ns, double* out, cudaStream_t s) {
  long long total = gc.P * nl * ns;
  int blk = 128;
  long long grd = (total + blk - 1) / blk;
  if (fop.form == FORM_RHO && ns == 2) {  // table-driven (the tables are uploaded once per device)
    static bool done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !done[dev]) {
      static double t2[2 * 5 * 16], t3[2 * 14 * 64];
      rap_rho_table<2>(t2);
      rap_rho_table<3>(t3);
      cudaMemcpyToSymbol(c_rap2, t2, sizeof(t2));
      cudaMemcpyToSymbol(c_rap3, t3, sizeof(t3));
      done[dev] = true;
    }
    const long long nth = gc.P * nl;
    const unsigned g2 = (unsigned)((nth + blk - 1) / blk);
    if (fop.g.sd == 2) rap_space_rho_kernel<2><<<g2, blk, 0, s>>>(fop, gc, nl, out);
    else rap_space_rho_kernel<3><<<g2, blk, 0, s>>>(fop, gc, nl, out);
    return;
  }
#define RS(SD, F, NS) rap_space_kernel<SD, F, NS><<<(unsigned)grd, blk, 0, s>>>(fop, gc, nl, out)
  if (fop.g.sd == 2) {
    if (ns == 2) { if (fop.form == FORM_RHO) RS(2, FORM_RHO, 2); else RS(2, FORM_MK, 2); }
    else { if (fop.form == FORM_RHO) RS(2, FORM_RHO, 5); else if (fop.form == FORM_MK) RS(2, FORM_MK, 5); else RS(2, FORM_B4, 5); }
  } else {
    if (ns == 2) { if (fop.form == FORM_RHO) RS(3, FORM_RHO, 2); else RS(3, FORM_MK, 2); }
    else { if (fop.form == FORM_RHO) RS(3, FORM_RHO, 5); else if (fop.form == FORM_MK) RS(3, FORM_MK, 5); else RS(3, FORM_B4, 5); }
  }
#undef RS
}

void launch_rap_time(const OpDesc& fop, int nlc, double* out, cudaStream_t s) {
  long long total = fop.g.P * nlc;
  int blk = 128;
  long long grd = (total + blk - 1) / blk;
#define RT(SD, F) rap_time_kernel<SD, F><<<(unsigned)grd, blk, 0, s>>>(fop, nlc, out)
  if (fop.g.sd == 2) {
    if (fop.form == FORM_RHO) RT(2, FORM_RHO); else if (fop.form == FORM_MK) RT(2, FORM_MK); else RT(2, FORM_B4);
  } else {
    if (fop.form == FORM_RHO) RT(3, FORM_RHO); else if (fop.form == FORM_MK) RT(3, FORM_MK); else RT(3, FORM_B4);
  }
#undef RT
}

void launch_rho_to_mk(const OpDesc& fop, int tau, double* out, cudaStream_t s) {
  int blk = 128;
  long long grd = (fop.g.P + blk - 1) / blk;
  if (fop.g.sd == 2) rho_to_mk_kernel<2><<<(unsigned)grd, blk, 0, s>>>(fop, tau, out);
  else rho_to_mk_kernel<3><<<(unsigned)grd, blk, 0, s>>>(fop, tau, out);
}

// ---------------------------------------------------------------------------------------
// Row-wise Gershgorin ratio max_i sum_j |A_ij| / |A_ii| of the eliminated level operator
// (bound on |lambda|_max(D^-1 A) for the per-level Jacobi weight). Rows of local
// planes [pa, pb]; a time-constant level has only two row types (interior, last plane), so the
// caller passes pa = 1 and the plane count is irrelevant apart from the last-row test.
template <int SD, int FORM>
__global__ void gersh_kernel(OpDesc op, int pa, int pb, unsigned long long* __restrict__ out) {
  constexpr int NOFF = SG<SD>::NOFF, CEN = SG<SD>::CEN;
  const Geom& g = op.g;
  const long long nper = g.P;
  long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double best = 0.0;
  if (idx < nper * (pb - pa + 1)) {
    const int p = pa + (int)(idx / nper);
    const long long pn = idx % nper;
    int c[3] = {0, 0, 0};
    if (pdecode<SD>(g, pn, c) && !is_cons<SD>(g, c, p)) {
      double diag = 0.0, sum = 0.0;
      // FORM_RHO: the element coefficients of layers p-1 and p once (not per weight)
      double ceL[SG<SD>::NE], keL[SG<SD>::NE], ceU[SG<SD>::NE], keU[SG<SD>::NE];
      if (FORM == FORM_RHO) {
        elem_ck<SD>(op, c, p - 1, ceL, keL);
        elem_ck<SD>(op, c, p, ceU, keU);
      }
      auto bw = [&](bool upper, int a, int bb, int k) -> double {
        if (FORM == FORM_RHO) {
          const double m = upper ? rho_weight<SD>(ceU, keU, k, 0, g.dx) : rho_weight<SD>(ceL, keL, k, 0, g.dx);
          const double kk = upper ? rho_weight<SD>(ceU, keU, k, 1, g.dx) : rho_weight<SD>(ceL, keL, k, 1, g.dx);
          return op.U[a][bb] * m + op.Tm[a][bb] * kk;
        }
        return block_weight<SD, FORM>(op, c, pn, upper ? p : p - 1, a, bb, k);
      };
      for (int k = 0; k < NOFF; ++k) {
        int nb[3] = {0, 0, 0};
        bool ok = true;
        for (int d = 0; d < SD; ++d) {
          nb[d] = c[d] + SG<SD>::od(k, d);
          ok = ok && nb[d] >= 0 && nb[d] < g.nn;
        }
        if (!ok) continue;
        // columns on planes p-1, p, p+1 (eliminated constrained columns are zero)
        double wlo = 0.0, wmid = 0.0, whi = 0.0;
        if (p >= 1) {  // layer p-1: top rows
          wlo = bw(false, 1, 0, k);
          wmid = bw(false, 1, 1, k);
        }
        if (p < g.nt) {  // layer p: bottom rows
          wmid += bw(true, 0, 0, k);
          whi = bw(true, 0, 1, k);
        }
        if (k == CEN) diag = wmid;
        if (p >= 1 && !is_cons<SD>(g, nb, p - 1)) sum += fabs(wlo);
        if (!is_cons<SD>(g, nb, p)) sum += fabs(wmid);
        if (p < g.nt && !is_cons<SD>(g, nb, p + 1)) sum += fabs(whi);
      }
      if (diag != 0.0) best = sum / fabs(diag);
    }
  }
  // block max, then one atomic per block (positive doubles order like their bit patterns)
  for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_down_sync(0xffffffffu, best, o));
  __shared__ double wm[8];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, wm[w]);
    atomicMax(out, (unsigned long long)__double_as_longlong(m));
  }
}

// The same Gershgorin ratio for the (2+1)D fine level of a space-time design with uniform capacity
// (configs 1, 3, 5), from the per-design k~ table (zero border: no element masks) with the Q1 weights
// in closed form: per row the 8 element conductivities of the two adjacent layers, ~100 flops instead of
// the generic kernel's per-weight element loops (config 3: 95 ms per design -> a few ms).
__global__ void __launch_bounds__(256) gersh_tv2d_kernel(OpDesc op, int pa, int pb, unsigned long long* __restrict__ out) {
  const Geom& g = op.g;
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double best = 0.0;
  if (idx < g.P * (long long)(pb - pa + 1)) {
    const int p = pa + (int)(idx / g.P);
    int c[3] = {0, 0, 0};
    if (pdecode<2>(g, idx % g.P, c) && !is_cons<2>(g, c, p)) {
      const int i = c[0], j = c[1], n = g.n;
      const long long w2 = n + 2;
      const bool hasL = p >= 1, hasU = p < g.nt;
      // k~ of the 4 elements (e = bx + 2 by: element (i - 1 + bx, j - 1 + by)) of layers p-1 and p
      double kL[4], kU[4], cm[4];
      for (int e = 0; e < 4; ++e) {
        const int ei = i - 1 + (e & 1), ej = j - 1 + (e >> 1);
        const long long col = (long long)(ej + 1) * w2 + (ei + 1);
        kL[e] = hasL ? __ldg(op.kt + (long long)(p - 1) * w2 * w2 + col) : 0.0;
        kU[e] = hasU ? __ldg(op.kt + (long long)p * w2 * w2 + col) : 0.0;
        cm[e] = (ei >= 0 && ei < n && ej >= 0 && ej < n) ? 1.0 : 0.0;  // element inside (uniform capacity)
      }
      const double sm = op.m.Cins * g.dx * g.dx / 36.0, sk = 1.0 / 6.0;
      double diag = 0.0, sum = 0.0;
      if (p >= 2 && i >= 2 && !g.walls && op.U[0][0] == 0.0 && op.U[0][1] == 0.0) {
        // rows without a constrained neighbour (neither the t = 0 plane nor the sink patch at x1 = 0):
        // the same weights, branch-free; neighbours outside the domain carry zero weight (their shared
        // elements have k~ = 0 in the zero-bordered table and no capacity)
        const double u10 = op.U[1][0], u11 = op.U[1][1];
        const double t00 = op.Tm[0][0], t01 = op.Tm[0][1], t10 = op.Tm[1][0], t11 = op.Tm[1][1];
        // sums over the elements shared by the node and the neighbour at offset (ox, oy):
        // index a = ox + 1 along x1 (0: element column 0, 1: both, 2: column 1), likewise b for x2
        double SL[3][3], SU[3][3], SM[3][3];
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            double l = 0.0, u = 0.0, m = 0.0;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int bx = e & 1, by = e >> 1;
              if ((a == 0 && bx != 0) || (a == 2 && bx != 1) || (b == 0 && by != 0) || (b == 2 && by != 1)) continue;
              l += kL[e];
              u += kU[e];
              m += cm[e];
            }
            SL[b][a] = l;
            SU[b][a] = u;
            SM[b][a] = m;
          }
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const int h = (a != 1) + (b != 1);
            const double mw = sm * SM[b][a] * (h == 0 ? 4.0 : (h == 1 ? 2.0 : 1.0));
            const double kf = sk * (h == 0 ? 4.0 : (h == 1 ? -1.0 : -2.0));
            const double KL = kf * SL[b][a], KU = hasU ? kf * SU[b][a] : 0.0;
            const double wlo = fma(u10, mw, t10 * KL);
            const double wmid = fma(u11, mw, fma(t11, KL, t00 * KU));
            const double whi = t01 * KU;
            if (a == 1 && b == 1) diag = wmid;
            sum += fabs(wlo) + fabs(wmid) + fabs(whi);
          }
        if (diag != 0.0) best = sum / fabs(diag);
      } else
      for (int k = 0; k < 9; ++k) {
        const int ox = (k % 3) - 1, oy = (k / 3) - 1;
        const int nb[3] = {i + ox, j + oy, 0};
        if (nb[0] < 0 || nb[0] > n || nb[1] < 0 || nb[1] > n) continue;
        // elements holding both the node and the neighbour, and the Q1 weights by Hamming distance
        double sL = 0.0, sU = 0.0, sM = 0.0;
        for (int e = 0; e < 4; ++e) {
          const int bx = e & 1, by = e >> 1;
          if ((ox == 1 && bx != 1) || (ox == -1 && bx != 0) || (oy == 1 && by != 1) || (oy == -1 && by != 0)) continue;
          sL += kL[e];
          sU += kU[e];
          sM += cm[e];
        }
        const int h = (ox != 0) + (oy != 0);
        const double mw = sm * sM * (h == 0 ? 4.0 : (h == 1 ? 2.0 : 1.0));
        const double kf = sk * (h == 0 ? 4.0 : (h == 1 ? -1.0 : -2.0));
        const double KL = kf * sL, KU = kf * sU;
        double wlo = 0.0, wmid = 0.0, whi = 0.0;
        if (hasL) {
          wlo = op.U[1][0] * mw + op.Tm[1][0] * KL;
          wmid = op.U[1][1] * mw + op.Tm[1][1] * KL;
        }
        if (hasU) {
          wmid += op.U[0][0] * mw + op.Tm[0][0] * KU;
          whi = op.U[0][1] * mw + op.Tm[0][1] * KU;
        }
        if (k == 4) diag = wmid;
        if (hasL && !is_cons<2>(g, nb, p - 1)) sum += fabs(wlo);
        if (!is_cons<2>(g, nb, p)) sum += fabs(wmid);
        if (hasU && !is_cons<2>(g, nb, p + 1)) sum += fabs(whi);
      }
      if (diag != 0.0) best = sum / fabs(diag);
    }
  }
  for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_down_sync(0xffffffffu, best, o));
  __shared__ double wm[8];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, wm[w]);
    atomicMax(out, (unsigned long long)__double_as_longlong(m));
  }
}

void launch_gersh(const OpDesc& op, int pa, int pb, unsigned long long* out, cudaStream_t s) {
  long long total = op.g.P * (long long)(pb - pa + 1);
  if (total <= 0) return;
  if (op.g.sd == 2 && op.form == FORM_RHO && !op.rho_tc && op.kt && op.m.dC == 0.0) {
    gersh_tv2d_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(op, pa, pb, out);
    return;
  }
  unsigned grd = (unsigned)((total + 255) / 256);
#define GK(SD, F) gersh_kernel<SD, F><<<grd, 256, 0, s>>>(op, pa, pb, out)
  if (op.g.sd == 2) {
    if (op.form == FORM_RHO) GK(2, FORM_RHO); else if (op.form == FORM_MK) GK(2, FORM_MK); else GK(2, FORM_B4);
  } else {
    if (op.form == FORM_RHO) GK(3, FORM_RHO); else if (op.form == FORM_MK) GK(3, FORM_MK); else GK(3, FORM_B4);
  }
#undef GK
}

// ---------------------------------------------------------------------------------------
// Dense coarsest operator: A[row][col] of the masked level operator (row-major, N x N).
template <int SD, int FORM>
__global__ void dense_assemble_kernel(OpDesc op, double* __restrict__ A) {
  constexpr int NOFF = SG<SD>::NOFF;
  const Geom& g = op.g;
  long long row = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (row >= g.N) return;
  int p = (int)(row / g.P);
  long long pn = row % g.P;
  int c[3] = {0, 0, 0};
  double* Ar = A + row * g.N;
  if (!pdecode<SD>(g, pn, c) || is_cons<SD>(g, c, p)) { Ar[row] = 1.0; return; }
  // layer p-1 (top rows: S^{tb} -> plane p-1, S^{tt} -> plane p); layer p (bottom rows)
  for (int side = 0; side < 2; ++side) {
    int tau = side == 0 ? p - 1 : p;
    if (tau < 0 || tau >= g.nt) continue;
    int a = side == 0 ? 1 : 0;
    for (int bb = 0; bb < 2; ++bb) {
      int q = tau + bb;  // plane of the trial node
      for (int k = 0; k < NOFF; ++k) {
        int nb[3] = {0, 0, 0};
        bool ok = true;
        for (int d = 0; d < SD; ++d) {
          nb[d] = c[d] + SG<SD>::od(k, d);
          ok = ok && nb[d] >= 0 && nb[d] < g.nn;
        }
        if (!ok) continue;
        if (is_cons<SD>(g, nb, q)) continue;
        double w = block_weight<SD, FORM>(op, c, pn, tau, a, bb, k);
        Ar[(long long)q * g.P + pidx<SD>(g, nb)] += w;
      }
    }
  }
}

void launch_dense_assemble(const OpDesc& op, double* A, cudaStream_t s) {
  int blk = 128;
  long long grd = (op.g.N + blk - 1) / blk;
#define DA(SD, F) dense_assemble_kernel<SD, F><<<(unsigned)grd, blk, 0, s>>>(op, A)
  if (op.g.sd == 2) {
    if (op.form == FORM_RHO) DA(2, FORM_RHO); else if (op.form == FORM_MK) DA(2, FORM_MK); else DA(2, FORM_B4);
  } else {
    if (op.form == FORM_RHO) DA(3, FORM_RHO); else if (op.form == FORM_MK) DA(3, FORM_MK); else DA(3, FORM_B4);
  }
#undef DA
}

}  // namespace st
