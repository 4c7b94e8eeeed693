// tiny2d.cu — small time-constant (2+1)D levels (stored M, K stencils): one thread per node.
//
// On a level of a few thousand to a few hundred thousand nodes the persistent TMA kernel (tc2d) is
// pure pipeline latency: each CTA owns one or two planes, so the barrier set-up, the weight loads
// and the first TMA round trip are never amortised (~6.5 us per launch whatever the size,
// scripts/level_lat.py). Here every node of every plane is an independent thread that reads its
// 3 x 3 x 3 neighbourhood and its 18 stencil weights through L1/L2 (the level fits in L2) — one
// round of independent loads. Row p of the operator (plane form):
//   (K x)_p   = S^tb x_{p-1} + (S^tt + S^bb) x_p + S^bt x_{p+1},  S^ab = U[a][b] M + Tm[a][b] K,
//   (K^T x)_p = S^bt x_{p-1} + (S^tt + S^bb) x_p + S^tb x_{p+1}   (M, K spatially symmetric),
// without the layer-p terms on the last plane; x on the t = 0 plane enters as 0 (eliminated
// columns); constrained rows are identity rows. Same modes as every level kernel.
// Opt-in (ST_TINY_NODES): measured no faster than the TMA kernels inside the V-cycle's CUDA graph,
// where the per-launch latency the ncu launch list shows for each small kernel largely overlaps.
#include "common.cuh"
#include "kernels.h"

namespace st {
namespace {

template <int MODE, bool TRANS>
__global__ void __launch_bounds__(256) tiny2d_kernel(OpDesc op, const double* __restrict__ x,
                                                     const double* __restrict__ b, double* __restrict__ y,
                                                     double omega) {
  constexpr bool NX = (MODE != MODE_JAC0);
  const Geom& g = op.g;
  const long long idx = blockIdx.x * 256LL + threadIdx.x;
  if (idx >= g.N) return;
  const int p = (int)(idx / g.P);
  const long long pn = idx - (long long)p * g.P;
  const int i = (int)(pn % g.pr), j = (int)(pn / g.pr);
  if (i >= g.nn) return;  // pad column: stays zero
  const int n = g.n;
  int c[3] = {i, j, 0};
  const double bv = (MODE != MODE_APPLY) ? __ldg(b + idx) : 0.0;
  if (is_cons<2>(g, c, p)) {
    const double xc = NX ? __ldg(x + idx) : 0.0;
    double o;
    if (MODE == MODE_APPLY) o = xc;
    else if (MODE == MODE_RESID) o = bv - xc;
    else if (MODE == MODE_JAC) o = fma(omega, bv - xc, xc);
    else o = omega * bv;
    y[idx] = o;
    return;
  }
  // stencil weights: own forward coefficients (k >= 4), the neighbours' mirrored ones (k < 4)
  const long long P = g.P;
  const double* Mb = op.st;
  const double* Kb = op.st + 5 * P;
  double wM[9], wK[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const int dx = (k % 3) - 1, dy = (k / 3) - 1;
    if (k >= 4) {
      wM[k] = __ldg(Mb + (k - 4) * P + pn);
      wK[k] = __ldg(Kb + (k - 4) * P + pn);
    } else {
      const int ni = i + dx, nj = j + dy;
      const bool v = ni >= 0 && ni <= n && nj >= 0 && nj <= n;
      const long long q = v ? (long long)nj * g.pr + ni : 0;
      wM[k] = v ? __ldg(Mb + (8 - k - 4) * P + q) : 0.0;
      wK[k] = v ? __ldg(Kb + (8 - k - 4) * P + q) : 0.0;
    }
  }
  // M x and K x on planes p-1, p, p+1 (x = 0 outside the domain and on the t = 0 plane)
  double Mx[3] = {0.0, 0.0, 0.0}, Kx[3] = {0.0, 0.0, 0.0};
  if (NX) {
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const int q = p - 1 + s;
      if (q < 0 || q > g.nt || q + g.pg0 == 0) continue;
      const double* xq = x + (long long)q * P;
      double m = 0.0, kk = 0.0;
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        const int ni = i + (k % 3) - 1, nj = j + (k / 3) - 1;
        const double v = (ni >= 0 && ni <= n && nj >= 0 && nj <= n) ? __ldg(xq + (long long)nj * g.pr + ni) : 0.0;
        m = fma(wM[k], v, m);
        kk = fma(wK[k], v, kk);
      }
      Mx[s] = m;
      Kx[s] = kk;
    }
  }
  const bool lay = p < g.nt;  // layer p (above plane p) exists
  const double (&U)[2][2] = op.U;
  const double (&T)[2][2] = op.Tm;
  // S^{ab} x_q = U[a][b] Mx_q + T[a][b] Kx_q
  auto S = [&](int a, int bb, int s) { return fma(U[a][bb], Mx[s], T[a][bb] * Kx[s]); };
  double Ax = TRANS ? S(0, 1, 0) + S(1, 1, 1) : S(1, 0, 0) + S(1, 1, 1);
  if (lay) Ax += TRANS ? S(0, 0, 1) + S(1, 0, 2) : S(0, 0, 1) + S(0, 1, 2);
  double o;
  if (MODE == MODE_APPLY) {
    o = Ax;
  } else if (MODE == MODE_RESID) {
    o = bv - Ax;
  } else {
    const double D = fma(U[1][1], wM[4], T[1][1] * wK[4]) + (lay ? fma(U[0][0], wM[4], T[0][0] * wK[4]) : 0.0);
    const double od = omega / D;
    o = (MODE == MODE_JAC) ? fma(od, bv - Ax, __ldg(x + idx)) : od * bv;
  }
  y[idx] = o;
}

template <int MODE>
void lt(const OpDesc& op, bool trans, const double* x, const double* b, double* y, double omega, cudaStream_t s) {
  const unsigned grid = (unsigned)((op.g.N + 255) / 256);
  if (trans) tiny2d_kernel<MODE, true><<<grid, 256, 0, s>>>(op, x, b, y, omega);
  else tiny2d_kernel<MODE, false><<<grid, 256, 0, s>>>(op, x, b, y, omega);
}

}  // namespace

// Masked operator of a replicated time-constant (2+1)D level with stored M, K; false if not covered.
bool launch_op_tiny2d(const OpDesc& op, int mode, bool trans, bool mask, const double* x, const double* b, double* y,
                      double omega, cudaStream_t s) {
  if (op.g.sd != 2 || !mask || op.form != FORM_MK || op.tvl) return false;
  switch (mode) {
    case MODE_APPLY: lt<MODE_APPLY>(op, trans, x, b, y, omega, s); break;
    case MODE_RESID: lt<MODE_RESID>(op, trans, x, b, y, omega, s); break;
    case MODE_JAC: lt<MODE_JAC>(op, trans, x, b, y, omega, s); break;
    default: lt<MODE_JAC0>(op, trans, x, b, y, omega, s); break;
  }
  return true;
}

}  // namespace st
