// transfer.cu — multigrid transfers between semi-coarsened levels.
// Prolongation P: linear interpolation along each coarsened direction (space: bi/trilinear,
// weights 1 and 1/2; time: 1 and 1/2 — non-causal). Restriction = P^T.
// Dirichlet masks: restriction output zero at coarse
// constrained nodes; prolongation never updates fine constrained nodes. Planes are mapped in
// global numbering (Geom::pg0), so a time slab can restrict into / prolong from a coarse slab
// or a replicated (agglomerated) coarse level.
#include "common.cuh"
#include "kernels.h"
#include "opcore.cuh"
#include "transfer.cuh"

namespace st {

template <int SD, bool SP, bool TM>
__global__ void restrict_kernel(Geom gf, Geom gc, const double* __restrict__ rf, double* __restrict__ rc) {
  pdl_wait();
  long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= gc.N) return;
  restrict_node<SD, SP, TM>(gf, gc, rf, rc, idx);
}

template <int SD, bool SP, bool TM>
__global__ void prolong_kernel(Geom gf, Geom gc, const double* __restrict__ ec, double* __restrict__ xf) {
  pdl_wait();
  long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= gf.N) return;
  prolong_node<SD, SP, TM>(gf, gc, ec, xf, idx);
}

// (2+1)D space coarsening, the hot transfer pair: no 64-bit index arithmetic per node, rows read
// coalesced. Prolongation: one thread per coarse node (I, J) of a plane updates the 2 x 2 fine nodes
// (2I, 2I+1) x (2J, 2J+1) with 16-byte loads / stores of the fine pairs (even pitch: 16-B aligned)
// and the 4 coarse corners loaded once (bilinear weights 1, 1/2, 1/4); fine nodes past
// the last node (the pad column n+1, row n+1) and constrained fine nodes are left alone.
__global__ void __launch_bounds__(128) prolong2s_kernel(Geom gf, Geom gc, const double* __restrict__ ec,
                                                        double* __restrict__ xf) {
  pdl_wait();
  const int I = blockIdx.x * 128 + threadIdx.x, J = blockIdx.y, p = blockIdx.z;
  if (I >= gc.nn) return;
  if (p + gf.pg0 == 0) return;  // initial-condition plane: constrained
  const int Pc = p + gf.pg0 - gc.pg0;
  if (Pc < 0 || Pc > gc.nt) return;
  const double* e0 = ec + (long long)Pc * gc.P + (long long)J * gc.pr + I;
  const bool hx = I + 1 < gc.nn, hy = J + 1 < gc.nn;  // fine column 2I+1 / row 2J+1 exist
  const double e00 = __ldg(e0);
  const double e10 = hx ? __ldg(e0 + 1) : 0.0;
  const double e01 = hy ? __ldg(e0 + gc.pr) : 0.0;
  const double e11 = (hx && hy) ? __ldg(e0 + gc.pr + 1) : 0.0;
  double* x0 = xf + (long long)p * gf.P + (long long)(2 * J) * gf.pr + 2 * I;
  // sink patch: fine node (0, j) with j in [plo, phi] is constrained (R-4)
  const bool m0 = I == 0 && 2 * J >= gf.plo && 2 * J <= gf.phi;
  const bool m1 = I == 0 && 2 * J + 1 >= gf.plo && 2 * J + 1 <= gf.phi;
  {
    double2 v = *reinterpret_cast<const double2*>(x0);
    if (!m0) v.x += e00;
    if (hx) v.y += 0.5 * (e00 + e10);
    *reinterpret_cast<double2*>(x0) = v;
  }
  if (hy) {
    double2 v = *reinterpret_cast<const double2*>(x0 + gf.pr);
    if (!m1) v.x += 0.5 * (e00 + e01);
    if (hx) v.y += 0.25 * ((e00 + e10) + (e01 + e11));
    *reinterpret_cast<double2*>(x0 + gf.pr) = v;
  }
}

__global__ void __launch_bounds__(128) restrict2s_kernel(Geom gf, Geom gc, const double* __restrict__ rf,
                                                         double* __restrict__ rc) {
  pdl_wait();
  const int I = blockIdx.x * 128 + threadIdx.x, J = blockIdx.y, Pp = blockIdx.z;
  if (I >= gc.pr) return;
  double* out = rc + (long long)Pp * gc.P + (long long)J * gc.pr + I;
  int C[3] = {I, J, 0};
  if (I >= gc.nn || is_cons<2>(gc, C, Pp)) { *out = 0.0; return; }
  const int q = Pp + gc.pg0 - gf.pg0;
  if (q < 0 || q > gf.nt) { *out = 0.0; return; }
  const double* rp = rf + (long long)q * gf.P;
  double acc = 0.0;
#pragma unroll
  for (int dy = -1; dy <= 1; ++dy) {
    const int fj = 2 * J + dy;
    if (fj < 0 || fj >= gf.nn) continue;
    const double wy = dy == 0 ? 1.0 : 0.5;
    const double* row = rp + (long long)fj * gf.pr;
    const int fi = 2 * I;
    double r = __ldg(row + fi);
    if (fi - 1 >= 0) r += 0.5 * __ldg(row + fi - 1);
    if (fi + 1 < gf.nn) r += 0.5 * __ldg(row + fi + 1);
    acc += wy * r;
  }
  *out = acc;
}

void launch_restrict(const Geom& gf, const Geom& gc, int kind, const double* rf, double* rc, cudaStream_t s) {
  if (gf.sd == 2 && kind == KIND_SPACE && gc.nt + 1 <= 65535) {
    launch_pdl(restrict2s_kernel, dim3((gc.pr + 127) / 128, gc.nn, gc.nt + 1), dim3(128), 0, s, gf, gc, rf, rc);
    return;
  }
  int blk = 256;
  unsigned grd = (unsigned)((gc.N + blk - 1) / blk);
  bool SPc = (kind == KIND_SPACE || kind == KIND_FULL), TMc = (kind == KIND_TIME || kind == KIND_FULL);
#define R(SD, A, B) launch_pdl(restrict_kernel<SD, A, B>, dim3(grd), dim3(blk), 0, s, gf, gc, rf, rc)
  if (gf.sd == 2) {
    if (SPc && TMc) R(2, true, true); else if (SPc) R(2, true, false); else R(2, false, true);
  } else {
    if (SPc && TMc) R(3, true, true); else if (SPc) R(3, true, false); else R(3, false, true);
  }
#undef R
}

void launch_prolong_add(const Geom& gf, const Geom& gc, int kind, const double* ec, double* xf, cudaStream_t s) {
  int blk = 256;
  unsigned grd = (unsigned)((gf.N + blk - 1) / blk);
  bool SPc = (kind == KIND_SPACE || kind == KIND_FULL), TMc = (kind == KIND_TIME || kind == KIND_FULL);
  // the paired kernel needs an even fine pitch (16-B aligned pairs): every internal vector has one
  if (gf.sd == 2 && kind == KIND_SPACE && gf.nt + 1 <= 65535 && gf.pr % 2 == 0 && gf.P % 2 == 0 && !gf.walls) {
    launch_pdl(prolong2s_kernel, dim3((gc.nn + 127) / 128, gc.nn, gf.nt + 1), dim3(128), 0, s, gf, gc, ec, xf);
    return;
  }
#define PR(SD, A, B) launch_pdl(prolong_kernel<SD, A, B>, dim3(grd), dim3(blk), 0, s, gf, gc, ec, xf)
  if (gf.sd == 2) {
    if (SPc && TMc) PR(2, true, true); else if (SPc) PR(2, true, false); else PR(2, false, true);
  } else {
    if (SPc && TMc) PR(3, true, true); else if (SPc) PR(3, true, false); else PR(3, false, true);
  }
#undef PR
}

}  // namespace st
