// transfer.cu — multigrid transfers between semi-coarsened levels.
// Prolongation P: linear interpolation along each coarsened direction (space: bi/trilinear,
// weights 1 and 1/2; time: 1 and 1/2 — non-causal). Restriction = P^T.
// Dirichlet masks: restriction output zero at coarse
// constrained nodes; prolongation never updates fine constrained nodes. Planes are mapped in
// global numbering (Geom::pg0), so a time slab can restrict into / prolong from a coarse slab
// or a replicated (agglomerated) coarse level.
#include "common.cuh"
#include "kernels.h"

namespace st {

template <int SD, bool SP, bool TM>
__global__ void restrict_kernel(Geom gf, Geom gc, const double* __restrict__ rf, double* __restrict__ rc) {
  long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= gc.N) return;
  int P = (int)(idx / gc.P);
  long long pc = idx % gc.P;
  int C[3] = {0, 0, 0};
  if (!pdecode<SD>(gc, pc, C) || is_cons<SD>(gc, C, P)) { rc[idx] = 0.0; return; }
  constexpr int NS = SP ? SG<SD>::NOFF : 1;
  const int Pg = P + gc.pg0;  // global coarse plane; fine planes in global numbering, then local
  double acc = 0.0;
#pragma unroll
  for (int at = (TM ? -1 : 0); at <= (TM ? 1 : 0); ++at) {
    int q = (TM ? 2 * Pg + at : Pg) - gf.pg0;
    if (q < 0 || q > gf.nt) continue;
    double wt = (at == 0) ? 1.0 : 0.5;
    const double* rp = rf + (long long)q * gf.P;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      int f[3] = {0, 0, 0};
      bool ok = true;
      double w = wt;
#pragma unroll
      for (int d = 0; d < SD; ++d) {
        int o = SP ? SG<SD>::od(k, d) : 0;
        f[d] = SP ? 2 * C[d] + o : C[d];
        ok = ok && f[d] >= 0 && f[d] < gf.nn;
        w *= (o == 0) ? 1.0 : 0.5;
      }
      if (ok) acc += w * __ldg(rp + pidx<SD>(gf, f));
    }
  }
  rc[idx] = acc;
}

template <int SD, bool SP, bool TM>
__global__ void prolong_kernel(Geom gf, Geom gc, const double* __restrict__ ec, double* __restrict__ xf) {
  long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= gf.N) return;
  int p = (int)(idx / gf.P);
  long long pf = idx % gf.P;
  int c[3] = {0, 0, 0};
  if (!pdecode<SD>(gf, pf, c) || is_cons<SD>(gf, c, p)) return;
  // time part (global plane numbering on both grids)
  const int pg = p + gf.pg0;
  int P0 = (TM ? (pg >> 1) : pg) - gc.pg0;
  int nP = (TM && (pg & 1)) ? 2 : 1;
  double acc = 0.0;
  for (int it = 0; it < nP; ++it) {
    int Pq = P0 + it;
    if (Pq < 0 || Pq > gc.nt) continue;  // only ghost rows of a slab can reach past the coarse slab
    double wt = (nP == 2) ? 0.5 : 1.0;
    const double* ep = ec + (long long)Pq * gc.P;
    // space part: corners of the coarse cell
    int lo[3] = {0, 0, 0}, cnt[3] = {1, 1, 1};
#pragma unroll
    for (int d = 0; d < SD; ++d) {
      if (SP) { lo[d] = c[d] >> 1; cnt[d] = (c[d] & 1) ? 2 : 1; }
      else lo[d] = c[d];
    }
    for (int m = 0; m < (1 << SD); ++m) {
      int C[3] = {0, 0, 0};
      bool ok = true;
      double w = wt;
#pragma unroll
      for (int d = 0; d < SD; ++d) {
        int bit = (m >> d) & 1;
        if (bit >= cnt[d]) ok = false;
        C[d] = lo[d] + bit;
        w *= (cnt[d] == 2) ? 0.5 : 1.0;
      }
      if (!ok) continue;
      acc += w * __ldg(ep + pidx<SD>(gc, C));
    }
  }
  xf[idx] += acc;
}

// (2+1)D space coarsening, the hot transfer pair: thread per (x1 node, x2 row, plane), no 64-bit
// index arithmetic; rows are read coalesced and the coarse row of the prolongation comes from L1.
__global__ void __launch_bounds__(128) prolong2s_kernel(Geom gf, Geom gc, const double* __restrict__ ec,
                                                        double* __restrict__ xf) {
  const int i = blockIdx.x * 128 + threadIdx.x, j = blockIdx.y, p = blockIdx.z;
  if (i >= gf.nn) return;
  int c[3] = {i, j, 0};
  if (is_cons<2>(gf, c, p)) return;
  const int Pc = p + gf.pg0 - gc.pg0;
  if (Pc < 0 || Pc > gc.nt) return;
  const double* e0 = ec + (long long)Pc * gc.P + (long long)(j >> 1) * gc.pr + (i >> 1);
  double v;
  if (!(i & 1) && !(j & 1)) v = __ldg(e0);
  else if (!(j & 1)) v = 0.5 * (__ldg(e0) + __ldg(e0 + 1));
  else if (!(i & 1)) v = 0.5 * (__ldg(e0) + __ldg(e0 + gc.pr));
  else v = 0.25 * ((__ldg(e0) + __ldg(e0 + 1)) + (__ldg(e0 + gc.pr) + __ldg(e0 + gc.pr + 1)));
  xf[(long long)p * gf.P + (long long)j * gf.pr + i] += v;
}

__global__ void __launch_bounds__(128) restrict2s_kernel(Geom gf, Geom gc, const double* __restrict__ rf,
                                                         double* __restrict__ rc) {
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
    restrict2s_kernel<<<dim3((gc.pr + 127) / 128, gc.nn, gc.nt + 1), 128, 0, s>>>(gf, gc, rf, rc);
    return;
  }
  int blk = 256;
  unsigned grd = (unsigned)((gc.N + blk - 1) / blk);
  bool SPc = (kind == KIND_SPACE || kind == KIND_FULL), TMc = (kind == KIND_TIME || kind == KIND_FULL);
#define R(SD, A, B) restrict_kernel<SD, A, B><<<grd, blk, 0, s>>>(gf, gc, rf, rc)
  if (gf.sd == 2) {
    if (SPc && TMc) R(2, true, true); else if (SPc) R(2, true, false); else R(2, false, true);
  } else {
    if (SPc && TMc) R(3, true, true); else if (SPc) R(3, true, false); else R(3, false, true);
  }
#undef R
}

void launch_prolong_add(const Geom& gf, const Geom& gc, int kind, const double* ec, double* xf, cudaStream_t s) {
  if (gf.sd == 2 && kind == KIND_SPACE && gf.nt + 1 <= 65535) {
    prolong2s_kernel<<<dim3((gf.nn + 127) / 128, gf.nn, gf.nt + 1), 128, 0, s>>>(gf, gc, ec, xf);
    return;
  }
  int blk = 256;
  unsigned grd = (unsigned)((gf.N + blk - 1) / blk);
  bool SPc = (kind == KIND_SPACE || kind == KIND_FULL), TMc = (kind == KIND_TIME || kind == KIND_FULL);
#define PR(SD, A, B) prolong_kernel<SD, A, B><<<grd, blk, 0, s>>>(gf, gc, ec, xf)
  if (gf.sd == 2) {
    if (SPc && TMc) PR(2, true, true); else if (SPc) PR(2, true, false); else PR(2, false, true);
  } else {
    if (SPc && TMc) PR(3, true, true); else if (SPc) PR(3, true, false); else PR(3, false, true);
  }
#undef PR
}

}  // namespace st
