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

void launch_restrict(const Geom& gf, const Geom& gc, int kind, const double* rf, double* rc, cudaStream_t s) {
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
