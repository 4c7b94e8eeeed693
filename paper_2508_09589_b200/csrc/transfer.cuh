// transfer.cuh — per-entry multigrid transfers: restriction r_c = m_f^c P^T r_f and
// prolongation x_f += m_f P e_c between semi-coarsened levels, used by the transfer kernels
// (transfer.cu). Planes in global numbering (Geom::pg0).
#pragma once
#include "common.cuh"
#include "opcore.cuh"

namespace st {

// one coarse entry idx of r_c = m_f^c P^T r_f
template <int SD, bool SP, bool TM>
__device__ __forceinline__ void restrict_node(const Geom& gf, const Geom& gc, const double* __restrict__ rf,
                                              double* __restrict__ rc, long long idx) {
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

// one fine entry idx of x_f += m_f P e_c
template <int SD, bool SP, bool TM>
__device__ __forceinline__ void prolong_node(const Geom& gf, const Geom& gc, const double* __restrict__ ec,
                                             double* __restrict__ xf, long long idx) {
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

}  // namespace st
