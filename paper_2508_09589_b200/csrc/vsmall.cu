// vsmall.cu — the small-level tail of the V-cycle as ONE thread-block-cluster kernel.
//
// Below ~24K nodes a level's kernels are pure launch / pipeline latency (~7 us each whatever the
// size; config 2 has 7 such levels, ~70 launches per V-cycle). Here a cluster of CTAs walks the
// same sequence the host V-cycle issues — pre-smoothing (first sweep from zero), residual,
// restriction, ..., the dense coarsest solve, prolongation + correction, post-smoothing — with a
// cluster barrier (release / acquire) between phases. Level vectors are read through L2
// (ld.global.cg) because they are written inside the kernel; stencils, the coarsest inverse and the
// level descriptors are read-only. Same operator algebra as the generic kernels (opcore.cuh), so the
// results equal the per-level launches up to summation order.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"
#include "opcore.cuh"

namespace cg = cooperative_groups;

namespace st {

namespace {

constexpr int VS_THREADS = 256;  // 255 registers per thread: the per-node rows of B4 levels are register-heavy

// one row of the masked level operator in mode `mode` (APPLY, RESID, JAC, JAC0)
template <int SD, int FORM, bool TRANS>
__device__ double node_row(const OpDesc& op, int mode, const double* x, const double* b, int p, const int* c,
                           long long pn, double omega) {
  constexpr int NOFF = SG<SD>::NOFF;
  const Geom& g = op.g;
  const long long gi = (long long)p * g.P + pn;
  const double bv = (mode != MODE_APPLY) ? __ldcg(b + gi) : 0.0;
  if (is_cons<SD>(g, c, p)) {
    const double xc = (mode != MODE_JAC0) ? __ldcg(x + gi) : 0.0;
    if (mode == MODE_APPLY) return xc;
    if (mode == MODE_RESID) return bv - xc;
    if (mode == MODE_JAC) return xc + omega * (bv - xc);
    return omega * bv;
  }
  double xm[NOFF], x0[NOFF], xp[NOFF];
  if (mode != MODE_JAC0) {
    if (p >= 1) load_nb<SD, true, true>(g, x, c, p - 1, xm);
    load_nb<SD, true, true>(g, x, c, p, x0);
    if (p < g.nt) load_nb<SD, true, true>(g, x, c, p + 1, xp);
  } else {
#pragma unroll
    for (int k = 0; k < NOFF; ++k) xm[k] = x0[k] = xp[k] = 0.0;
  }
  double Ax = 0.0, D = 0.0, bot, top, db, dt;
  if (p >= 1) {
    layer_eval<SD, FORM, TRANS, true, true>(op, c, pn, p - 1, xm, x0, bot, top, db, dt);
    Ax += top;
    D += dt;
  }
  if (p < g.nt) {
    layer_eval<SD, FORM, TRANS, true, true>(op, c, pn, p, x0, xp, bot, top, db, dt);
    Ax += bot;
    D += db;
  }
  if (mode == MODE_APPLY) return Ax;
  if (mode == MODE_RESID) return bv - Ax;
  if (mode == MODE_JAC) return __ldcg(x + gi) + omega * (bv - Ax) / D;
  return omega * bv / D;
}

template <int SD, bool TRANS>
__device__ void op_phase(const SmallLevel& L, int mode, const double* x, const double* b, double* y, int t0, int nth) {
  const Geom& g = L.op.g;
  for (long long idx = t0; idx < g.N; idx += nth) {
    const int p = (int)(idx / g.P);
    const long long pn = idx % g.P;
    int c[3] = {0, 0, 0};
    if (!pdecode<SD>(g, pn, c)) continue;  // pads stay zero
    double v;
    if (L.op.form == FORM_MK) v = node_row<SD, FORM_MK, TRANS>(L.op, mode, x, b, p, c, pn, L.omega);
    else v = node_row<SD, FORM_B4, TRANS>(L.op, mode, x, b, p, c, pn, L.omega);
    y[idx] = v;
  }
}

// restriction r_c = m_f^c P^T r_f of coarse node idx (transfer.cu, global plane numbering)
template <int SD>
__device__ void restrict_phase(const Geom& gf, const Geom& gc, int kind, const double* rf, double* rc, int t0,
                               int nth) {
  const bool SP = kind == KIND_SPACE || kind == KIND_FULL, TM = kind == KIND_TIME || kind == KIND_FULL;
  for (long long idx = t0; idx < gc.N; idx += nth) {
    const int P = (int)(idx / gc.P);
    const long long pc = idx % gc.P;
    int C[3] = {0, 0, 0};
    if (!pdecode<SD>(gc, pc, C) || is_cons<SD>(gc, C, P)) { rc[idx] = 0.0; continue; }
    const int Pg = P + gc.pg0;
    double acc = 0.0;
    for (int at = (TM ? -1 : 0); at <= (TM ? 1 : 0); ++at) {
      const int q = (TM ? 2 * Pg + at : Pg) - gf.pg0;
      if (q < 0 || q > gf.nt) continue;
      const double wt = (at == 0) ? 1.0 : 0.5;
      const double* rp = rf + (long long)q * gf.P;
      const int NS = SP ? SG<SD>::NOFF : 1;
      for (int k = 0; k < NS; ++k) {
        int f[3] = {0, 0, 0};
        bool ok = true;
        double w = wt;
        for (int d = 0; d < SD; ++d) {
          const int o = SP ? SG<SD>::od(k, d) : 0;
          f[d] = SP ? 2 * C[d] + o : C[d];
          ok = ok && f[d] >= 0 && f[d] < gf.nn;
          w *= (o == 0) ? 1.0 : 0.5;
        }
        if (ok) acc += w * __ldcg(rp + pidx<SD>(gf, f));
      }
    }
    rc[idx] = acc;
  }
}

// prolongation + correction x_f += m_f P e_c of fine node idx
template <int SD>
__device__ void prolong_phase(const Geom& gf, const Geom& gc, int kind, const double* ec, double* xf, int t0, int nth) {
  const bool SP = kind == KIND_SPACE || kind == KIND_FULL, TM = kind == KIND_TIME || kind == KIND_FULL;
  for (long long idx = t0; idx < gf.N; idx += nth) {
    const int p = (int)(idx / gf.P);
    const long long pf = idx % gf.P;
    int c[3] = {0, 0, 0};
    if (!pdecode<SD>(gf, pf, c) || is_cons<SD>(gf, c, p)) continue;
    const int pg = p + gf.pg0;
    const int P0 = (TM ? (pg >> 1) : pg) - gc.pg0;
    const int nP = (TM && (pg & 1)) ? 2 : 1;
    double acc = 0.0;
    for (int it = 0; it < nP; ++it) {
      const int Pq = P0 + it;
      if (Pq < 0 || Pq > gc.nt) continue;
      const double wt = (nP == 2) ? 0.5 : 1.0;
      const double* ep = ec + (long long)Pq * gc.P;
      int lo[3] = {0, 0, 0}, cnt[3] = {1, 1, 1};
      for (int d = 0; d < SD; ++d) {
        if (SP) { lo[d] = c[d] >> 1; cnt[d] = (c[d] & 1) ? 2 : 1; }
        else lo[d] = c[d];
      }
      for (int m = 0; m < (1 << SD); ++m) {
        int C[3] = {0, 0, 0};
        bool ok = true;
        double w = wt;
        for (int d = 0; d < SD; ++d) {
          const int bit = (m >> d) & 1;
          if (bit >= cnt[d]) ok = false;
          C[d] = lo[d] + bit;
          w *= (cnt[d] == 2) ? 0.5 : 1.0;
        }
        if (ok) acc += w * __ldcg(ep + pidx<SD>(gc, C));
      }
    }
    xf[idx] = __ldcg(xf + idx) + acc;
  }
}

template <int SD, bool TRANS>
__global__ void __launch_bounds__(VS_THREADS) vsmall_kernel(const __grid_constant__ SmallCycle cyc) {
  cg::cluster_group cl = cg::this_cluster();
  const int nth = (int)(blockDim.x * cl.num_blocks());
  const int t0 = (int)(cl.block_rank() * blockDim.x + threadIdx.x);
  const int total = cyc.npre + cyc.npost;
  double* curs[kMaxSmall];
  int l = 0;
  for (; l < cyc.nlev; ++l) {
    const SmallLevel& L = cyc.L[l];
    if (L.dense) {  // x = A^-1 b (transpose for the adjoint), rows strided over the cluster
      const int N = (int)L.op.g.N;
      for (int row = t0; row < N; row += nth) {
        double acc = 0.0;
        if (!TRANS)
          for (int j = 0; j < N; ++j) acc += __ldg(L.Ainv + (long long)row * N + j) * __ldcg(L.b + j);
        else
          for (int j = 0; j < N; ++j) acc += __ldg(L.Ainv + (long long)j * N + row) * __ldcg(L.b + j);
        L.x[row] = acc;
      }
      cl.sync();
      break;
    }
    double* cur = (total % 2 == 1) ? L.x : L.t;
    double* oth = (cur == L.x) ? L.t : L.x;
    op_phase<SD, TRANS>(L, MODE_JAC0, nullptr, L.b, cur, t0, nth);
    cl.sync();
    for (int s = 1; s < cyc.npre; ++s) {
      op_phase<SD, TRANS>(L, MODE_JAC, cur, L.b, oth, t0, nth);
      cl.sync();
      double* tmp = cur; cur = oth; oth = tmp;
    }
    op_phase<SD, TRANS>(L, MODE_RESID, cur, L.b, L.r, t0, nth);
    cl.sync();
    const SmallLevel& N = cyc.L[l + 1];
    restrict_phase<SD>(L.op.g, N.op.g, N.kind, L.r, N.b, t0, nth);
    cl.sync();
    curs[l] = cur;
  }
  for (l = l - 1; l >= 0; --l) {
    const SmallLevel& L = cyc.L[l];
    const SmallLevel& N = cyc.L[l + 1];
    double* cur = curs[l];
    double* oth = (cur == L.x) ? L.t : L.x;
    prolong_phase<SD>(L.op.g, N.op.g, N.kind, N.x, cur, t0, nth);
    cl.sync();
    for (int s = 0; s < cyc.npost; ++s) {
      op_phase<SD, TRANS>(L, MODE_JAC, cur, L.b, oth, t0, nth);
      cl.sync();
      double* tmp = cur; cur = oth; oth = tmp;
    }
  }
}

template <int SD, bool TRANS>
cudaError_t launch_vs(const SmallCycle& cyc, cudaStream_t s, int cluster) {
  auto kern = vsmall_kernel<SD, TRANS>;
  static int tried16 = 0;
  if (cluster > 8 && !tried16) {
    tried16 = 1;
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cluster, 1, 1);
  cfg.blockDim = dim3(VS_THREADS, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, cyc);
}

}  // namespace

// The levels of `cyc` must be replicated (no slab communication), the last one dense. Tries a
// 16-CTA (non-portable) cluster, then 8.
void launch_vsmall(const SmallCycle& cyc, int sd, bool trans, cudaStream_t s) {
  static int cl = 16;
  for (;;) {
    cudaError_t e;
    if (sd == 2) e = trans ? launch_vs<2, true>(cyc, s, cl) : launch_vs<2, false>(cyc, s, cl);
    else e = trans ? launch_vs<3, true>(cyc, s, cl) : launch_vs<3, false>(cyc, s, cl);
    if (e == cudaSuccess || cl <= 8) return;
    cudaGetLastError();
    cl = 8;
  }
}

}  // namespace st
