// vsmall.cu — the small-level tail of the V-cycle in ONE kernel launch.
//
// Below ~24K nodes a level's kernels are pure launch / pipeline latency (~6 us each whatever the
// size; config 2 has 4-7 such levels, ~9 launches per level and V-cycle). Two variants walk the same
// sequence the host V-cycle issues — pre-smoothing (first sweep from zero), residual, restriction,
// ..., the dense coarsest solve, prolongation + correction, post-smoothing:
//   * SM (`launch_vtail`, opt-in ST_VTAIL=1): one CTA of 512 threads with every level vector of the tail in
//     shared memory (x and b per level; one residual and one ping-pong scratch shared by all levels),
//     __syncthreads between phases. Level l0's b is copied in from global memory and its x out.
//   * cluster (`launch_vsmall`, opt-in ST_VSMALL=1): a thread-block cluster, vectors read through L2
//     (ld.global.cg) between cluster barriers.
// Both are measured slower than the per-level kernels inside the V-cycle's CUDA graph (DESIGN.md
// sec. 9) and are kept as experiments.
// Stencils, the coarsest inverse and the level descriptors are read-only global data. Same operator
// algebra as the generic kernels (opcore.cuh): the results equal the per-level launches up to
// summation order.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"
#include "opcore.cuh"

namespace cg = cooperative_groups;

namespace st {

namespace {

constexpr int VS_THREADS = 256;  // 255 registers per thread: the per-node rows of B4 levels are register-heavy
constexpr int VT_THREADS = 512;

// vector load: shared memory (SM) or through L2 (vectors written earlier in the same kernel)
template <bool SM>
__device__ __forceinline__ double ldv(const double* p) {
  if (SM) return *p;
  return __ldcg(p);
}

// one row of the masked level operator in mode `mode` (APPLY, RESID, JAC, JAC0)
template <int SD, int FORM, bool TRANS, bool SM>
__device__ double node_row(const OpDesc& op, int mode, const double* x, const double* b, int p, const int* c,
                           long long pn, double omega) {
  constexpr int NOFF = SG<SD>::NOFF;
  const Geom& g = op.g;
  const long long gi = (long long)p * g.P + pn;
  const double bv = (mode != MODE_APPLY) ? ldv<SM>(b + gi) : 0.0;
  if (is_cons<SD>(g, c, p)) {
    const double xc = (mode != MODE_JAC0) ? ldv<SM>(x + gi) : 0.0;
    if (mode == MODE_APPLY) return xc;
    if (mode == MODE_RESID) return bv - xc;
    if (mode == MODE_JAC) return xc + omega * (bv - xc);
    return omega * bv;
  }
  double xm[NOFF], x0[NOFF], xp[NOFF];
  if (mode != MODE_JAC0) {
    if (p >= 1) load_nb<SD, true, !SM, SM>(g, x, c, p - 1, xm);
    load_nb<SD, true, !SM, SM>(g, x, c, p, x0);
    if (p < g.nt) load_nb<SD, true, !SM, SM>(g, x, c, p + 1, xp);
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
  if (mode == MODE_JAC) return ldv<SM>(x + gi) + omega * (bv - Ax) / D;
  return omega * bv / D;
}

template <int SD, bool TRANS, bool SM>
__device__ void op_phase(const SmallLevel& L, int mode, const double* x, const double* b, double* y, int t0, int nth) {
  const Geom& g = L.op.g;
  for (long long idx = t0; idx < g.N; idx += nth) {
    const int p = (int)(idx / g.P);
    const long long pn = idx % g.P;
    int c[3] = {0, 0, 0};
    if (!pdecode<SD>(g, pn, c)) continue;  // pads stay zero
    double v;
    if (L.op.form == FORM_MK) v = node_row<SD, FORM_MK, TRANS, SM>(L.op, mode, x, b, p, c, pn, L.omega);
    else v = node_row<SD, FORM_B4, TRANS, SM>(L.op, mode, x, b, p, c, pn, L.omega);
    y[idx] = v;
  }
}

// restriction r_c = m_f^c P^T r_f of coarse node idx (transfer.cu, global plane numbering)
template <int SD, bool SM>
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
        if (ok) acc += w * ldv<SM>(rp + pidx<SD>(gf, f));
      }
    }
    rc[idx] = acc;
  }
}

// prolongation + correction x_f += m_f P e_c of fine node idx
template <int SD, bool SM>
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
        if (ok) acc += w * ldv<SM>(ep + pidx<SD>(gc, C));
      }
    }
    xf[idx] = ldv<SM>(xf + idx) + acc;
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
    op_phase<SD, TRANS, false>(L, MODE_JAC0, nullptr, L.b, cur, t0, nth);
    cl.sync();
    for (int s = 1; s < cyc.npre; ++s) {
      op_phase<SD, TRANS, false>(L, MODE_JAC, cur, L.b, oth, t0, nth);
      cl.sync();
      double* tmp = cur; cur = oth; oth = tmp;
    }
    op_phase<SD, TRANS, false>(L, MODE_RESID, cur, L.b, L.r, t0, nth);
    cl.sync();
    const SmallLevel& N = cyc.L[l + 1];
    restrict_phase<SD, false>(L.op.g, N.op.g, N.kind, L.r, N.b, t0, nth);
    cl.sync();
    curs[l] = cur;
  }
  for (l = l - 1; l >= 0; --l) {
    const SmallLevel& L = cyc.L[l];
    const SmallLevel& N = cyc.L[l + 1];
    double* cur = curs[l];
    double* oth = (cur == L.x) ? L.t : L.x;
    prolong_phase<SD, false>(L.op.g, N.op.g, N.kind, N.x, cur, t0, nth);
    cl.sync();
    for (int s = 0; s < cyc.npost; ++s) {
      op_phase<SD, TRANS, false>(L, MODE_JAC, cur, L.b, oth, t0, nth);
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

// Single-CTA tail with every vector in shared memory: smem = [x_0 b_0 | x_1 b_1 | ... | r | t] with
// level k's vectors of op.g.N doubles; r (residual) and t (Jacobi ping-pong) are shared by all
// levels — a level's pre-smoothing starts in the buffer that makes it end in x (t is free during
// the recursion); an odd post-smoothing count ends in t and is copied back.
template <int SD, bool TRANS>
__global__ void __launch_bounds__(VT_THREADS) vtail_kernel(const __grid_constant__ SmallCycle cyc) {
  extern __shared__ double sv[];
  const int t0 = threadIdx.x, nth = blockDim.x;
  double* xs[kMaxSmall];
  double* bs[kMaxSmall];
  long long off = 0, nmax = 0;
  for (int k = 0; k < cyc.nlev; ++k) {
    const long long n = cyc.L[k].op.g.N;
    xs[k] = sv + off;
    bs[k] = sv + off + n;
    off += 2 * n;
    nmax = n > nmax ? n : nmax;
  }
  double* rsc = sv + off;
  double* tsc = rsc + nmax;
  {  // level 0's right-hand side from global memory
    const long long n0 = cyc.L[0].op.g.N;
    for (long long i = t0; i < n0; i += nth) bs[0][i] = __ldcg(cyc.L[0].b + i);
  }
  __syncthreads();
  int l = 0;
  for (; l < cyc.nlev; ++l) {
    const SmallLevel& L = cyc.L[l];
    if (L.dense) {  // x = A^-1 b (transpose for the adjoint)
      const int N = (int)L.op.g.N;
      for (int row = t0; row < N; row += nth) {
        double acc = 0.0;
        if (!TRANS)
          for (int j = 0; j < N; ++j) acc += __ldg(L.Ainv + (long long)row * N + j) * bs[l][j];
        else
          for (int j = 0; j < N; ++j) acc += __ldg(L.Ainv + (long long)j * N + row) * bs[l][j];
        xs[l][row] = acc;
      }
      __syncthreads();
      break;
    }
    double* cur = (cyc.npre % 2 == 1) ? xs[l] : tsc;
    double* oth = (cur == xs[l]) ? tsc : xs[l];
    op_phase<SD, TRANS, true>(L, MODE_JAC0, nullptr, bs[l], cur, t0, nth);
    __syncthreads();
    for (int s = 1; s < cyc.npre; ++s) {
      op_phase<SD, TRANS, true>(L, MODE_JAC, cur, bs[l], oth, t0, nth);
      __syncthreads();
      double* tmp = cur; cur = oth; oth = tmp;
    }
    op_phase<SD, TRANS, true>(L, MODE_RESID, cur, bs[l], rsc, t0, nth);
    __syncthreads();
    const SmallLevel& N = cyc.L[l + 1];
    restrict_phase<SD, true>(L.op.g, N.op.g, N.kind, rsc, bs[l + 1], t0, nth);
    __syncthreads();
  }
  for (l = l - 1; l >= 0; --l) {
    const SmallLevel& L = cyc.L[l];
    const SmallLevel& N = cyc.L[l + 1];
    double* cur = xs[l];
    double* oth = tsc;
    prolong_phase<SD, true>(L.op.g, N.op.g, N.kind, xs[l + 1], cur, t0, nth);
    __syncthreads();
    for (int s = 0; s < cyc.npost; ++s) {
      op_phase<SD, TRANS, true>(L, MODE_JAC, cur, bs[l], oth, t0, nth);
      __syncthreads();
      double* tmp = cur; cur = oth; oth = tmp;
    }
    if (cur != xs[l]) {
      for (long long i = t0; i < L.op.g.N; i += nth) xs[l][i] = cur[i];
      __syncthreads();
    }
  }
  const long long n0 = cyc.L[0].op.g.N;
  for (long long i = t0; i < n0; i += nth) cyc.L[0].x[i] = xs[0][i];
}

}  // namespace

// dynamic shared memory of the single-CTA tail of `cyc` (bytes)
size_t vtail_smem_bytes(const SmallCycle& cyc) {
  long long off = 0, nmax = 0;
  for (int k = 0; k < cyc.nlev; ++k) {
    off += 2 * cyc.L[k].op.g.N;
    nmax = cyc.L[k].op.g.N > nmax ? cyc.L[k].op.g.N : nmax;
  }
  return (size_t)(off + 2 * nmax) * sizeof(double);
}

void launch_vtail(const SmallCycle& cyc, int sd, bool trans, cudaStream_t s) {
  const size_t bytes = vtail_smem_bytes(cyc);
  static bool attr[4] = {false, false, false, false};  // one per instantiation (same pointer type)
  void (*kern)(SmallCycle) = sd == 2 ? (trans ? vtail_kernel<2, true> : vtail_kernel<2, false>)
                                     : (trans ? vtail_kernel<3, true> : vtail_kernel<3, false>);
  const int id = (sd == 2 ? 0 : 2) + (trans ? 1 : 0);
  if (!attr[id]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr[id] = true;
  }
  kern<<<1, VT_THREADS, bytes, s>>>(cyc);
}

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
