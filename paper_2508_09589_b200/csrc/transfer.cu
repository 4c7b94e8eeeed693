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

// (3+1)D space coarsening, prolongation (the level-0 transfer of config 4): one thread per coarse node
// (I, J, K) of a plane loads its 8 coarse corners once and updates the 2 x 2 x 2 fine nodes from
// (2I, 2J, 2K) as four 16-byte pairs (trilinear weights 1, 1/2, 1/4, 1/8); no 64-bit
// index arithmetic per fine node. Fine nodes past the last node and constrained fine nodes are left alone.
__global__ void __launch_bounds__(128) prolong3s_kernel(Geom gf, Geom gc, const double* __restrict__ ec,
                                                        double* __restrict__ xf) {
  pdl_wait();
  const int ij = blockIdx.x * 128 + threadIdx.x, K = blockIdx.y, p = blockIdx.z;
  if (ij >= gc.nn * gc.nn) return;
  const int I = ij % gc.nn, J = ij / gc.nn;
  if (p + gf.pg0 == 0) return;  // initial-condition plane: constrained
  const int Pc = p + gf.pg0 - gc.pg0;
  if (Pc < 0 || Pc > gc.nt) return;
  const long long rsc = (long long)gc.pr * gc.nn, rsf = (long long)gf.pr * gf.nn;  // slice strides
  const double* e0 = ec + (long long)Pc * gc.P + (long long)K * rsc + (long long)J * gc.pr + I;
  const bool hx = I + 1 < gc.nn, hy = J + 1 < gc.nn, hz = K + 1 < gc.nn;  // fine 2I+1 / 2J+1 / 2K+1 exist
  double e[2][2][2];  // [dz][dy][dx]
#pragma unroll
  for (int dz = 0; dz < 2; ++dz)
#pragma unroll
    for (int dy = 0; dy < 2; ++dy)
#pragma unroll
      for (int dx = 0; dx < 2; ++dx) {
        const bool ok = (!dx || hx) && (!dy || hy) && (!dz || hz);
        e[dz][dy][dx] = ok ? __ldg(e0 + dz * rsc + dy * gc.pr + dx) : 0.0;
      }
  double* x0 = xf + (long long)p * gf.P + (long long)(2 * K) * rsf + (long long)(2 * J) * gf.pr + 2 * I;
#pragma unroll
  for (int fz = 0; fz < 2; ++fz) {
    if (fz && !hz) continue;
#pragma unroll
    for (int fy = 0; fy < 2; ++fy) {
      if (fy && !hy) continue;
      // sums over the coarse corners the fine node (.., 2J+fy, 2K+fz) sees, at dx = 0 and dx = 1
      double s0 = e[0][0][0], s1 = e[0][0][1];
      if (fy) { s0 += e[0][1][0]; s1 += e[0][1][1]; }
      if (fz) {
        double t0 = e[1][0][0], t1 = e[1][0][1];
        if (fy) { t0 += e[1][1][0]; t1 += e[1][1][1]; }
        s0 += t0;
        s1 += t1;
      }
      const double w = (fy ? 0.5 : 1.0) * (fz ? 0.5 : 1.0);
      const int fj = 2 * J + fy, fk = 2 * K + fz;
      const bool cons = I == 0 && fj >= gf.plo && fj <= gf.phi && fk >= gf.plo && fk <= gf.phi;  // sink patch
      double2* xp = reinterpret_cast<double2*>(x0 + fz * rsf + (long long)fy * gf.pr);
      double2 v = *xp;
      if (!cons) v.x += w * s0;
      if (hx) v.y += (0.5 * w) * (s0 + s1);
      *xp = v;
    }
  }
}

// Time coarsening (both sd), the transfer pair of every time level: the two grids share the spatial
// grid and its padded layout, so one thread owns a 16-byte pair of one plane (even pitch: pairs never
// straddle a row) and no 64-bit index arithmetic is left per node. Same arithmetic, masks and slab plane
// mapping as restrict_node / prolong_node<SD, false, true>.
template <int SD>
__device__ __forceinline__ void pair_mask(const Geom& g, int off, bool* k0, bool* k1) {
  int c[3] = {off % g.pr, 0, 0};
  const int t = off / g.pr;
  c[1] = t % g.nn;
  c[2] = (SD == 3) ? t / g.nn : 0;
  *k0 = c[0] < g.nn && !is_patch<SD>(g, c);   // real, unconstrained node
  c[0] += 1;
  *k1 = c[0] < g.nn && !is_patch<SD>(g, c);
}

template <int SD>
__global__ void __launch_bounds__(128) prolong_t_kernel(Geom gf, Geom gc, const double* __restrict__ ec,
                                                        double* __restrict__ xf) {
  pdl_wait();
  const int off = 2 * (blockIdx.x * 128 + threadIdx.x), p = blockIdx.y;
  if (off >= gf.P) return;
  const int pg = p + gf.pg0;
  if (pg == 0) return;  // initial-condition plane: constrained
  bool k0, k1;
  pair_mask<SD>(gf, off, &k0, &k1);
  if (!k0 && !k1) return;
  const int P0 = (pg >> 1) - gc.pg0;
  const bool odd = pg & 1;
  const double wt = odd ? 0.5 : 1.0;
  double a0 = 0.0, a1 = 0.0;
  if (P0 >= 0 && P0 <= gc.nt) {
    const double2 e = __ldg(reinterpret_cast<const double2*>(ec + (long long)P0 * gc.P + off));
    a0 += wt * e.x;
    a1 += wt * e.y;
  }
  if (odd && P0 + 1 >= 0 && P0 + 1 <= gc.nt) {
    const double2 e = __ldg(reinterpret_cast<const double2*>(ec + (long long)(P0 + 1) * gc.P + off));
    a0 += wt * e.x;
    a1 += wt * e.y;
  }
  double2* xp = reinterpret_cast<double2*>(xf + (long long)p * gf.P + off);
  double2 v = *xp;
  if (k0) v.x += a0;
  if (k1) v.y += a1;
  *xp = v;
}

template <int SD>
__global__ void __launch_bounds__(128) restrict_t_kernel(Geom gf, Geom gc, const double* __restrict__ rf,
                                                         double* __restrict__ rc) {
  pdl_wait();
  const int off = 2 * (blockIdx.x * 128 + threadIdx.x), P = blockIdx.y;
  if (off >= gc.P) return;
  double2* out = reinterpret_cast<double2*>(rc + (long long)P * gc.P + off);
  const int Pg = P + gc.pg0;
  bool k0, k1;
  pair_mask<SD>(gc, off, &k0, &k1);
  double a0 = 0.0, a1 = 0.0;
  if (Pg != 0 && (k0 || k1)) {
#pragma unroll
    for (int at = -1; at <= 1; ++at) {
      const int q = 2 * Pg + at - gf.pg0;
      if (q < 0 || q > gf.nt) continue;
      const double wt = (at == 0) ? 1.0 : 0.5;
      const double2 r = __ldg(reinterpret_cast<const double2*>(rf + (long long)q * gf.P + off));
      a0 += wt * r.x;
      a1 += wt * r.y;
    }
  }
  *out = make_double2(k0 ? a0 : 0.0, k1 ? a1 : 0.0);
}

// the paired time kernels need the same even-pitch layout on both grids
static bool time_pair_ok(const Geom& gf, const Geom& gc) {
  return gf.pr == gc.pr && gf.P == gc.P && gf.nn == gc.nn && gf.pr % 2 == 0 && gf.P % 2 == 0 &&
         gf.P < (1ll << 30) && gf.nt + 1 <= 65535 && gc.nt + 1 <= 65535;
}

void launch_restrict(const Geom& gf, const Geom& gc, int kind, const double* rf, double* rc, cudaStream_t s) {
  if (gf.sd == 2 && kind == KIND_SPACE && gc.nt + 1 <= 65535) {
    launch_pdl(restrict2s_kernel, dim3((gc.pr + 127) / 128, gc.nn, gc.nt + 1), dim3(128), 0, s, gf, gc, rf, rc);
    return;
  }
  if (kind == KIND_TIME && time_pair_ok(gf, gc)) {
    const dim3 grid((unsigned)((gc.P / 2 + 127) / 128), gc.nt + 1);
    if (gf.sd == 2) launch_pdl(restrict_t_kernel<2>, grid, dim3(128), 0, s, gf, gc, rf, rc);
    else launch_pdl(restrict_t_kernel<3>, grid, dim3(128), 0, s, gf, gc, rf, rc);
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
  if (gf.sd == 3 && kind == KIND_SPACE && gf.nt + 1 <= 65535 && gc.nn <= 65535 && gf.pr % 2 == 0 && !gf.walls) {
    launch_pdl(prolong3s_kernel, dim3((gc.nn * gc.nn + 127) / 128, gc.nn, gf.nt + 1), dim3(128), 0, s, gf, gc, ec, xf);
    return;
  }
  if (kind == KIND_TIME && time_pair_ok(gf, gc)) {
    const dim3 grid((unsigned)((gf.P / 2 + 127) / 128), gf.nt + 1);
    if (gf.sd == 2) launch_pdl(prolong_t_kernel<2>, grid, dim3(128), 0, s, gf, gc, ec, xf);
    else launch_pdl(prolong_t_kernel<3>, grid, dim3(128), 0, s, gf, gc, ec, xf);
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
