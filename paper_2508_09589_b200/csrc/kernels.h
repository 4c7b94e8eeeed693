// kernels.h — host launchers of libst's CUDA kernels (internal).
#pragma once
#include <cuda_runtime.h>
#include "st.h"
#include "common.cuh"

namespace st {

// ops.cu
void launch_op(const OpDesc& op, int mode, bool trans, bool mask, const double* x, const double* b, double* y,
               double omega, cudaStream_t s);
// fast2d.cu: specialised (2+1)D kernels; false if the operator form is not covered
bool launch_op_fast2d(const OpDesc& op, int mode, bool trans, bool mask, const double* x, const double* b, double* y,
                      double omega, cudaStream_t s);
// tma2d.cu: TMA-streamed (2+1)D kernel (fine level, time-constant MK levels)
bool launch_op_tma2d(const OpDesc& op, int mode, bool trans, bool mask, const double* x, const double* b, double* y,
                     double omega, cudaStream_t s);
// tc2d.cu: lean TMA kernel for time-constant levels (fine from rho, stored MK), masked modes
bool launch_op_tc2d(const OpDesc& op, int mode, bool trans, bool mask, const double* x, const double* b, double* y,
                    double omega, cudaStream_t s);
// damped-Jacobi sweep from x + P e, e the correction of a space-coarsened next level (2D, one GPU)
bool launch_op_tc2d_pro(const OpDesc& op, const Geom& gc, bool trans, const double* x, const double* e,
                        const double* b, double* y, double omega, cudaStream_t s);
// tc3d.cu: (3+1)D TMA kernel for time-constant levels (fine from rho, stored MK), masked modes
bool launch_op_tc3d(const OpDesc& op, int mode, bool trans, bool mask, const double* x, const double* b, double* y,
                    double omega, cudaStream_t s);
// tc3r.cu: (3+1)D fine level of a time-constant design (element-layer products, full-row tiles)
bool launch_op_tc3r(const OpDesc& op, int mode, bool trans, bool mask, const double* x, const double* b, double* y,
                    double omega, cudaStream_t s);
// tv2d.cu: fine level of a space-time design with uniform capacity (configs 1, 3, 5), masked modes
bool launch_op_tv2d(const OpDesc& op, int mode, bool trans, bool mask, const double* x, const double* b, double* y,
                    double omega, cudaStream_t s);
void launch_rap_space(const OpDesc& fop, const Geom& gc, int nl, int ns, double* out, cudaStream_t s);
void launch_rap_time(const OpDesc& fop, int nlc, double* out, cudaStream_t s);
void launch_rho_to_mk(const OpDesc& fop, int tau, double* out, cudaStream_t s);
void launch_dense_assemble(const OpDesc& op, double* A, cudaStream_t s);
// max over rows of local planes [pa, pb] of sum_j |A_ij| / |A_ii| (bits of a positive double, atomicMax)
void launch_gersh(const OpDesc& op, int pa, int pb, unsigned long long* out, cudaStream_t s);

// transfer.cu — restriction r_c = m_f^c P^T r_f, prolongation x_f += m_f P e_c
void launch_restrict(const Geom& gf, const Geom& gc, int kind, const double* rf, double* rc, cudaStream_t s);
void launch_prolong_add(const Geom& gf, const Geom& gc, int kind, const double* ec, double* xf, cudaStream_t s);

// krylov.cu — deterministic reductions (fixed block count, last-block finalisation)
struct RedWs {
  double* partial;      // [kMaxBlocks * kMaxK]
  unsigned int* counter;
};
constexpr int kRedBlocks = 148 * 6;
constexpr int kMaxDots = 17;
constexpr int kMaxBasis = 256;  // longest basis of a multi-AXPY / linear combination (coarse GMRES(<= 255))
// out[0..k-1] = V_j . w (j < k), out[k] = w . w
void launch_mdot(const double* w, const double* V, long long ldv, int k, long long n, double* out, RedWs ws,
                 cudaStream_t s);
// w -= sum_j h[j] s2[j] V_j (h, s2 on device; s2 = null: 1); out[0] = ||w||^2 after
void launch_maxpy_norm(double* w, const double* V, long long ldv, int k, const double* h, const double* s2,
                       long long n, double* out, RedWs ws, cudaStream_t s);
// w -= sum_j s2_j h_j V_j, then out[0..k-1] = V^T w (new w), out[k] = ||w||^2; k <= 16 (false otherwise:
// nothing launched)
bool launch_maxpy_dots(double* w, const double* V, long long ldv, int k, const double* h, const double* s2,
                       long long n, double* out, RedWs ws, cudaStream_t s);
// x += sum_j y[j] Z_j (y on device)
void launch_lincomb(double* x, const double* Z, long long ldz, int k, const double* y, long long n, cudaStream_t s);
// v = w / sqrt(nrm2[0]) (nrm2 on device) or v = alpha * w
void launch_scale_dev(const double* w, double* v, const double* nrm2, long long n, cudaStream_t s);
void launch_scale(const double* w, double* v, double alpha, long long n, cudaStream_t s);
// two 64-bit hashes of the bit patterns of a[0..n) (order-free sums; exact design-change detection)
void launch_fingerprint(const double* a, long long n, unsigned long long* out, cudaStream_t s);
// GMRES(k) smoother bookkeeping on the device (single-thread kernels): st holds g[k+1], the Givens
// cs[k], sn[k], the Hessenberg H[k][k+1] and y[k] (at st + gm_y_offset(k)).
void launch_gm_init(double* st, int k, const double* nrm2, cudaStream_t s);           // g = (||r0||, 0, ...)
void launch_gm_col(double* st, int k, int j, const double* h, const double* nrm2w, cudaStream_t s);
void launch_gm_solve(double* st, int k, int mcols, cudaStream_t s);                  // y = R^-1 g (first mcols)
int gm_y_offset(int k);

// misc.cu
// Per-design conductivity table of a (2+1)D space-time design, read by tv2d: layers 0 .. nl-1 of
// k~(rho) = kins + dk rho^pk stored with a zero border, kt[t][gj+1][gi+1] (pitch n+2), plus a zero
// layer nl; (nl+1) (n+2)^2 doubles. rho: [nl][n][n].
void launch_ktilde(const double* rho, int n, int nl, const MatsDev& m, double* kt, cudaStream_t s);
void launch_source(const Geom& g, const st_source_t& src, double qscale, double tau, double* f, cudaStream_t s);
void launch_mask_free(const Geom& g, const double* in, double* out, cudaStream_t s);       // out = m_f .* in
void launch_copy_cons(const Geom& g, const double* src, double* dst, cudaStream_t s);     // dst_c = src_c
void launch_relayout(const Geom& gs, const double* src, const Geom& gd, double* dst, cudaStream_t s);
void launch_set_bc_values(const Geom& g, double T0, double* x, cudaStream_t s);          // x_c = xD
void launch_rhs_combine(const Geom& g, const double* f, const double* KxD, double T0, double* b, cudaStream_t s);
void launch_xd(const Geom& g, double T0, double* x, cudaStream_t s);
void launch_sensitivity(const OpDesc& op, const double* T, const double* lam, double* dJ, cudaStream_t s);
// dense coarsest level on its nf free nodes (fidx: free stored indices, fpos: stored index -> free
// position or -1): Ainv = (A[fidx][fidx])^-1 (A: the assembled N x N operator); x = A^-1 b on the free
// nodes, x = b elsewhere
void launch_dense_invert(const double* A, long long N, const int* fidx, int nf, double* Ainv, int* info,
                         cudaStream_t s);
void launch_dense_solve(const double* Ainv, int nf, const int* fidx, const int* fpos, long long N, bool trans,
                        const double* b, double* x, cudaStream_t s);

// design.cu — config-5 design update (density filter, OC)
void launch_filter(int sd, int n, int nl, int tdir, int lo_ok, int hi_ok, double r, const double* ghosted, double* out,
                   int mode, cudaStream_t s);
void launch_filter_w(int sd, int n, int nl, int tdir, int lo_ok, int hi_ok, double r, double* out, cudaStream_t s);
void launch_filter_pack(long long count, const double* src, const double* W, double* dst, cudaStream_t s);
void launch_oc_sum(const double* rho, const double* dj, long long n, double lam, double move, double lo,
                   double* partial, unsigned* counter, double* out, cudaStream_t s);
void launch_pnorm_sum(const Geom& g, int nl, const double* T, double P, double* partial, unsigned* counter, double* out,
                      cudaStream_t s);
void launch_pnorm_grad(const Geom& g, int p0, int np, int ntg, const double* T, double P, double scale, double* out,
                       cudaStream_t s);
void launch_oc_apply(const double* rho, const double* dj, long long n, double lam, double move, double lo, double* out,
                     cudaStream_t s);

}  // namespace st
