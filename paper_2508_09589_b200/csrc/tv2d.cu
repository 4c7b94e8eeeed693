// tv2d.cu — (2+1)D fine-level operator for a space-time (time-varying) design with uniform
// capacity, sm_100a, fp64 (BASELINE configs 1, 3, 5: C = 1, k = k(rho) per element and layer).
//
// Same operator and modes as op_kernel (ops.cu; plane form in DESIGN.md sec. 7) with the upwind
// capacity factor and a symmetric conduction factor (as tc2d.cu). With uniform capacity the mass
// is the same separable stencil on every layer; the stiffness of layer tau, K^(tau), comes from
// the element conductivities of that layer. Per plane q the kernel forms
//   M x_q (separable),  Kb_q = K^(q-1) x_q  (layer below),  Ka_q = K^(q) x_q  (layer above)
// and completes row q-1 = carry + t00 Ka_{q-1} + t01 Kb_q (K^T: - M x_q), carry for row q =
// M (x_q - x_{q-1}) + t01 Ka_{q-1} + t11 Kb_q (K^T: M x_q).
// Design: persistent one-wave grid over (tile, plane) work as tc2d; per plane
// ONE mbarrier-tracked TMA group brings the x tile, the b tile and the layer tile into a ring
// slot (SRC 0: the 34 x 9 box of the per-design k~ table of layer q, op.kt, filled once per
// design by launch_ktilde; SRC 1: the 5 x 36 x 9 forward stiffness coefficients of layer q), so a
// plane costs one barrier wait and one __syncthreads (slot release). Layer boxes start at
// (max(x0-2, 0), max(y0-1, 0)): a tile-mode fp64 TMA box must start at a non-negative, 16-byte
// aligned coordinate (else an illegal instruction: scripts/dev/tma_neg.cu, scripts/dev/tv_probe.sh);
// entries beyond the last node / element are zero-filled, entries left of / below the domain are
// read from the (zero-initialised) ring and masked. SRC 0 keeps the 6 element conductivities of
// the layer below in registers and applies K through the 4 element "brackets" of x at the node
// (shared by the layer-below and layer-above products); SRC 1 re-reads the layer below from the
// previous ring slot, which is only refilled after the plane is done. The first plane of a
// segment is peeled (no layer below it), so the steady-state body has no such selects.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace st {
namespace tv {

constexpr int TX = 32, TYT = 4, RY = 2, TY = TYT * RY;   // node tile 32 x 8
constexpr int HX = TX + 4, HY = TY + 2;                  // x tile 36 x 10 (col 0 unused)
constexpr int XS = 368, BS = 256;                        // slot sizes (doubles, multiples of 128 B)
constexpr int EY = TY + 1;                               // layer box rows y0-1 .. y0+7
constexpr int EX0 = TX + 2, EX1 = TX + 4;                // box columns from x0-2: elements x0-1 .. x0+31 /
                                                         // nodes x0-1 .. x0+32 (even widths: 16-B rows)
constexpr int ET0 = EX0 * EY, ET1 = EX1 * EY;
constexpr int RS0 = 320, RS1 = 1664;                     // layer slot: rho box / 5 coefficient boxes
constexpr int NB0 = 6, NB1 = 4;                          // ring depth (planes)
constexpr int NTH = TX * TYT;
constexpr unsigned XBYTES = HX * HY * 8, BBYTES = TX * TY * 8;

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @P1 bra DONE_%=;\n"
      " bra WAIT_%=;\n"
      "DONE_%=:\n}\n" ::"r"(su32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(
          su32(dst)),
      "l"((uint64_t)map), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma4(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];\n" ::"r"(
          su32(dst)),
      "l"((uint64_t)map), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

__device__ __forceinline__ double ap9(const double (&w)[9], const double (&nb)[RY + 2][3], int r) {
  double a = w[4] * nb[r + 1][1];
  double b = w[0] * nb[r][0];
  a = fma(w[1], nb[r][1], a);
  b = fma(w[2], nb[r][2], b);
  a = fma(w[3], nb[r + 1][0], a);
  b = fma(w[5], nb[r + 1][2], b);
  a = fma(w[6], nb[r + 2][0], a);
  b = fma(w[7], nb[r + 2][1], b);
  a = fma(w[8], nb[r + 2][2], a);
  return a + b;
}

// 1/d for the per-plane Jacobi diagonal: approximate reciprocal (MUFU.RCP64H) + two Newton steps
// (full double accuracy for the positive, normal diagonals; no branch, no double division)
__device__ __forceinline__ double rcp_d(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  r = r * fma(-d, r, 2.0);
  return r * fma(-d, r, 2.0);
}

// the 9 stiffness weights (x 6) of a node from the forward coefficients of a layer box: its own
// (centre, +1 0, -1 +1, 0 +1, +1 +1) and the mirrored ones of the (i-1, j-1), (i, j-1), (i+1, j-1),
// (i-1, j) neighbours (the operator is symmetric in space)
// (mi: i >= 1, mj: j >= 1; neighbours beyond the last node are zero-filled by the TMA)
__device__ __forceinline__ void wk_box(const double* ct, int L, bool mi, bool mj, double (&w)[9]) {
  constexpr int EX = EX1, ET = ET1;
  w[4] = ct[0 * ET + L];
  w[5] = ct[1 * ET + L];
  w[6] = ct[2 * ET + L];
  w[7] = ct[3 * ET + L];
  w[8] = ct[4 * ET + L];
  w[0] = (mi && mj) ? ct[4 * ET + L - EX - 1] : 0.0;
  w[1] = mj ? ct[3 * ET + L - EX] : 0.0;
  w[2] = mj ? ct[2 * ET + L - EX + 1] : 0.0;
  w[3] = mi ? ct[1 * ET + L - 1] : 0.0;
}

// one (tile, plane-range) segment of a CTA's work list and the planes it loads
struct Seg {
  int p0, p1, qs, qe;  // rows p0 .. p1-1; planes qs .. qe (qs = p0 - 1 reloads the plane below)
  int x0, y0, bx, by;  // node tile origin, layer box origin
};
__device__ __forceinline__ bool next_seg(Sched& s, int ntx, int nt, Seg& sg) {
  long long tile;
  if (!sched_next(s, tile, sg.p0, sg.p1)) return false;
  sg.qs = max(sg.p0 - 1, 0);
  sg.qe = min(sg.p1, nt);
  sg.x0 = (int)(tile % ntx) * TX;
  sg.y0 = (int)(tile / ntx) * TY;
  sg.bx = max(sg.x0 - 2, 0);  // stored-stencil box origin (x0 is a multiple of 32)
  sg.by = max(sg.y0 - 1, 0);
  return true;
}

// SRC: 0 = fine level from rho (the per-design k~ table op.kt, one entry per element and layer); 1 = stored per-layer
// stiffness of a time-varying Galerkin space level (uniform capacity: the separable mass op.msc)
template <int SRC, int MODE, bool TRANS>
__global__ void __launch_bounds__(NTH, SRC == 0 ? 4 : 3)
    tv2d_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmb,
                const __grid_constant__ CUtensorMap tml, OpDesc op, const double* __restrict__ x,
                double* __restrict__ y, double omega, long long wtot, int kchunk, int ntx) {
  constexpr bool NX = (MODE != MODE_JAC0);
  constexpr bool NBV = (MODE != MODE_APPLY);
  constexpr bool ND = (MODE == MODE_JAC || MODE == MODE_JAC0);
  constexpr int NB = SRC == 0 ? NB0 : NB1;
  constexpr int RS = SRC == 0 ? RS0 : RS1;
  constexpr int EX = SRC == 0 ? EX0 : EX1;
  constexpr unsigned LBYTES = (SRC == 0 ? ET0 : 5 * ET1) * 8;
  extern __shared__ __align__(128) double smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  double* xs = smem + 16;                    // [NB][XS]
  double* bs = xs + (NX ? NB * XS : 0);      // [NB][BS]
  double* ls = bs + (NBV ? NB * BS : 0);     // [NB][RS] layer boxes (layer q arrives with plane q)

  const Geom& g = op.g;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
  const int n = g.n, pr = g.pr;
  const long long P = g.P;
  const long long NP = g.nt + 1;
  const int xo = (ty * RY) * HX + tx + 1;
  const int bo = (ty * RY) * TX + tx;

  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < NB; ++k) mbar_init(&bar[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  const double sm = SRC == 0 ? g.dx * g.dx * (1.0 / 36.0) * op.m.Cins : op.msc;
  const double sk = SRC == 0 ? 1.0 / 6.0 : 1.0;
  const double t00 = op.Tm[0][0] * sk, t01 = op.Tm[0][1] * sk, t11 = op.Tm[1][1] * sk;
  const unsigned tx_plane = (NX ? XBYTES : 0u) + (NBV ? BBYTES : 0u);

  // zero the ring once: box entries a thread reads outside the domain (clamped origin, masked
  // by 0) are then finite; the generic-proxy stores are ordered before the first TMA write
  for (int k = tid; k < NB * ((NX ? XS : 0) + (NBV ? BS : 0) + RS); k += NTH) xs[k] = 0.0;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();  // barriers initialised, ring zeroed
  pdl_wait();       // the previous kernel's writes are visible from here on

  const long long tiles = wtot / NP;
  // producer (thread 0): walks this CTA's (segment, plane) sequence NB-1 planes ahead of the
  // consumer, across segment boundaries; a slot is refilled only after the __syncthreads that
  // ends the plane consuming it
  Sched psc;
  sched_init(psc, tiles, (int)NP, kchunk);
  Seg ps;
  bool pv = next_seg(psc, ntx, g.nt, ps);
  int pq = ps.qs;
  auto issue_next = [&](unsigned slot) {
    if (!pv) return;
    const int q = pq;
    const bool wb = NBV && q >= ps.p0 && q < ps.p1;
    const bool hl = SRC == 0 || q < g.nt;  // layer q (SRC 0: layer nt of the padded k~ table is zero)
    mbar_expect_tx(&bar[slot], tx_plane - ((NBV && !wb) ? BBYTES : 0u) + (hl ? LBYTES : 0u));
    if (NX) tma3(xs + slot * XS, &tmx, &bar[slot], ps.x0, ps.y0, q);
    if (wb) tma3(bs + slot * BS, &tmb, &bar[slot], ps.x0, ps.y0, q);
    if (hl) {
      if (SRC == 0) tma3(ls + slot * RS, &tml, &bar[slot], ps.x0, ps.y0, q);  // padded: element x0-1 at x0
      else tma4(ls + slot * RS, &tml, &bar[slot], ps.bx, ps.by, 0, 2 * q + 1);
    }
    if (++pq > ps.qe) {
      pv = next_seg(psc, ntx, g.nt, ps);
      pq = ps.qs;
    }
  };
  if (tid == 0)
    for (int k = 0; k < NB - 1; ++k) issue_next((unsigned)k);

  Sched csc;
  sched_init(csc, tiles, (int)NP, kchunk);
  Seg cs;
  unsigned cur = 0u, prv = NB - 1, phase = 0u;
  while (next_seg(csc, ntx, g.nt, cs)) {
    const int p0 = cs.p0, p1 = cs.p1, qs = cs.qs, qe = cs.qe;
    const int x0 = cs.x0, y0 = cs.y0, bx = cs.bx, by = cs.by;
    const int i = x0 + tx, j0 = y0 + ty * RY;
    bool act[RY], patch[RY];
    double cy[RY], smc[RY];
    const double cx = (i == 0 || i == n) ? 2.0 : 4.0;
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      const int j = j0 + r;
      act[r] = (i <= n) && (j <= n);
      patch[r] = i == 0 && j >= g.plo && j <= g.phi;
      cy[r] = (j == 0 || j == n) ? 2.0 : 4.0;
      smc[r] = sm * cx * cy[r];  // capacity part of the Jacobi diagonal (separable mass centre)
    }
    // box entry of element (i-1, j0-1) (SRC 0: padded table, box from (x0, y0) = element
    // (x0-1, y0-1); outside the domain the border / the TMA fill is zero) / of node (i, j0) (SRC 1:
    // entries left of / below the domain are read from the ring (finite) and masked)
    const int lo = SRC == 0 ? (ty * RY) * EX + tx : (j0 - by) * EX + (i - bx);

    double kc[RY + 1][2];  // SRC 0: element conductivities of layer q-1 (below plane q)
    double dCc[RY];        // centre stiffness weight of layer q-1
    double Mprev[RY], Kaprev[RY], carry[RY], dcarry[RY];
    double* yrow = y + (long long)(qs - 1) * P + (long long)j0 * pr + i;

    // one plane q; FIRST: the segment's first plane (no layer below it in this segment)
    auto plane = [&](int q, auto first_tag) -> bool {
      constexpr bool FIRST = decltype(first_tag)::value;
      mbar_wait(&bar[cur], (phase >> cur) & 1u);
      phase ^= 1u << cur;
      const bool has = q < g.nt;
      const double* xq = xs + cur * XS + xo;
      double kn[RY + 1][2];
      double dCn[RY];
      if (SRC == 0) {  // k~ of layer q (zero outside the domain and beyond the last layer)
        const double* rd = ls + cur * RS + lo;
#pragma unroll
        for (int s2 = 0; s2 <= RY; ++s2)
#pragma unroll
          for (int d = 0; d < 2; ++d) kn[s2][d] = rd[s2 * EX + d];
        double rs2[RY + 1];
#pragma unroll
        for (int s2 = 0; s2 <= RY; ++s2) rs2[s2] = kn[s2][0] + kn[s2][1];
#pragma unroll
        for (int r = 0; r < RY; ++r) dCn[r] = 4.0 * (rs2[r] + rs2[r + 1]);
      }
      double Mq[RY], Kb[RY], Ka[RY];
      if (NX && q + g.pg0 > 0) {
        double nb[RY + 2][3];
#pragma unroll
        for (int s2 = 0; s2 < RY + 2; ++s2)
#pragma unroll
          for (int c = 0; c < 3; ++c) nb[s2][c] = xq[s2 * HX + c];
        double rsum[RY + 2];
#pragma unroll
        for (int s2 = 0; s2 < RY + 2; ++s2) rsum[s2] = fma(cx, nb[s2][1], nb[s2][0] + nb[s2][2]);
        if (j0 == 0) rsum[0] = 0.0;  // row j = -1 aliases the previous plane's last row
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          Mq[r] = fma(cy[r], rsum[r + 1], rsum[r] + rsum[r + 2]);
          if (SRC == 0) {
            // element brackets: sum_e k_e (K_e x)_node with K_e the unit Q1 stiffness (x 6)
            const double c4 = 4.0 * nb[r + 1][1];
            const double bsw = c4 - fma(2.0, nb[r][0], nb[r][1] + nb[r + 1][0]);
            const double bse = c4 - fma(2.0, nb[r][2], nb[r][1] + nb[r + 1][2]);
            const double bnw = c4 - fma(2.0, nb[r + 2][0], nb[r + 2][1] + nb[r + 1][0]);
            const double bne = c4 - fma(2.0, nb[r + 2][2], nb[r + 2][1] + nb[r + 1][2]);
            Ka[r] = fma(kn[r][0], bsw, fma(kn[r][1], bse, fma(kn[r + 1][0], bnw, kn[r + 1][1] * bne)));
            Kb[r] = FIRST ? 0.0 : fma(kc[r][0], bsw, fma(kc[r][1], bse, fma(kc[r + 1][0], bnw, kc[r + 1][1] * bne)));
          } else {
            const int L = lo + r * EX;  // node (i, j0 + r) in the box
            double wv[9];
            if (!FIRST) {
              wk_box(ls + prv * RS, L, i >= 1, j0 + r >= 1, wv);
              Kb[r] = ap9(wv, nb, r);
            } else {
              Kb[r] = 0.0;
            }
            if (has) {
              wk_box(ls + cur * RS, L, i >= 1, j0 + r >= 1, wv);
              Ka[r] = ap9(wv, nb, r);
            } else {
              Ka[r] = 0.0;
            }
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < RY; ++r) Mq[r] = Kb[r] = Ka[r] = 0.0;
      }
      if (SRC == 1) {
#pragma unroll
        for (int r = 0; r < RY; ++r) dCn[r] = has ? ls[cur * RS + lo + r * EX] : 0.0;
      }
      if (!FIRST && q - 1 >= p0) {  // row q-1 complete (bottom part of layer q-1)
        const double* bp = bs + prv * BS + bo;
        if (q - 1 + g.pg0 == 0) {
#pragma unroll
          for (int r = 0; r < RY; ++r) {
            if (!act[r]) continue;
            const double xc = NX ? __ldg(x + (yrow - y) + r * pr) : 0.0;
            const double bv = NBV ? bp[r * TX] : 0.0;
            double o;
            if (MODE == MODE_APPLY) o = xc;
            else if (MODE == MODE_RESID) o = bv - xc;
            else if (MODE == MODE_JAC) o = fma(omega, bv - xc, xc);
            else o = omega * bv;
            yrow[r * pr] = o;
          }
        } else {
          const double* xp = xs + prv * XS + xo;
#pragma unroll
          for (int r = 0; r < RY; ++r) {
            const double bot = fma(t00, Kaprev[r], t01 * Kb[r]);
            const double Ax = TRANS ? fma(-sm, Mq[r], carry[r] + bot) : carry[r] + bot;
            const double od = ND ? omega * rcp_d(fma(t00, dCc[r], dcarry[r])) : 0.0;
            double o;
            if (MODE == MODE_APPLY) o = Ax;
            else if (MODE == MODE_RESID) o = bp[r * TX] - Ax;
            else if (MODE == MODE_JAC) o = fma(od, bp[r * TX] - Ax, xp[(r + 1) * HX + 1]);
            else o = od * bp[r * TX];
            if (act[r]) yrow[r * pr] = patch[r] ? 0.0 : o;
          }
        }
      }
#pragma unroll
      for (int r = 0; r < RY; ++r) {  // top part of layer q-1 -> row q; diagonal carried likewise
        if (FIRST) {
          carry[r] = dcarry[r] = 0.0;
        } else {
          const double cap = TRANS ? Mq[r] : Mq[r] - Mprev[r];
          carry[r] = fma(sm, cap, fma(t01, Kaprev[r], t11 * Kb[r]));
          dcarry[r] = fma(t11, dCc[r], smc[r]);
        }
        Mprev[r] = Mq[r];
        Kaprev[r] = Ka[r];
        dCc[r] = dCn[r];
      }
      if (SRC == 0) {
#pragma unroll
        for (int s2 = 0; s2 <= RY; ++s2) { kc[s2][0] = kn[s2][0]; kc[s2][1] = kn[s2][1]; }
      }
      __syncthreads();  // slot of plane q-1 consumed by every thread
      if (tid == 0) issue_next(prv);
      yrow += P;
      prv = cur;
      if (++cur == NB) cur = 0u;
      return q < qe;  // plane qe's slot (now prv) stays until the next plane's barrier: tail row
    };
    if (plane(qs, std::true_type{}))
      for (int q = qs + 1; plane(q, std::false_type{}); ++q) {
      }
    if (p1 == g.nt + 1) {  // last row: top part of layer nt-1 only
      const double* bq = bs + prv * BS + bo;
      const double* xq = xs + prv * XS + xo;
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        const double od = ND ? omega / dcarry[r] : 0.0;
        const double Ax = carry[r];
        double o;
        if (MODE == MODE_APPLY) o = Ax;
        else if (MODE == MODE_RESID) o = bq[r * TX] - Ax;
        else if (MODE == MODE_JAC) o = fma(od, bq[r * TX] - Ax, xq[(r + 1) * HX + 1]);
        else o = od * bq[r * TX];
        if (act[r]) yrow[r * pr] = patch[r] ? 0.0 : o;
      }
    }
  }
}

}  // namespace tv

// ---------------------------------------------------------------------------------------
namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn_tv() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    else
      cudaGetLastError();
  }
  return fn;
}

bool map3_tv(CUtensorMap* m, const void* base, unsigned long long d0, unsigned long long d1, unsigned long long d2,
             unsigned long long s1, unsigned long long s2, unsigned b0, unsigned b1) {
  auto fn = encode_fn_tv();
  if (!fn || ((uintptr_t)base & 15u) || (s1 & 15u) || (s2 & 15u)) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1, s2};
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 4D map of the stored per-layer stencils [layer][M|K][5][node]: dims (nn, nn, 5, 2 nl), box 34 x 9 x 5 x 1
bool map4_tv(CUtensorMap* m, const void* base, unsigned long long nn, unsigned long long nl2, unsigned long long s1,
             unsigned long long s2, unsigned long long s3) {
  auto fn = encode_fn_tv();
  if (!fn || ((uintptr_t)base & 15u) || (s1 & 15u) || (s2 & 15u) || (s3 & 15u)) return false;
  cuuint64_t dims[4] = {nn, nn, 5, nl2};
  cuuint64_t strides[3] = {s1, s2, s3};
  cuuint32_t box[4] = {(cuuint32_t)tv::EX1, (cuuint32_t)tv::EY, 5, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int SRC, int MODE, bool TRANS>
void ltv(const CUtensorMap& mx, const CUtensorMap& mb, const CUtensorMap& ml, const OpDesc& op, const double* x,
         double* y, double omega, cudaStream_t s) {
  using namespace tv;
  const Geom& g = op.g;
  auto kern = tv2d_kernel<SRC, MODE, TRANS>;
  constexpr bool NX = (MODE != MODE_JAC0), NBV = (MODE != MODE_APPLY);
  constexpr int RS = SRC == 0 ? RS0 : RS1, NB = SRC == 0 ? NB0 : NB1;
  constexpr size_t bytes = sizeof(double) * (16 + NB * ((NX ? XS : 0) + (NBV ? BS : 0) + RS));
  static int resident = 0, nsm = 0;
  if (!resident) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, kern, NTH, bytes);
    if (resident < 1) resident = 1;
  }
  const long long ntx = (g.nn + TX - 1) / TX, nty = (g.nn + TY - 1) / TY;
  const long long wtot = ntx * nty * (g.nt + 1);
  long long grid = persistent_grid(op, nsm, resident, wtot);
  const long long tiles = ntx * nty;
  const int NPl = g.nt + 1;
  int kauto;
  if (tiles >= grid) {
    // at least one tile per CTA: the strided schedule over whole tile columns, one chunk. Measured at
    // 1024^2 x 1024 (profiles/r02/kbench_c3_chunk.log): fine JAC sweep 10.7 ms (round-1 sliced
    // 16-plane chunks) -> 6.8 ms, DRAM reads 46.2 -> 30.4 GB (the x / b / k~ reads are 25.8 GB);
    // K = 16 / 32 / 64 / 128: 9.0 / 8.7 / 8.1 / 7.4 ms. A large partial last group (its tile columns
    // split into plane ranges over all CTAs) loses the reuse: then the grid is trimmed so that the
    // tiles form equal full groups — 512^2 (1089 tiles: 1 group of 592 + 497) 1105 -> 946 us with 2
    // groups of 545, while 1024^2 (4257 tiles: 7 x 592 + 113) keeps its wave (8 x 533: 6.81 -> 7.59
    // ms; profiles/r02/kbench_trim.log). max_ctas < 0 forces the trim.
    const long long part = tiles % grid;
    if (op.max_ctas < 0 || (op.max_ctas == 0 && part * 5 >= grid * 2)) {
      const long long groups = (tiles + grid - 1) / grid;
      grid = (tiles + groups - 1) / groups;
    }
    kauto = NPl;
  } else {
    // fewer tiles than CTAs: CTAs share a tile's planes (contiguous ranges of the partial group);
    // with long runs (>= 256 planes per CTA) chunks keep neighbouring tiles at nearby planes: 512^2 x
    // 512 fine sweep 1114 (one chunk) -> 942 us (K = 64), its stored-stencil level 1 694 -> 576 us
    // (K = 32); short runs keep one chunk
    kauto = wtot / grid >= 256 ? (SRC == 0 ? 64 : 32) : NPl;
  }
  // st_options_t chunk_planes overrides (parity tests force chunked schedules on small grids)
  const int kch = chunk_planes(op, NPl, kauto);
  launch_pdl(kern, dim3((unsigned)grid), dim3(TX, TYT, 1), bytes, s, mx, mb, ml, op, x, y, omega, wtot, kch, (int)ntx);
}
}  // namespace

// Masked modes of the fine level of a space-time design with uniform capacity; false if not covered.
bool launch_op_tv2d(const OpDesc& op, int mode, bool trans, bool mask, const double* x, const double* b, double* y,
                    double omega, cudaStream_t s) {
  if (op.g.walls) return false;  // Example 2's cold walls: the generic kernels (is_cons)
  const Geom& g = op.g;
  const bool rho_tv = op.form == FORM_RHO && !op.rho_tc && op.m.dC == 0.0;
  const bool mk_tv = op.form == FORM_MK && op.tvl && op.msep;
  if (g.sd != 2 || !mask || !(rho_tv || mk_tv)) return false;
  if (op.U[0][0] != 0.0 || op.U[0][1] != 0.0 || op.U[1][0] != -1.0 || op.U[1][1] != 1.0) return false;
  if (op.Tm[0][1] != op.Tm[1][0]) return false;
  CUtensorMap mx{}, mb{};
  const unsigned long long nn = g.nn, s1 = (unsigned long long)g.pr * 8, s2 = (unsigned long long)g.P * 8;
  const bool nx = (mode != MODE_JAC0), nbv = (mode != MODE_APPLY);
  if (nx && !map3_tv(&mx, x - (g.pr + 2), (unsigned long long)g.pr + 2, nn + 1, g.nt + 1, s1, s2, tv::HX, tv::HY))
    return false;
  if (nbv && !map3_tv(&mb, b, nn, nn, g.nt + 1, s1, s2, tv::TX, tv::TY)) return false;
  CUtensorMap ml{};  // layer boxes from (x0-1, y0-1); entries outside the domain are zero-filled
  if (g.nt < 1) return false;
  if (rho_tv) {
    const unsigned long long ne = (unsigned long long)g.n;
    const unsigned long long w2 = ne + 2;  // padded table [nt+1][n+2][n+2] (launch_ktilde)
    if (!op.kt || !map3_tv(&ml, op.kt, w2, w2, g.nt + 1, w2 * 8, w2 * w2 * 8, tv::EX0, tv::EY)) return false;
  } else if (!map4_tv(&ml, op.st, nn, 2ull * g.nt, s1, s2, 5ull * s2)) {
    return false;
  }
#define C4(M)                                                                            \
  case M:                                                                                \
    if (rho_tv) { if (trans) ltv<0, M, true>(mx, mb, ml, op, x, y, omega, s);           \
                  else ltv<0, M, false>(mx, mb, ml, op, x, y, omega, s); }              \
    else { if (trans) ltv<1, M, true>(mx, mb, ml, op, x, y, omega, s);                  \
           else ltv<1, M, false>(mx, mb, ml, op, x, y, omega, s); }                     \
    break;
  switch (mode) {
    C4(MODE_APPLY)
    C4(MODE_RESID)
    C4(MODE_JAC)
    C4(MODE_JAC0)
  }
#undef C4
  return true;
}

}  // namespace st
