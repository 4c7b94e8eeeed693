// common.cuh — internal types and device helpers of libst (B200, sm_100a, fp64).
//
// Operator algebra (derivation in DESIGN.md "Plane form"): the element matrix of the
// stabilised CG space-time element factorises as
//     A_e = C_e (U (x) M_sp) + k~_e (Tm (x) K_sp),  U = [[0,0],[-1,1]], Tm = dt/6 [[2,1],[1,2]]
// (time index: row = test, col = trial; bottom = 0, top = 1). Every multigrid level of the
// Galerkin hierarchy is stored per element LAYER tau (planes tau, tau+1)
// as a 2x2 time block of symmetric spatial stencils S^{ab}_tau:
//     (K x)_p = S^{tb}_{p-1} x_{p-1} + S^{tt}_{p-1} x_p + S^{bb}_p x_p + S^{bt}_p x_{p+1}.
// Forms: RHO (fine level, matrix-free: M, K stencils from rho on the fly), MK (S^{ab} =
// U[a][b] M_tau + Tm[a][b] K_tau, stored M, K), B4 (S^{ab} = U[a][b] M_tau + K^{ab}_tau: five
// stored stencils per layer, time-varying levels below a time coarsening).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace st {

enum Form { FORM_RHO = 0, FORM_MK = 1, FORM_B4 = 2, FORM_DENSE = 3 };
enum Kind { KIND_FINE = 0, KIND_SPACE = 1, KIND_TIME = 2, KIND_FULL = 3 };
enum Mode { MODE_APPLY = 0, MODE_RESID = 1, MODE_JAC = 2, MODE_JAC0 = 3 };

// Level geometry: n^sd x nt elements, (n+1)^sd (nt+1) nodes. Storage: x1 rows of pitch pr
// (pr = nn for the caller's dense layout; internal vectors use an even pitch so that every
// row and plane starts 16-byte aligned — TMA tiles); pad entries are kept at zero.
struct Geom {
  int sd;
  int n, nn, nt;
  int pr;        // row pitch (elements) of the x1 rows
  long long P;   // stored entries per time plane (pr * nn^(sd-1))
  long long N;   // stored entries (P * (nt+1))
  int plo, phi;  // sink patch: transverse node range at x1 = 0 (plo > phi: none)
  double dx, dt;
  int pg0;       // global index of local plane 0 (time slabs); 0 on one GPU
  int walls;     // 1: every spatial boundary node is constrained (T = 0, Example 2's cold walls)
};

struct MatsDev {
  double Cins, dC, pc;   // C = Cins + dC rho^pc
  double kins, dk, pk;   // k~ = kins + dk rho^pk   (already rescaled by tau/L^2)
};

// Operator descriptor, passed by value to kernels.
struct OpDesc {
  Geom g;
  int form;
  int nl;                 // stored layers: 1 (time-constant) or the (local) layer count
  int tvl;                // per-layer (time-varying) storage; a slab may hold a single layer
  double U[2][2], Tm[2][2];
  const double* rho;      // FORM_RHO
  const double* kt;       // FORM_RHO, space-time (2+1)D design: k~ per element (set with rho), or null
  int rho_tc;             // rho time-constant
  MatsDev m;
  const double* st;       // MK: [nl][2][NC][P]; B4: [nl][5][NC][P] = M, Kbb, Kbt, Ktb, Ktt
  int msep;               // MK: the stored M equals msc x (Q1 mass pattern of this grid), i.e. the
  double msc;             //     separable [1,4,1] (x) [1,4,1] stencil (uniform capacity; nested spaces)
  // kernel selection and persistent-schedule controls (st_options_t: kernel_family, chunk_planes,
  // max_ctas), read per launch
  int family;             // ST_KERNELS_* (st.h)
  int chunk;              // planes per time chunk: 0 automatic, > 0 forced, < 0 no chunking
  int max_ctas;           // cap on the persistent grid (0: one full wave)
};

template <int SD> struct SG {
  static constexpr int NOFF = SD == 2 ? 9 : 27;
  static constexpr int CEN = SD == 2 ? 4 : 13;
  static constexpr int NC = SD == 2 ? 5 : 14;     // center + forward offsets
  static constexpr int NE = SD == 2 ? 4 : 8;      // elements around a node
  // offset component d (0 = x1) of stencil index k = (dz+1)*9 + (dy+1)*3 + (dx+1)
  __host__ __device__ static constexpr int od(int k, int d) {
    return d == 0 ? (k % 3) - 1 : (d == 1 ? ((k / 3) % 3) - 1 : (k / 9) - 1);
  }
};

// spatial element-matrix entries by Hamming distance h between local corners
// 2D: M = dx^2/36 [4,2,1], K = 1/6 [4,-1,-2];  3D: M = dx^3/216 [8,4,2,1], K = dx [1/3,0,-1/12,-1/12]
template <int SD> __device__ __forceinline__ double mtab(int h, double dx) {
  if (SD == 2) return (h == 0 ? 4.0 : (h == 1 ? 2.0 : 1.0)) * (dx * dx / 36.0);
  return (h == 0 ? 8.0 : (h == 1 ? 4.0 : (h == 2 ? 2.0 : 1.0))) * (dx * dx * dx / 216.0);
}
template <int SD> __device__ __forceinline__ double ktab(int h, double dx) {
  if (SD == 2) return (h == 0 ? 4.0 : (h == 1 ? -1.0 : -2.0)) * (1.0 / 6.0);
  return (h == 0 ? (1.0 / 3.0) : (h == 1 ? 0.0 : (-1.0 / 12.0))) * dx;
}

__device__ __forceinline__ double powp(double r, double p) {
  if (p == 3.0) return r * r * r;
  if (p == 1.0) return r;
  if (p == 2.0) return r * r;
  if (p == 4.0) { double q = r * r; return q * q; }
  if (p == 0.0) return 1.0;
  return pow(r, p);
}
__device__ __forceinline__ double dpowp(double r, double p) {  // d/dr r^p
  if (p == 3.0) return 3.0 * r * r;
  if (p == 1.0) return 1.0;
  if (p == 2.0) return 2.0 * r;
  if (p == 4.0) return 4.0 * r * r * r;
  if (p == 0.0) return 0.0;
  return p * pow(r, p - 1.0);
}

// constrained node test (R-2, R-4): t = 0 plane, or sink patch at x1 = 0
// spatial Dirichlet node (value 0 at all t): the sink patch, or with g.walls every boundary node
template <int SD> __device__ __forceinline__ bool is_patch(const Geom& g, const int* c) {
  if (g.walls) {
    bool w = c[0] == 0 || c[0] == g.n || c[1] == 0 || c[1] == g.n;
    if (SD == 3) w = w || c[2] == 0 || c[2] == g.n;
    return w;
  }
  if (c[0] != 0) return false;
  bool in = (c[1] >= g.plo && c[1] <= g.phi);
  if (SD == 3) in = in && (c[2] >= g.plo && c[2] <= g.phi);
  return in;
}
template <int SD> __device__ __forceinline__ bool is_cons(const Geom& g, const int* c, int p) {
  if (p + g.pg0 == 0) return true;  // initial-condition plane (global t = 0)
  return is_patch<SD>(g, c);
}

template <int SD> __device__ __forceinline__ long long pidx(const Geom& g, const int* c) {
  long long r = c[0] + (long long)g.pr * c[1];
  if (SD == 3) r += (long long)g.pr * g.nn * c[2];
  return r;
}

// decode an in-plane storage offset into node coordinates; false for pad entries
template <int SD> __device__ __forceinline__ bool pdecode(const Geom& g, long long pn, int* c) {
  c[0] = (int)(pn % g.pr);
  long long t = pn / g.pr;
  c[1] = (int)(t % g.nn);
  c[2] = (SD == 3) ? (int)(t / g.nn) : 0;
  return c[0] < g.nn;
}

// Work list of the persistent stencil kernels: (tile, time plane) items ordered by time chunks
// (chunk-major, then tile, then plane); CTA c owns a contiguous range of the list, so with chunks
// a CTA sweeps a run of tiles over the same few planes and the halo it shares with the previous
// tile of its run is still in L2. The nch = ceil(NP / K) chunks are balanced
// (sizes differ by at most one plane: a 1-plane tail chunk would give one CTA a run of 1-plane
// segments that bounds the whole launch). Decodes item w into a segment (tile, planes [p0, p1))
// that stays inside one chunk and one tile and ends at or before wend.
__device__ __forceinline__ void work_segment(long long w, long long wend, long long tiles, int NP, int K,
                                             long long* tile, int* p0, int* p1) {
  const int nch = (NP + K - 1) / K;
  const int pp = (int)(w / tiles);  // chunk c covers items [tiles * cs(c), tiles * cs(c+1))
  int c = (int)(((long long)pp * nch) / NP);
  while (c + 1 < nch && (int)((long long)(c + 1) * NP / nch) <= pp) ++c;
  while (c > 0 && (int)((long long)c * NP / nch) > pp) --c;
  const int cs = (int)((long long)c * NP / nch), ce = (int)((long long)(c + 1) * NP / nch);
  const int Kc = ce - cs;
  const long long r = w - tiles * cs;
  *tile = r / Kc;
  *p0 = cs + (int)(r % Kc);
  const long long rem = wend - w;
  *p1 = (rem < ce - *p0) ? *p0 + (int)rem : ce;
}

// Strided chunk schedule of the persistent stencil kernels tv2d / tc3r: the NP
// planes are cut into nch balanced chunks of ~K planes; inside a chunk the tiles form groups of
// G = gridDim.x consecutive tiles, and CTA b takes tile kG + b of every full group k for all the
// chunk's planes (one segment per group), then an equal share of the (tile, plane) items of the last,
// partial group (contiguous, tile-major). At any moment CTA b and its tile neighbours' CTAs work on
// neighbouring tiles at about the same plane: the halo rows / columns two tiles share are requested
// twice within a short interval and the second request hits L2 (the round-1 slice-per-CTA schedule put
// a CTA's neighbour tiles 16 planes apart in time on the same CTA: ~10 % L2 hit rate at 1024^2 x 1024,
// 1.8x the algorithmic DRAM reads, profiles/r02). nch = 1 (K = NP): one chunk.
struct Sched {
  long long tiles, w, we;
  int NP, nch, c, cs, Kc, k, nfull;
};
__device__ __forceinline__ void sched_init(Sched& s, long long tiles, int NP, int K) {
  s.tiles = tiles;
  s.NP = NP;
  s.nch = (NP + K - 1) / K;
  s.c = -1;
  s.w = s.we = 0;
  s.cs = s.Kc = 0;
  s.k = s.nfull = 0;
}
// next segment (tile, rows [p0, p1)) of this CTA; false when the CTA's work is done
__device__ __forceinline__ bool sched_next(Sched& s, long long& tile, int& p0, int& p1) {
  const long long G = gridDim.x, b = blockIdx.x;
  for (;;) {
    if (s.c >= 0) {
      if (s.k < s.nfull) {  // full group k: tile k G + b over every plane of the chunk
        tile = s.k * G + b;
        p0 = s.cs;
        p1 = s.cs + s.Kc;
        ++s.k;
        return true;
      }
      if (s.w < s.we) {  // partial group: a contiguous share of its (tile, plane) items
        const long long r = s.w;
        tile = (long long)s.nfull * G + r / s.Kc;
        p0 = s.cs + (int)(r % s.Kc);
        const long long rem = s.we - s.w;
        p1 = (rem < s.cs + s.Kc - p0) ? p0 + (int)rem : s.cs + s.Kc;
        s.w += p1 - p0;
        return true;
      }
    }
    if (++s.c >= s.nch) return false;
    s.cs = (int)((long long)s.c * s.NP / s.nch);
    s.Kc = (int)((long long)(s.c + 1) * s.NP / s.nch) - s.cs;
    s.nfull = (int)(s.tiles / G);
    s.k = 0;
    const long long items = (s.tiles - (long long)s.nfull * G) * s.Kc;
    s.w = items * b / G;
    s.we = items * (b + 1) / G;
  }
}

// Programmatic dependent launch (PDL) of the V-cycle's level kernels: launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, a kernel's CTAs may start (barrier init, smem
// carve-up, tensor-map use) while the previous kernel in the stream drains; pdl_wait() — before the
// kernel's first global-memory access — blocks until that kernel has completed and its writes are
// visible (a no-op for a plain launch). On the latency-bound coarse levels this hides part of the
// launch gap between consecutive kernels of the V-cycle's CUDA graph.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
#ifdef ST_NO_PDL
  cfg.numAttrs = 0;  // A/B builds: plain stream-ordered launches
#else
  cfg.numAttrs = 1;
#endif
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// planes per time chunk of a persistent stencil kernel's work list: the option when forced
// (op.chunk > 0), one chunk (tile-major order) when chunking is off (op.chunk < 0), else the
// kernel's automatic choice `auto_k` (only tv2d chunks automatically)
inline int chunk_planes(const OpDesc& op, int NP, int auto_k) {
  if (op.chunk > 0) return op.chunk < NP ? op.chunk : NP;
  if (op.chunk < 0) return NP;
  return auto_k < 1 ? 1 : (auto_k < NP ? auto_k : NP);
}

// persistent grid: one wave (nsm x resident CTAs), at most wtot / minw CTAs, at most op.max_ctas
inline long long persistent_grid(const OpDesc& op, int nsm, int resident, long long wtot) {
  long long grid = (long long)nsm * resident;
  // large levels: >= 4 planes per CTA (one reload plane per segment); small levels: every CTA a
  // short chain so that the TMA round trips of a level overlap (launch-latency bound there)
  const long long minw = (wtot >= 16LL * nsm * resident) ? 4 : 1;
  if (grid > wtot / minw) grid = wtot / minw;
  if (op.max_ctas > 0 && grid > op.max_ctas) grid = op.max_ctas;
  if (grid < 1) grid = 1;
  return grid;
}

}  // namespace st
