// comm.cu — time-slab transport of libst: halo planes between time
// neighbours, sums of Krylov inner products, gathers for agglomerated coarse levels.
//
// Two transports behind one interface:
//   * NCCL (one process per GPU; NVLink 5 / NVSwitch): grouped ncclSend/ncclRecv for the two
//     halo planes, ncclAllReduce / ncclAllGather for reductions and agglomeration, all enqueued
//     on the context stream (no host synchronisation). libnccl is opened at run time
//     (dlopen, reusing the copy the process already loaded, e.g. PyTorch's), so libst has no
//     link-time NCCL dependency.
//   * HOST callbacks (st_host_comm_t): device buffers staged through pinned host memory and
//     handed to caller-supplied functions (the Python binding implements them with
//     torch.distributed, e.g. gloo). Used to run and test the slab path with several ranks on
//     one GPU: the ranks never wait on each other inside a kernel, only on the host.
#include <dlfcn.h>

#include <cstring>
#include <string>
#include <vector>

#include "comm.h"

namespace st {

namespace {
// minimal NCCL ABI (types from nccl.h, stable across 2.x)
typedef enum { ncclSuccess_ = 0 } ncclResult_t_;
typedef int (*p_ncclGetUniqueId)(void* id);
typedef int (*p_ncclCommInitRank)(void** comm, int nranks, const char* id /* ncclUniqueId by value */, int rank);
typedef int (*p_ncclCommDestroy)(void* comm);
typedef int (*p_ncclGroupStart)();
typedef int (*p_ncclGroupEnd)();
typedef int (*p_ncclSend)(const void* buf, size_t count, int dtype, int peer, void* comm, cudaStream_t s);
typedef int (*p_ncclRecv)(void* buf, size_t count, int dtype, int peer, void* comm, cudaStream_t s);
typedef int (*p_ncclAllReduce)(const void* s, void* r, size_t count, int dtype, int op, void* comm, cudaStream_t st);
typedef int (*p_ncclAllGather)(const void* s, void* r, size_t count, int dtype, void* comm, cudaStream_t st);
typedef const char* (*p_ncclGetErrorString)(int);
typedef int (*p_ncclCommCount)(void* comm, int* count);
typedef int (*p_ncclCommUserRank)(void* comm, int* rank);
constexpr int kNcclDouble = 8;  // ncclFloat64
constexpr int kNcclSum = 0;

struct NcclApi {
  bool ok = false;
  p_ncclGetUniqueId getUniqueId = nullptr;
  void* commInitRank = nullptr;  // called through a by-value ncclUniqueId wrapper below
  p_ncclCommDestroy commDestroy = nullptr;
  p_ncclGroupStart groupStart = nullptr;
  p_ncclGroupEnd groupEnd = nullptr;
  p_ncclSend send = nullptr;
  p_ncclRecv recv = nullptr;
  p_ncclAllReduce allReduce = nullptr;
  p_ncclAllGather allGather = nullptr;
  p_ncclGetErrorString errStr = nullptr;
  p_ncclCommCount commCount = nullptr;
  p_ncclCommUserRank commUserRank = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
  api.getUniqueId = (p_ncclGetUniqueId)dlsym(h, "ncclGetUniqueId");
  api.commInitRank = dlsym(h, "ncclCommInitRank");
  api.commDestroy = (p_ncclCommDestroy)dlsym(h, "ncclCommDestroy");
  api.groupStart = (p_ncclGroupStart)dlsym(h, "ncclGroupStart");
  api.groupEnd = (p_ncclGroupEnd)dlsym(h, "ncclGroupEnd");
  api.send = (p_ncclSend)dlsym(h, "ncclSend");
  api.recv = (p_ncclRecv)dlsym(h, "ncclRecv");
  api.allReduce = (p_ncclAllReduce)dlsym(h, "ncclAllReduce");
  api.allGather = (p_ncclAllGather)dlsym(h, "ncclAllGather");
  api.errStr = (p_ncclGetErrorString)dlsym(h, "ncclGetErrorString");
  api.commCount = (p_ncclCommCount)dlsym(h, "ncclCommCount");
  api.commUserRank = (p_ncclCommUserRank)dlsym(h, "ncclCommUserRank");
  api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.groupStart && api.groupEnd && api.send &&
           api.recv && api.allReduce && api.allGather;
  return api;
}

struct UniqueId {
  char internal[ST_NCCL_ID_BYTES];
};
typedef int (*p_ncclCommInitRankById)(void** comm, int nranks, UniqueId id, int rank);

void nccl_check(int r, const char* what) {
  if (r != 0) {
    const char* e = nccl().errStr ? nccl().errStr(r) : "?";
    throw CommError{std::string(what) + ": " + e};
  }
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CommError{std::string(what) + ": " + cudaGetErrorString(e)};
}

double* host_stage(Comm& c, size_t count) {
  if (c.hcap < count) {
    if (c.hbuf) cudaFreeHost(c.hbuf);
    c.hbuf = nullptr;
    cuda_check(cudaMallocHost((void**)&c.hbuf, count * sizeof(double)), "cudaMallocHost");
    c.hcap = count;
  }
  return c.hbuf;
}
}  // namespace

bool nccl_available() { return nccl().ok; }

int nccl_unique_id(char* out) {
  if (!nccl().ok) return -1;
  UniqueId id;
  int r = nccl().getUniqueId(&id);
  if (r != 0) return r;
  memcpy(out, id.internal, ST_NCCL_ID_BYTES);
  return 0;
}

int nccl_comm_init(const char* id_bytes, int rank, int size, void** comm) {
  if (!nccl().ok) return -1;
  UniqueId id;
  memcpy(id.internal, id_bytes, ST_NCCL_ID_BYTES);
  return ((p_ncclCommInitRankById)nccl().commInitRank)(comm, size, id, rank);
}

int nccl_comm_destroy(void* comm) {
  if (!nccl().ok || !comm) return -1;
  return nccl().commDestroy(comm);
}

int nccl_comm_count(void* comm, int* count, int* rank) {
  if (!nccl().ok || !comm || !nccl().commCount || !nccl().commUserRank) return -1;
  if (nccl().commCount(comm, count) != 0) return -1;
  if (nccl().commUserRank(comm, rank) != 0) return -1;
  return 0;
}

std::string nccl_selftest(void* comm, int rank, int size, cudaStream_t s) {
  NcclApi& api = nccl();
  if (!api.ok) return "libnccl.so.2 not available";
  const int n = 64;
  double* d = nullptr;
  if (cudaMalloc((void**)&d, (size_t)(5 + size) * n * sizeof(double)) != cudaSuccess) return "cudaMalloc";
  double* a = d;              // allreduce: every rank contributes (rank + 1) * (i + 1)
  double* g = d + n;          // allgather target: size * n
  double* sl = g + size * n;  // send to rank - 1 (ring), receive from rank + 1
  double* rl = sl + n;
  double* sh = rl + n;        // send to rank + 1, receive from rank - 1
  std::vector<double> h((size_t)(5 + size) * n, 0.0);  // a | g[size] | sl | rl | sh | rh
  for (int i = 0; i < n; ++i) {
    h[i] = (rank + 1.0) * (i + 1.0);
    h[(size_t)(size + 1) * n + i] = 1000.0 * rank + i;      // sl
    h[(size_t)(size + 3) * n + i] = -1000.0 * rank - i;     // sh
  }
  std::string err;
  try {
    cuda_check(cudaMemcpyAsync(d, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, s), "H2D");
    nccl_check(api.allReduce(a, a, n, kNcclDouble, kNcclSum, comm, s), "ncclAllReduce");
    nccl_check(api.allGather(a, g, n, kNcclDouble, comm, s), "ncclAllGather");
    const int lo = (rank + size - 1) % size, hi = (rank + 1) % size;
    double* rh = sh + n;
    nccl_check(api.groupStart(), "ncclGroupStart");
    nccl_check(api.send(sl, n, kNcclDouble, lo, comm, s), "ncclSend");
    nccl_check(api.recv(rl, n, kNcclDouble, hi, comm, s), "ncclRecv");
    nccl_check(api.send(sh, n, kNcclDouble, hi, comm, s), "ncclSend");
    nccl_check(api.recv(rh, n, kNcclDouble, lo, comm, s), "ncclRecv");
    nccl_check(api.groupEnd(), "ncclGroupEnd");
    std::vector<double> o(h.size());
    cuda_check(cudaMemcpyAsync(o.data(), d, h.size() * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
    cuda_check(cudaStreamSynchronize(s), "sync");
    const double tri = size * (size + 1) / 2.0;
    for (int i = 0; i < n && err.empty(); ++i) {
      if (o[i] != tri * (i + 1.0)) err = "allreduce value";
      for (int r = 0; r < size && err.empty(); ++r)
        if (o[(size_t)(1 + r) * n + i] != tri * (i + 1.0)) err = "allgather value";
      if (err.empty() && o[(size_t)(size + 2) * n + i] != 1000.0 * hi + i) err = "send/recv (from rank + 1)";
      if (err.empty() && o[(size_t)(size + 4) * n + i] != -1000.0 * lo - i) err = "send/recv (from rank - 1)";
    }
  } catch (const CommError& e) {
    err = e.msg;
  }
  cudaFree(d);
  return err;
}

void comm_release(Comm& c) {
  if (c.hbuf) cudaFreeHost(c.hbuf);
  c.hbuf = nullptr;
  c.hcap = 0;
}

// Halo planes: send_lo -> rank-1 (received there into its recv_hi), send_hi -> rank+1; receive
// recv_lo from rank-1 and recv_hi from rank+1. Pointers of a missing neighbour are ignored.
void comm_halo(Comm& c, const double* send_lo, double* recv_lo, const double* send_hi, double* recv_hi,
               long long count, cudaStream_t s) {
  if (c.size <= 1) return;
  const bool lo = c.rank > 0, hi = c.rank < c.size - 1;
  if (c.kind == ST_COMM_NCCL) {
    NcclApi& api = nccl();
    nccl_check(api.groupStart(), "ncclGroupStart");
    if (lo) {
      nccl_check(api.send(send_lo, (size_t)count, kNcclDouble, c.rank - 1, c.nccl, s), "ncclSend");
      nccl_check(api.recv(recv_lo, (size_t)count, kNcclDouble, c.rank - 1, c.nccl, s), "ncclRecv");
    }
    if (hi) {
      nccl_check(api.send(send_hi, (size_t)count, kNcclDouble, c.rank + 1, c.nccl, s), "ncclSend");
      nccl_check(api.recv(recv_hi, (size_t)count, kNcclDouble, c.rank + 1, c.nccl, s), "ncclRecv");
    }
    nccl_check(api.groupEnd(), "ncclGroupEnd");
    return;
  }
  // host transport: lower neighbour first (a chain: rank 0 pairs with 1 first, 1 with 0, ...)
  double* h = host_stage(c, 2 * (size_t)count);
  for (int side = 0; side < 2; ++side) {
    const bool on = side == 0 ? lo : hi;
    if (!on) continue;
    const double* sd = side == 0 ? send_lo : send_hi;
    double* rd = side == 0 ? recv_lo : recv_hi;
    cuda_check(cudaMemcpyAsync(h, sd, count * sizeof(double), cudaMemcpyDeviceToHost, s), "halo D2H");
    cuda_check(cudaStreamSynchronize(s), "halo sync");
    const int peer = side == 0 ? c.rank - 1 : c.rank + 1;
    if (c.host.sendrecv(c.host.user, peer, h, h + count, count) != 0) throw CommError{"host sendrecv failed"};
    cuda_check(cudaMemcpyAsync(rd, h + count, count * sizeof(double), cudaMemcpyHostToDevice, s), "halo H2D");
    cuda_check(cudaStreamSynchronize(s), "halo sync");
  }
}

// one direction only: every rank r < size-1 receives recv_hi from rank r+1, which sends send_lo
void comm_shift_down(Comm& c, const double* send_lo, double* recv_hi, long long count, cudaStream_t s) {
  if (c.size <= 1) return;
  const bool lo = c.rank > 0, hi = c.rank < c.size - 1;
  if (c.kind == ST_COMM_NCCL) {
    NcclApi& api = nccl();
    nccl_check(api.groupStart(), "ncclGroupStart");
    if (lo) nccl_check(api.send(send_lo, (size_t)count, kNcclDouble, c.rank - 1, c.nccl, s), "ncclSend");
    if (hi) nccl_check(api.recv(recv_hi, (size_t)count, kNcclDouble, c.rank + 1, c.nccl, s), "ncclRecv");
    nccl_check(api.groupEnd(), "ncclGroupEnd");
    return;
  }
  // host: implemented as a halo exchange with dummy payloads in the unused direction
  double* h = host_stage(c, 2 * (size_t)count);
  for (int side = 0; side < 2; ++side) {
    const bool on = side == 0 ? lo : hi;
    if (!on) continue;
    if (side == 0) {
      cuda_check(cudaMemcpyAsync(h, send_lo, count * sizeof(double), cudaMemcpyDeviceToHost, s), "shift D2H");
      cuda_check(cudaStreamSynchronize(s), "shift sync");
    } else {
      memset(h, 0, count * sizeof(double));
    }
    const int peer = side == 0 ? c.rank - 1 : c.rank + 1;
    if (c.host.sendrecv(c.host.user, peer, h, h + count, count) != 0) throw CommError{"host sendrecv failed"};
    if (side == 1) {
      cuda_check(cudaMemcpyAsync(recv_hi, h + count, count * sizeof(double), cudaMemcpyHostToDevice, s), "shift H2D");
      cuda_check(cudaStreamSynchronize(s), "shift sync");
    }
  }
}

void comm_allreduce(Comm& c, double* d, long long count, cudaStream_t s) {
  if (c.size <= 1) return;
  if (c.kind == ST_COMM_NCCL) {
    nccl_check(nccl().allReduce(d, d, (size_t)count, kNcclDouble, kNcclSum, c.nccl, s), "ncclAllReduce");
    return;
  }
  double* h = host_stage(c, (size_t)count);
  cuda_check(cudaMemcpyAsync(h, d, count * sizeof(double), cudaMemcpyDeviceToHost, s), "allreduce D2H");
  cuda_check(cudaStreamSynchronize(s), "allreduce sync");
  if (c.host.allreduce_sum(c.host.user, h, count) != 0) throw CommError{"host allreduce failed"};
  cuda_check(cudaMemcpyAsync(d, h, count * sizeof(double), cudaMemcpyHostToDevice, s), "allreduce H2D");
  cuda_check(cudaStreamSynchronize(s), "allreduce sync");
}

// recv (size * count) = concatenation over ranks of every rank's send (count)
void comm_allgather(Comm& c, const double* send, double* recv, long long count, cudaStream_t s) {
  if (c.size <= 1) {
    if (recv != send) cuda_check(cudaMemcpyAsync(recv, send, count * sizeof(double), cudaMemcpyDeviceToDevice, s), "copy");
    return;
  }
  if (c.kind == ST_COMM_NCCL) {
    nccl_check(nccl().allGather(send, recv, (size_t)count, kNcclDouble, c.nccl, s), "ncclAllGather");
    return;
  }
  double* h = host_stage(c, (size_t)count * (c.size + 1));
  cuda_check(cudaMemcpyAsync(h, send, count * sizeof(double), cudaMemcpyDeviceToHost, s), "allgather D2H");
  cuda_check(cudaStreamSynchronize(s), "allgather sync");
  if (c.host.allgather(c.host.user, h, h + count, count) != 0) throw CommError{"host allgather failed"};
  cuda_check(cudaMemcpyAsync(recv, h + count, (size_t)count * c.size * sizeof(double), cudaMemcpyHostToDevice, s),
             "allgather H2D");
  cuda_check(cudaStreamSynchronize(s), "allgather sync");
}

}  // namespace st
