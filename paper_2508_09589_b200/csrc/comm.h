// comm.h — time-slab transport of libst (internal). See comm.cu.
#pragma once
#include <cuda_runtime.h>

#include <string>

#include "st.h"

namespace st {

struct CommError {
  std::string msg;
};

struct Comm {
  int rank = 0, size = 1;
  int kind = ST_COMM_NONE;
  void* nccl = nullptr;     // ncclComm_t (caller-owned)
  st_host_comm_t host{};    // host-callback transport
  double* hbuf = nullptr;   // pinned staging (host transport)
  size_t hcap = 0;
};

bool nccl_available();
int nccl_unique_id(char* out);                                  // ST_NCCL_ID_BYTES bytes
int nccl_comm_init(const char* id, int rank, int size, void** comm);
int nccl_comm_destroy(void* comm);
// ncclCommCount / ncclCommUserRank of a communicator (-1 on failure)
int nccl_comm_count(void* comm, int* count, int* rank);
// exercise every NCCL entry point the slab path uses on a communicator (any size, including 1):
// allreduce, allgather and a grouped send/recv exchange with the ring neighbours (self when size 1);
// returns "" on success, else the first failure
std::string nccl_selftest(void* comm, int rank, int size, cudaStream_t s);
void comm_release(Comm& c);
// halo planes with both time neighbours (count doubles each)
void comm_halo(Comm& c, const double* send_lo, double* recv_lo, const double* send_hi, double* recv_hi,
               long long count, cudaStream_t s);
// one direction: rank r sends send_lo to r-1 and receives recv_hi from r+1
void comm_shift_down(Comm& c, const double* send_lo, double* recv_hi, long long count, cudaStream_t s);
void comm_allreduce(Comm& c, double* d, long long count, cudaStream_t s);  // in place, sum
void comm_allgather(Comm& c, const double* send, double* recv, long long count, cudaStream_t s);

}  // namespace st
