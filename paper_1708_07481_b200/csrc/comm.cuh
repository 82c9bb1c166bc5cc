// Communicator handle for row-sharded solves (comm.cu).
#pragma once
#include "common.cuh"

namespace spb {

struct Comm {
  void* nccl;  // ncclComm_t (null for a single rank or the host transport)
  int nranks;
  int rank;
  // host transport (spb_comm_init_host): collectives staged through host memory
  spb_allreduce_cb host_allreduce = nullptr;
  spb_allgather_cb host_allgather = nullptr;
  void* host_user = nullptr;
};

// In-place float64 sum over ranks (no-op for one rank).
int comm_allreduce_f64(const Comm* c, double* buf, size_t count, cudaStream_t st);
// recv[r * bytes_per_rank ...] = send of rank r.
int comm_allgather_bytes(const Comm* c, const void* send, void* recv, size_t bytes_per_rank,
                         cudaStream_t st);

}  // namespace spb
