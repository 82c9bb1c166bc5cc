// Communicator handle for row-sharded solves (comm.cu).
#pragma once
#include "common.cuh"

namespace spb {

struct Comm {
  void* nccl;  // ncclComm_t (null for a single rank)
  int nranks;
  int rank;
};

// In-place float64 sum over ranks (no-op for one rank).
int comm_allreduce_f64(const Comm* c, double* buf, size_t count, cudaStream_t st);
// recv[r * bytes_per_rank ...] = send of rank r.
int comm_allgather_bytes(const Comm* c, const void* send, void* recv, size_t bytes_per_rank,
                         cudaStream_t st);

}  // namespace spb
