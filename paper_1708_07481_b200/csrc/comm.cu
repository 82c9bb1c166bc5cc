// Multi-GPU plumbing for row-sharded solves: NCCL over
// NVLink/NVSwitch, one process per GPU.
//
// NCCL is resolved at run time from the process (torch has already loaded the
// venv's libnccl.so.2; the same library is used, never a second copy), so the
// shared object itself has no link-time dependency on NCCL.
#include <dlfcn.h>

#include <vector>

#include <nccl.h>

#include "comm.cuh"

namespace spb {
namespace {

struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

NcclApi& api() {
  static NcclApi a;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      a.getUniqueId = (decltype(a.getUniqueId))dlsym(h, "ncclGetUniqueId");
      a.commInitRank = (decltype(a.commInitRank))dlsym(h, "ncclCommInitRank");
      a.commDestroy = (decltype(a.commDestroy))dlsym(h, "ncclCommDestroy");
      a.allReduce = (decltype(a.allReduce))dlsym(h, "ncclAllReduce");
      a.allGather = (decltype(a.allGather))dlsym(h, "ncclAllGather");
      a.getErrorString = (decltype(a.getErrorString))dlsym(h, "ncclGetErrorString");
      a.ok = a.getUniqueId && a.commInitRank && a.commDestroy && a.allReduce && a.allGather;
    }
  }
  return a;
}

int nccl_fail(ncclResult_t r, const char* what) {
  const char* msg = api().getErrorString ? api().getErrorString(r) : "?";
  set_error("NCCL %s failed: %s", what, msg);
  return SPB_ERR_CUDA;
}

}  // namespace

int comm_allreduce_f64(const Comm* c, double* buf, size_t count, cudaStream_t st) {
  if (!c || c->nranks <= 1 || count == 0) return SPB_OK;
  if (c->host_allreduce) {
    std::vector<double> h(count);
    SPB_CUDA(cudaMemcpyAsync(h.data(), buf, sizeof(double) * count, cudaMemcpyDeviceToHost, st));
    SPB_CUDA(cudaStreamSynchronize(st));
    if (c->host_allreduce(c->host_user, h.data(), (int64_t)count) != 0) {
      set_error("host allreduce callback failed");
      return SPB_ERR_CALLBACK;
    }
    SPB_CUDA(cudaMemcpyAsync(buf, h.data(), sizeof(double) * count, cudaMemcpyHostToDevice, st));
    SPB_CUDA(cudaStreamSynchronize(st));
    return SPB_OK;
  }
  ncclResult_t r = api().allReduce(buf, buf, count, ncclFloat64, ncclSum, (ncclComm_t)c->nccl, st);
  return r == ncclSuccess ? SPB_OK : nccl_fail(r, "allreduce");
}

int comm_allgather_bytes(const Comm* c, const void* send, void* recv, size_t bytes_per_rank,
                         cudaStream_t st) {
  if (!c || c->nranks <= 1) {
    if (send != recv && bytes_per_rank)
      SPB_CUDA(cudaMemcpyAsync(recv, send, bytes_per_rank, cudaMemcpyDeviceToDevice, st));
    return SPB_OK;
  }
  if (c->host_allgather) {
    std::vector<char> hs(bytes_per_rank), hr(bytes_per_rank * (size_t)c->nranks);
    SPB_CUDA(cudaMemcpyAsync(hs.data(), send, bytes_per_rank, cudaMemcpyDeviceToHost, st));
    SPB_CUDA(cudaStreamSynchronize(st));
    if (c->host_allgather(c->host_user, hs.data(), hr.data(), (int64_t)bytes_per_rank) != 0) {
      set_error("host allgather callback failed");
      return SPB_ERR_CALLBACK;
    }
    SPB_CUDA(cudaMemcpyAsync(recv, hr.data(), hr.size(), cudaMemcpyHostToDevice, st));
    SPB_CUDA(cudaStreamSynchronize(st));
    return SPB_OK;
  }
  ncclResult_t r = api().allGather(send, recv, bytes_per_rank, ncclInt8, (ncclComm_t)c->nccl, st);
  return r == ncclSuccess ? SPB_OK : nccl_fail(r, "allgather");
}

}  // namespace spb

using namespace spb;

extern "C" int spb_comm_unique_id(void* out, int32_t bytes) {
  if (bytes < (int)sizeof(ncclUniqueId)) {
    set_error("unique id buffer needs %d bytes", (int)sizeof(ncclUniqueId));
    return SPB_ERR_CONTRACT;
  }
  if (!api().ok) {
    set_error("libnccl.so.2 not available in this process");
    return SPB_ERR_CUDA;
  }
  ncclUniqueId id;
  ncclResult_t r = api().getUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "getUniqueId");
  memcpy(out, &id, sizeof(id));
  return SPB_OK;
}

extern "C" int spb_comm_init(int32_t nranks, int32_t rank, const void* id, void** comm_out) {
  if (nranks < 1 || rank < 0 || rank >= nranks) {
    set_error("bad communicator shape");
    return SPB_ERR_CONTRACT;
  }
  Comm* c = new Comm();
  c->nranks = nranks;
  c->rank = rank;
  c->nccl = nullptr;
  if (nranks > 1) {
    if (!api().ok) {
      delete c;
      set_error("libnccl.so.2 not available in this process");
      return SPB_ERR_CUDA;
    }
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    ncclComm_t nc = nullptr;
    ncclResult_t r = api().commInitRank(&nc, nranks, uid, rank);
    if (r != ncclSuccess) {
      delete c;
      return nccl_fail(r, "commInitRank");
    }
    c->nccl = nc;
  }
  *comm_out = c;
  return SPB_OK;
}

extern "C" int spb_comm_init_host(int32_t nranks, int32_t rank, spb_allreduce_cb allreduce,
                                  spb_allgather_cb allgather, void* user, void** comm_out) {
  if (nranks < 1 || rank < 0 || rank >= nranks || !allreduce || !allgather) {
    set_error("bad host communicator");
    return SPB_ERR_CONTRACT;
  }
  Comm* c = new Comm();
  c->nranks = nranks;
  c->rank = rank;
  c->nccl = nullptr;
  c->host_allreduce = allreduce;
  c->host_allgather = allgather;
  c->host_user = user;
  *comm_out = c;
  return SPB_OK;
}

// One-rank NCCL communicator driven through the same resolved entry points the
// sharded solver uses (unique id, init, float64 all-reduce, byte all-gather,
// destroy). A single-GPU box cannot form a larger communicator, so this is the
// check that the run-time NCCL binding itself works where the library is loaded.
extern "C" int spb_comm_selftest(void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!api().ok) {
    set_error("libnccl.so.2 not available in this process");
    return SPB_ERR_CUDA;
  }
  ncclUniqueId id;
  ncclResult_t r = api().getUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "getUniqueId");
  ncclComm_t nc = nullptr;
  r = api().commInitRank(&nc, 1, id, 0);
  if (r != ncclSuccess) return nccl_fail(r, "commInitRank");
  constexpr int kN = 1024;
  std::vector<double> h(kN), back(kN), gathered(kN);
  for (int i = 0; i < kN; ++i) h[i] = 0.5 * i - 3.0;
  double *d = nullptr, *g = nullptr;
  int rc = SPB_OK;
  auto body = [&]() -> int {
    SPB_CUDA(cudaMalloc(&d, sizeof(double) * kN));
    SPB_CUDA(cudaMalloc(&g, sizeof(double) * kN));
    SPB_CUDA(cudaMemcpyAsync(d, h.data(), sizeof(double) * kN, cudaMemcpyHostToDevice, st));
    r = api().allReduce(d, d, kN, ncclFloat64, ncclSum, nc, st);
    if (r != ncclSuccess) return nccl_fail(r, "allreduce");
    r = api().allGather(d, g, sizeof(double) * kN, ncclInt8, nc, st);
    if (r != ncclSuccess) return nccl_fail(r, "allgather");
    SPB_CUDA(cudaMemcpyAsync(back.data(), d, sizeof(double) * kN, cudaMemcpyDeviceToHost, st));
    SPB_CUDA(cudaMemcpyAsync(gathered.data(), g, sizeof(double) * kN, cudaMemcpyDeviceToHost, st));
    SPB_CUDA(cudaStreamSynchronize(st));
    for (int i = 0; i < kN; ++i)
      if (back[i] != h[i] || gathered[i] != h[i]) {
        set_error("NCCL one-rank collectives returned wrong data at %d", i);
        return SPB_ERR_CUDA;
      }
    return SPB_OK;
  };
  rc = body();
  cudaFree(d);
  cudaFree(g);
  api().commDestroy(nc);
  return rc;
}

extern "C" int spb_comm_destroy(void* comm) {
  Comm* c = (Comm*)comm;
  if (!c) return SPB_OK;
  if (c->nccl) api().commDestroy((ncclComm_t)c->nccl);
  delete c;
  return SPB_OK;
}
