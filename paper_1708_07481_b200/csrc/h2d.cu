// Host -> device staging of a large pageable host array through a caller-provided
// pinned ring, by several host threads (the public API's numpy inputs: the C3 x0
// block is 432 MB of float64, its arc list 160 MB).
//
// A pageable cudaMemcpy runs at ~11 GB/s on the B200 hosts (one driver thread stages
// it). Here thread t owns chunks t, t + T, t + 2T, ... and two slots of the ring: it
// copies (or narrows float64 -> float32, round to nearest even as numpy's astype
// does) a chunk into a free slot and enqueues that slot's DMA on the caller's stream;
// no thread waits for another, and the only host synchronisation is a slot's own
// previous DMA. The reference has no counterpart (its arrays stay on the host).
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "common.cuh"

namespace spb {
namespace {

constexpr size_t kSlot = 4u << 20;  // bytes per ring slot
constexpr int kSlotsPerThread = 2;

struct StageJob {
  const char* src;
  char* dst;            // device
  size_t count;         // elements
  int src_esz, dst_esz; // 8 -> 4 narrows float64 to float32; equal sizes copy bytes
  char* ring;
  int threads;
  cudaStream_t st;
  std::atomic<int> err{0};
};

void stage_worker(StageJob* job, int t) {
  const size_t per = kSlot / (size_t)job->dst_esz;  // elements per chunk
  const size_t nchunks = (job->count + per - 1) / per;
  cudaEvent_t ev[kSlotsPerThread];
  bool used[kSlotsPerThread] = {false, false};
  for (auto& e : ev)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) job->err = 1;
  int slot = 0;
  for (size_t c = (size_t)t; c < nchunks && !job->err; c += (size_t)job->threads) {
    char* buf = job->ring + ((size_t)t * kSlotsPerThread + slot) * kSlot;
    if (used[slot] && cudaEventSynchronize(ev[slot]) != cudaSuccess) job->err = 1;
    const size_t off = c * per, m = std::min(per, job->count - off);
    if (job->src_esz == job->dst_esz) {
      std::memcpy(buf, job->src + off * job->src_esz, m * job->src_esz);
    } else {
      const double* s = reinterpret_cast<const double*>(job->src) + off;
      float* d = reinterpret_cast<float*>(buf);
      for (size_t i = 0; i < m; ++i) d[i] = (float)s[i];
    }
    if (cudaMemcpyAsync(job->dst + off * job->dst_esz, buf, m * job->dst_esz,
                        cudaMemcpyHostToDevice, job->st) != cudaSuccess ||
        cudaEventRecord(ev[slot], job->st) != cudaSuccess)
      job->err = 1;
    used[slot] = true;
    slot ^= 1;
  }
  // the ring is the caller's to reuse on return: wait for this thread's DMAs
  for (int s = 0; s < kSlotsPerThread; ++s) {
    if (used[s] && cudaEventSynchronize(ev[s]) != cudaSuccess) job->err = 1;
    cudaEventDestroy(ev[s]);
  }
}

}  // namespace
}  // namespace spb

using namespace spb;

extern "C" size_t spb_h2d_ring_bytes(int32_t threads) {
  return (size_t)std::max(threads, 1) * kSlotsPerThread * kSlot;
}

extern "C" int spb_h2d_staged(const void* src, int64_t count, int32_t src_esz, int32_t dst_esz,
                              void* dst_dev, void* pinned_ring, size_t ring_bytes, int32_t threads,
                              void* stream) {
  if (count < 0 || threads < 1 || !(src_esz == dst_esz || (src_esz == 8 && dst_esz == 4)) ||
      dst_esz <= 0 || ring_bytes < spb_h2d_ring_bytes(threads)) {
    set_error("h2d staging: bad element sizes, thread count or ring size");
    return SPB_ERR_CONTRACT;
  }
  if (count == 0) return SPB_OK;
  StageJob job;
  job.src = (const char*)src;
  job.dst = (char*)dst_dev;
  job.count = (size_t)count;
  job.src_esz = src_esz;
  job.dst_esz = dst_esz;
  job.ring = (char*)pinned_ring;
  job.threads = threads;
  job.st = (cudaStream_t)stream;
  int dev = 0;
  SPB_CUDA(cudaGetDevice(&dev));
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t)
    pool.emplace_back([&job, t, dev] {
      if (cudaSetDevice(dev) != cudaSuccess) job.err = 1;
      stage_worker(&job, t);
    });
  stage_worker(&job, 0);
  for (auto& th : pool) th.join();
  if (job.err) {
    set_error("h2d staging: CUDA error in a staging thread (%s)",
              cudaGetErrorString(cudaGetLastError()));
    return SPB_ERR_CUDA;
  }
  return SPB_OK;
}
