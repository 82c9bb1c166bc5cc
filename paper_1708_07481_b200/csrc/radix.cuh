// Stable LSD radix sort of (uint64 key, uint32 payload) pairs, 8-bit digits:
// per-tile digit histograms, one device-wide exclusive scan, stable scatter
// (items of a tile ranked in index order). Used by the CSR build (csr_build.cu)
// and the locality ordering (reorder.cu).
#pragma once
#include <utility>

#include "common.cuh"
#include "scan.cuh"

namespace spb {
namespace {

constexpr int kSortThreads = 256;
constexpr int kSortRounds = 16;
constexpr int kSortTile = kSortThreads * kSortRounds;  // 4096 items per tile
constexpr int kRadix = 256;

__global__ void radix_hist(const uint64_t* __restrict__ keys, int64_t count, int shift,
                           int64_t ntiles, int* __restrict__ counts) {
  __shared__ int h[kRadix];
  h[threadIdx.x] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * kSortTile;
#pragma unroll 4
  for (int r = 0; r < kSortRounds; ++r) {
    int64_t i = base + r * kSortThreads + threadIdx.x;
    if (i < count) atomicAdd(&h[(keys[i] >> shift) & 0xff], 1);
  }
  __syncthreads();
  counts[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// Stable scatter: items of a tile are ranked in index order (round, warp, lane).
__global__ void radix_scatter(const uint64_t* __restrict__ kin, const uint32_t* __restrict__ pin,
                              int64_t count, int shift, int64_t ntiles,
                              const int* __restrict__ offsets, uint64_t* __restrict__ kout,
                              uint32_t* __restrict__ pout) {
  __shared__ int running[kRadix];
  __shared__ int wcnt[kSortThreads / 32][kRadix];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  running[t] = offsets[(int64_t)t * ntiles + blockIdx.x];
  int64_t base = (int64_t)blockIdx.x * kSortTile;
  const unsigned lt = (1u << lane) - 1u;
  for (int r = 0; r < kSortRounds; ++r) {
#pragma unroll
    for (int w = 0; w < kSortThreads / 32; ++w) wcnt[w][t] = 0;
    __syncthreads();
    int64_t i = base + r * kSortThreads + t;
    bool valid = i < count;
    uint64_t k = valid ? kin[i] : 0;
    uint32_t p = valid ? pin[i] : 0;
    int d = valid ? (int)((k >> shift) & 0xff) : kRadix;  // kRadix = none
    unsigned peers = __match_any_sync(0xffffffffu, d);
    int lrank = __popc(peers & lt);
    if (valid && lrank == 0) wcnt[warp][d] = __popc(peers);
    __syncthreads();
    if (valid) {
      int pos = running[d] + lrank;
      for (int w = 0; w < warp; ++w) pos += wcnt[w][d];
      kout[pos] = k;
      pout[pos] = p;
    }
    __syncthreads();
    int add = 0;
#pragma unroll
    for (int w = 0; w < kSortThreads / 32; ++w) add += wcnt[w][t];
    running[t] += add;
    __syncthreads();
  }
}

// Sorts `count` pairs by key bits [0, bits); the result lands in (*kin, *pin)
// (the buffers are swapped pass by pass). counts: kRadix * ntiles + 1 ints;
// scan_tmp: scan_workspace_ints(kRadix * ntiles) ints.
inline int radix_sort_pairs(uint64_t** kin, uint32_t** pin, uint64_t** kout, uint32_t** pout,
                            int64_t count, int bits, int* counts, int* scan_tmp, cudaStream_t st) {
  const int64_t ntiles = ceil_div(count, kSortTile);
  for (int shift = 0; count > 0 && shift < bits; shift += 8) {
    radix_hist<<<ntiles, kSortThreads, 0, st>>>(*kin, count, shift, ntiles, counts);
    SPB_TRY(exclusive_scan_i32(counts, counts, (int64_t)kRadix * ntiles, scan_tmp, nullptr, st));
    radix_scatter<<<ntiles, kSortThreads, 0, st>>>(*kin, *pin, count, shift, ntiles, counts, *kout,
                                                   *pout);
    SPB_LAUNCH_CHECK();
    std::swap(*kin, *kout);
    std::swap(*pin, *pout);
  }
  return SPB_OK;
}

}  // namespace
}  // namespace spb
