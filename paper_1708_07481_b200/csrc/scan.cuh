// Device-wide exclusive prefix sum of int32 (three-phase reduce/scan/propagate).
#pragma once
#include "common.cuh"

namespace spb {
namespace {  // internal linkage: every TU that includes this gets its own copy

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

// Block-level exclusive scan of one int per thread; returns the block total.
__device__ __forceinline__ int block_excl_scan(int v, int* smem_warp, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int nw = blockDim.x >> 5;
    int w = lane < nw ? smem_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    smem_warp[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  int before = warp > 0 ? smem_warp[warp - 1] : 0;
  total = smem_warp[(blockDim.x >> 5) - 1];
  __syncthreads();
  return before + x - v;
}

__global__ void scan_tile_sums(const int* __restrict__ in, int64_t n, int* __restrict__ sums) {
  __shared__ int sw[32];
  int64_t base = (int64_t)blockIdx.x * kScanTile + threadIdx.x * kScanItems;
  int s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i)
    if (base + i < n) s += in[base + i];
  int tot;
  block_excl_scan(s, sw, tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// Single CTA: exclusive scan of the tile sums, in chunks, carrying the offset.
__global__ void scan_sums_serial(int* __restrict__ sums, int64_t ntiles, int* __restrict__ total) {
  __shared__ int sw[32];
  int carry = 0;
  for (int64_t base = 0; base < ntiles; base += blockDim.x) {
    int64_t i = base + threadIdx.x;
    int v = i < ntiles ? sums[i] : 0;
    int tot;
    int ex = block_excl_scan(v, sw, tot);
    if (i < ntiles) sums[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void scan_tiles_apply(const int* __restrict__ in, int64_t n,
                                 const int* __restrict__ sums, int* __restrict__ out) {
  __shared__ int sw[32];
  int64_t base = (int64_t)blockIdx.x * kScanTile + threadIdx.x * kScanItems;
  int v[kScanItems];
  int s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = base + i < n ? in[base + i] : 0;
    s += v[i];
  }
  int tot;
  int ex = block_excl_scan(s, sw, tot) + sums[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = ex;
    ex += v[i];
  }
}

inline size_t scan_workspace_ints(int64_t n) { return (size_t)ceil_div(n, kScanTile) + 1; }

// out may alias in. total (device int*) may be null.
inline int exclusive_scan_i32(const int* in, int* out, int64_t n, int* tmp, int* total,
                              cudaStream_t st) {
  int64_t ntiles = ceil_div(n, kScanTile);
  if (ntiles == 0) {
    if (total) SPB_CUDA(cudaMemsetAsync(total, 0, sizeof(int), st));
    return SPB_OK;
  }
  scan_tile_sums<<<ntiles, kScanThreads, 0, st>>>(in, n, tmp);
  scan_sums_serial<<<1, kScanThreads, 0, st>>>(tmp, ntiles, total);
  scan_tiles_apply<<<ntiles, kScanThreads, 0, st>>>(in, n, tmp, out);
  SPB_LAUNCH_CHECK();
  return SPB_OK;
}

}  // namespace
}  // namespace spb
