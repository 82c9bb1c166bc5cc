// Locality ordering of the vertices for the Laplacian SpMM (an internal
// relabelling of the solve; nothing the reference computes -- its
// laplacian_apply, graph.py:253-278, runs scipy's csr_matvecs in the given order).
//
// Why: at C3/C4 the SpMM gathers one X row (ncols floats) per stored entry from
// an X block far larger than L2 (216 MB at C3), in the random order of the
// DC-SBM's vertex ids: ncu shows a 26 % L2 hit rate and 6.5 GB of DRAM reads per
// launch. Most edges of a block-model graph stay inside a block (5:1 at C3), so
// numbering the vertices block by block keeps the rows that a wave of warps
// gathers inside one block's few MB of X, which stay L2-resident.
//
// How (no labels are known up front): a few random-walk smoothing steps of
// 16 seeded random columns, Y <- D^-1 W Y, average each vertex's values over its
// neighbourhood; inside a block the walk mixes in a couple of steps while the
// between-block leak is slow, so vertices of one block end up with nearly the
// same 16-vector. Its sign pattern against the degree-weighted column means
// (the stationary component) is a 16-bit locality-sensitive key; a stable radix
// sort of the keys gives the new order perm[new] = old.
//
// The permuted CSR keeps every row's entries in their original order (only the
// column ids are renumbered), so the SpMM's per-row sums are bit-identical to
// the unpermuted ones; the solver maps x0 / refills / results through perm.
#include "common.cuh"
#include "dense.cuh"
#include "radix.cuh"
#include "scan.cuh"

namespace spb {
namespace {

constexpr int kWalkCols = 16;
constexpr int kMeanBlocks = 256;  // fixed: the reduction order does not depend on the device

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__global__ void walk_init(int32_t n, uint64_t seed, float* __restrict__ y) {
  const int64_t total = (int64_t)n * kWalkCols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t h = mix64(seed + 0x9e3779b97f4a7c15ull * (uint64_t)(i + 1));
    y[i] = (float)((double)(h >> 11) * 0x1.0p-53 - 0.5);
  }
}

// yout[i] = (sum_e w_e yin[col_e]) / d_i : one warp per row, eight neighbours
// in flight (four lanes per 16-float row).
template <typename T>
__global__ void __launch_bounds__(256)
walk_step(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
          const T* __restrict__ cv, const T* __restrict__ deg, const float* __restrict__ yin,
          float* __restrict__ yout) {
  const int lane = threadIdx.x & 31, g = lane >> 2, gl = lane & 3;
  const int32_t row = (int32_t)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (row >= n) return;
  const int32_t e0 = rp[row], e1 = rp[row + 1];
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int32_t eb = e0; eb < e1; eb += 32) {
    const int32_t my = eb + lane;
    int32_t cj = 0;
    float wv = 0.f;
    if (my < e1) {
      cj = __ldg(ci + my);
      wv = (float)__ldg(cv + my);
    }
    const int cnt = min(32, e1 - eb);
    for (int kk = 0; kk < cnt; kk += 8) {
      const int k = kk + g;
      const int srcl = k < cnt ? k : 0;
      const int32_t j = __shfl_sync(0xffffffffu, cj, srcl);
      const float w = __shfl_sync(0xffffffffu, wv, srcl);
      if (k < cnt) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(yin + (int64_t)j * kWalkCols) + gl);
        acc.x = fmaf(w, v.x, acc.x);
        acc.y = fmaf(w, v.y, acc.y);
        acc.z = fmaf(w, v.z, acc.z);
        acc.w = fmaf(w, v.w, acc.w);
      }
    }
    __syncwarp();
  }
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
    acc.w += __shfl_xor_sync(0xffffffffu, acc.w, o);
  }
  if (g == 0) {
    const float d = (float)deg[row];
    const float s = d > 0.f ? 1.f / d : 0.f;
    reinterpret_cast<float4*>(yout + (int64_t)row * kWalkCols)[gl] =
        make_float4(acc.x * s, acc.y * s, acc.z * s, acc.w * s);
  }
}

// Degree-weighted column sums, fixed-order two-level reduction:
// part[b][c] (c < 16) and part[b][16] = sum d.
template <typename T>
__global__ void __launch_bounds__(256)
wmean_partial(int32_t n, const T* __restrict__ deg, const float* __restrict__ y,
              double* __restrict__ part) {
  double s[kWalkCols + 1];
#pragma unroll
  for (int c = 0; c <= kWalkCols; ++c) s[c] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double d = (double)deg[i];
#pragma unroll
    for (int c = 0; c < kWalkCols; ++c) s[c] += d * (double)y[i * kWalkCols + c];
    s[kWalkCols] += d;
  }
  __shared__ double sm[8][kWalkCols + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c <= kWalkCols; ++c) {
    const double v = warp_sum(s[c]);
    if (lane == 0) sm[warp][c] = v;
  }
  __syncthreads();
  if (threadIdx.x <= kWalkCols) {
    double v = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += sm[w][threadIdx.x];
    part[blockIdx.x * (kWalkCols + 1) + threadIdx.x] = v;
  }
}

// one warp per column: lane-strided partials, then a fixed shuffle tree
__global__ void wmean_final(const double* __restrict__ part, int nb, float* __restrict__ mean) {
  const int lane = threadIdx.x & 31, c = threadIdx.x >> 5;
  if (c > kWalkCols) return;
  double v = 0.0, d = 0.0;
  for (int b = lane; b < nb; b += 32) {
    v += part[b * (kWalkCols + 1) + c];
    d += part[b * (kWalkCols + 1) + kWalkCols];
  }
  v = warp_sum(v);
  d = warp_sum(d);
  if (lane == 0 && c < kWalkCols) mean[c] = d > 0.0 ? (float)(v / d) : 0.f;
}

__global__ void walk_keys(int32_t n, const float* __restrict__ y, const float* __restrict__ mean,
                          uint64_t* __restrict__ keys, uint32_t* __restrict__ pay) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t k = 0;
#pragma unroll
    for (int c = 0; c < kWalkCols; ++c) k |= (y[i * kWalkCols + c] > mean[c] ? 1u : 0u) << c;
    keys[i] = k;
    pay[i] = (uint32_t)i;
  }
}

__global__ void perm_counts(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ perm,
                            int32_t* __restrict__ cnt, int32_t* __restrict__ inv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = perm[i];
    cnt[i] = rp[p + 1] - rp[p];
    inv[p] = (int32_t)i;
  }
}

// one warp per new row: entries in their original order, columns renumbered
template <typename T>
__global__ void __launch_bounds__(256)
perm_entries(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
             const T* __restrict__ cv, const T* __restrict__ deg, const int32_t* __restrict__ perm,
             const int32_t* __restrict__ inv, const int32_t* __restrict__ nrp,
             int32_t* __restrict__ oci, T* __restrict__ ocv, T* __restrict__ odeg) {
  const int lane = threadIdx.x & 31;
  const int32_t row = (int32_t)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (row >= n) return;
  const int32_t p = perm[row];
  const int32_t e0 = rp[p], len = rp[p + 1] - e0, o0 = nrp[row];
  for (int32_t k = lane; k < len; k += 32) {
    oci[o0 + k] = inv[__ldg(ci + e0 + k)];
    ocv[o0 + k] = cv[e0 + k];
  }
  if (lane == 0 && odeg) odeg[row] = deg[p];
}

template <typename S, typename D>
__global__ void permute_rows_k(const S* __restrict__ s, int64_t lds, D* __restrict__ d, int64_t ldd,
                               int64_t rows, int32_t cols, const int32_t* __restrict__ idx,
                               int scatter) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols;
    const int32_t c = (int32_t)(i - r * cols);
    const int64_t q = idx[r];
    if (scatter)
      d[q * ldd + c] = (D)s[r * lds + c];
    else
      d[r * ldd + c] = (D)s[q * lds + c];
  }
}

template <typename S, typename D>
int permute_rows_t(const void* s, int64_t lds, void* d, int64_t ldd, int64_t rows, int32_t cols,
                   const int32_t* idx, int scatter, cudaStream_t st) {
  const int64_t total = rows * cols;
  if (total <= 0) return SPB_OK;
  const int grid = (int)std::min<int64_t>(ceil_div(total, 256), (int64_t)num_sms() * 8);
  permute_rows_k<S, D><<<grid, 256, 0, st>>>((const S*)s, lds, (D*)d, ldd, rows, cols, idx, scatter);
  SPB_LAUNCH_CHECK();
  return SPB_OK;
}

struct OrderLayout {
  float *ya, *yb, *mean;
  double* part;
  uint64_t *ka, *kb;
  uint32_t *pa, *pb;
  int *counts, *scan_tmp;
};

OrderLayout carve_order(Arena& a, int64_t n) {
  OrderLayout L;
  const int64_t ntiles = ceil_div(std::max<int64_t>(n, 1), kSortTile);
  L.ya = a.take<float>(n * kWalkCols);
  L.yb = a.take<float>(n * kWalkCols);
  L.mean = a.take<float>(kWalkCols);
  L.part = a.take<double>((size_t)kMeanBlocks * (kWalkCols + 1));
  L.ka = a.take<uint64_t>(n);
  L.kb = a.take<uint64_t>(n);
  L.pa = a.take<uint32_t>(n);
  L.pb = a.take<uint32_t>(n);
  L.counts = a.take<int>((size_t)kRadix * ntiles + 1);
  L.scan_tmp = a.take<int>(scan_workspace_ints(std::max<int64_t>(kRadix * ntiles, n + 1)) + 8);
  return L;
}

int grid_rows(int64_t n) {
  return (int)std::min<int64_t>(ceil_div(std::max<int64_t>(n, 1), 256), (int64_t)num_sms() * 16);
}

template <typename T>
int vertex_order_t(int32_t n, const int32_t* rp, const int32_t* ci, const T* cv, const T* deg,
                   int steps, uint64_t seed, OrderLayout& L, int32_t* perm, cudaStream_t st) {
  walk_init<<<grid_rows((int64_t)n * kWalkCols), 256, 0, st>>>(n, seed, L.ya);
  SPB_LAUNCH_CHECK();
  float *yi = L.ya, *yo = L.yb;
  const int64_t wblocks = ceil_div((int64_t)n * 32, 256);
  for (int s = 0; s < steps; ++s) {
    walk_step<T><<<wblocks, 256, 0, st>>>(n, rp, ci, cv, deg, yi, yo);
    SPB_LAUNCH_CHECK();
    std::swap(yi, yo);
  }
  wmean_partial<T><<<kMeanBlocks, 256, 0, st>>>(n, deg, yi, L.part);
  wmean_final<<<1, 32 * (kWalkCols + 1), 0, st>>>(L.part, kMeanBlocks, L.mean);
  walk_keys<<<grid_rows(n), 256, 0, st>>>(n, yi, L.mean, L.ka, L.pa);
  SPB_LAUNCH_CHECK();
  uint64_t *kin = L.ka, *kout = L.kb;
  uint32_t *pin = L.pa, *pout = L.pb;
  SPB_TRY(radix_sort_pairs(&kin, &pin, &kout, &pout, n, kWalkCols, L.counts, L.scan_tmp, st));
  SPB_CUDA(cudaMemcpyAsync(perm, pin, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st));
  return SPB_OK;
}

template <typename T>
int csr_permute_t(int32_t n, const int32_t* rp, const int32_t* ci, const T* cv, const T* deg,
                  const int32_t* perm, int* scan_tmp, int32_t* inv, int32_t* nrp, int32_t* oci,
                  T* ocv, T* odeg, cudaStream_t st) {
  perm_counts<<<grid_rows(n), 256, 0, st>>>(n, rp, perm, nrp, inv);
  SPB_LAUNCH_CHECK();
  SPB_TRY(exclusive_scan_i32(nrp, nrp, n, scan_tmp, nrp + n, st));
  perm_entries<T><<<ceil_div((int64_t)n * 32, 256), 256, 0, st>>>(n, rp, ci, cv, deg, perm, inv,
                                                                   nrp, oci, ocv, odeg);
  SPB_LAUNCH_CHECK();
  return SPB_OK;
}

}  // namespace

int permute_rows(int sdt, const void* s, int64_t lds, int ddt, void* d, int64_t ldd, int64_t rows,
                 int32_t cols, const int32_t* idx, int scatter, cudaStream_t st) {
  if (sdt == SPB_F64 && ddt == SPB_F64)
    return permute_rows_t<double, double>(s, lds, d, ldd, rows, cols, idx, scatter, st);
  if (sdt == SPB_F64 && ddt == SPB_F32)
    return permute_rows_t<double, float>(s, lds, d, ldd, rows, cols, idx, scatter, st);
  if (sdt == SPB_F32 && ddt == SPB_F64)
    return permute_rows_t<float, double>(s, lds, d, ldd, rows, cols, idx, scatter, st);
  return permute_rows_t<float, float>(s, lds, d, ldd, rows, cols, idx, scatter, st);
}

}  // namespace spb

using namespace spb;

extern "C" size_t spb_vertex_order_workspace(int32_t n) {
  Arena a;
  a.dry = true;
  carve_order(a, std::max<int32_t>(n, 1));
  return a.used + 1024;
}

extern "C" int spb_vertex_order(int dtype, int32_t n, const int32_t* row_ptr, const int32_t* col,
                                const void* val, const void* deg, int32_t steps, uint64_t seed,
                                void* ws, size_t ws_bytes, int32_t* perm, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype != SPB_F32 && dtype != SPB_F64) {
    set_error("unknown dtype %d", dtype);
    return SPB_ERR_DOMAIN;
  }
  if (n < 0 || steps < 0) {
    set_error("vertex order: negative n or steps");
    return SPB_ERR_CONTRACT;
  }
  if (n == 0) return SPB_OK;
  Arena a;
  a.base = (char*)ws;
  a.cap = ws_bytes;
  OrderLayout L = carve_order(a, n);
  if (a.used > ws_bytes) {
    set_error("vertex order workspace too small (%zu < %zu)", ws_bytes, a.used);
    return SPB_ERR_WORKSPACE;
  }
  if (dtype == SPB_F32)
    return vertex_order_t<float>(n, row_ptr, col, (const float*)val, (const float*)deg, steps, seed,
                                 L, perm, st);
  return vertex_order_t<double>(n, row_ptr, col, (const double*)val, (const double*)deg, steps,
                                seed, L, perm, st);
}

extern "C" size_t spb_csr_permute_workspace(int32_t n) {
  return sizeof(int) * (scan_workspace_ints(std::max<int64_t>(n, 1) + 1) + 8) + 256;
}

extern "C" int spb_csr_permute(int dtype, int32_t n, const int32_t* row_ptr, const int32_t* col,
                               const void* val, const void* deg, const int32_t* perm, void* ws,
                               size_t ws_bytes, int32_t* inv, int32_t* out_row_ptr,
                               int32_t* out_col, void* out_val, void* out_deg, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype != SPB_F32 && dtype != SPB_F64) {
    set_error("unknown dtype %d", dtype);
    return SPB_ERR_DOMAIN;
  }
  if (n < 0) {
    set_error("csr permute: negative n");
    return SPB_ERR_CONTRACT;
  }
  if (ws_bytes < spb_csr_permute_workspace(n)) {
    set_error("csr permute workspace too small");
    return SPB_ERR_WORKSPACE;
  }
  if (n == 0) {
    SPB_CUDA(cudaMemsetAsync(out_row_ptr, 0, sizeof(int32_t), st));
    return SPB_OK;
  }
  int* tmp = (int*)ws;
  if (dtype == SPB_F32)
    return csr_permute_t<float>(n, row_ptr, col, (const float*)val, (const float*)deg, perm, tmp,
                                inv, out_row_ptr, out_col, (float*)out_val, (float*)out_deg, st);
  return csr_permute_t<double>(n, row_ptr, col, (const double*)val, (const double*)deg, perm, tmp,
                               inv, out_row_ptr, out_col, (double*)out_val, (double*)out_deg, st);
}

extern "C" int spb_permute_rows(int src_dtype, const void* src, int64_t lds, int dst_dtype,
                                void* dst, int64_t ldd, int64_t rows, int32_t cols,
                                const int32_t* idx, int scatter, void* stream) {
  if ((src_dtype != SPB_F32 && src_dtype != SPB_F64) ||
      (dst_dtype != SPB_F32 && dst_dtype != SPB_F64)) {
    set_error("unknown dtype");
    return SPB_ERR_DOMAIN;
  }
  if (lds < cols || ldd < cols || rows < 0) {
    set_error("permute_rows shape contract violated");
    return SPB_ERR_CONTRACT;
  }
  return permute_rows(src_dtype, src, lds, dst_dtype, dst, ldd, rows, cols, idx, scatter,
                      (cudaStream_t)stream);
}
