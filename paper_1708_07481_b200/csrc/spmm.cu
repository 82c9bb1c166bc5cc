// (b) Matrix-free Laplacian block product on the symmetrised CSR:
//     Y[i, :] = d_i X[i, :] - sum_{e in row i} W_e X[col_e, :]
// Replaces laplacian_apply (graph.py:253-278) / LaplacianOperator.apply
// (graph.py:316-317), which run scipy's serial csr_matvecs twice (A and A').
//
// One warp per row. The row's (col, val) pairs are loaded 32 at a time,
// coalesced, and broadcast with shuffles. The dense block is vertex-major, so a
// neighbour's row of X is one contiguous run of ncols values, read as 128-bit
// vectors (float4 / double2). When the row is narrower than a warp's vector
// width the warp splits into lane groups that walk different neighbours and
// are combined with xor-shuffles at the end.
#include <cstdlib>

#include "common.cuh"

namespace spb {
namespace {

template <typename T> struct Vec;
template <> struct Vec<float> { using type = float4; static constexpr int N = 4; };
template <> struct Vec<double> { using type = double2; static constexpr int N = 2; };

template <typename V> __device__ __forceinline__ V vzero();
template <> __device__ __forceinline__ float4 vzero<float4>() { return make_float4(0, 0, 0, 0); }
template <> __device__ __forceinline__ double2 vzero<double2>() { return make_double2(0, 0); }

__device__ __forceinline__ void vfma(float4& a, float s, const float4& x) {
  a.x = fmaf(s, x.x, a.x); a.y = fmaf(s, x.y, a.y); a.z = fmaf(s, x.z, a.z); a.w = fmaf(s, x.w, a.w);
}
__device__ __forceinline__ void vfma(double2& a, double s, const double2& x) {
  a.x = fma(s, x.x, a.x); a.y = fma(s, x.y, a.y);
}
__device__ __forceinline__ void vshfl_add(float4& a, int o) {
  a.x += __shfl_xor_sync(0xffffffffu, a.x, o); a.y += __shfl_xor_sync(0xffffffffu, a.y, o);
  a.z += __shfl_xor_sync(0xffffffffu, a.z, o); a.w += __shfl_xor_sync(0xffffffffu, a.w, o);
}
__device__ __forceinline__ void vshfl_add(double2& a, int o) {
  a.x += __shfl_xor_sync(0xffffffffu, a.x, o); a.y += __shfl_xor_sync(0xffffffffu, a.y, o);
}
__device__ __forceinline__ float4 vaxpy_out(float d, const float4& x, const float4& a) {
  return make_float4(fmaf(d, x.x, -a.x), fmaf(d, x.y, -a.y), fmaf(d, x.z, -a.z), fmaf(d, x.w, -a.w));
}
__device__ __forceinline__ double2 vaxpy_out(double d, const double2& x, const double2& a) {
  return make_double2(fma(d, x.x, -a.x), fma(d, x.y, -a.y));
}
__device__ __forceinline__ float vget(const float4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}
__device__ __forceinline__ double vget(const double2& v, int i) { return i == 0 ? v.x : v.y; }

// Vectorised path: ldx, ldy multiples of the vector width, pointers aligned.
// GS = lanes per neighbour group (power of two), chunks = vectors per row panel.
template <typename T, int GS>
__global__ void __launch_bounds__(256)
spmm_vec(int32_t r0, int32_t r1, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
         const T* __restrict__ cv, const T* __restrict__ deg, const T* __restrict__ x,
         int64_t ldx, int c0, int ncols, T* __restrict__ y, int64_t ldy, int64_t xoff) {
  using V = typename Vec<T>::type;
  constexpr int VN = Vec<T>::N;
  constexpr int NG = 32 / GS;
  const int lane = threadIdx.x & 31;
  const int g = lane / GS, gl = lane % GS;
  const int32_t row = r0 + (int32_t)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (row >= r1) return;
  const int nvec = (ncols + VN - 1) / VN;
  const int32_t e0 = rp[row], e1 = rp[row + 1];
  for (int vbase = 0; vbase < nvec; vbase += GS) {
    const int v = vbase + gl;
    const bool act = v < nvec;
    const int64_t coff = c0 + (int64_t)v * VN;
    V acc = vzero<V>();
    for (int32_t eb = e0; eb < e1; eb += 32) {
      const int32_t my = eb + lane;
      int32_t cj = 0;
      T wv = T(0);
      if (my < e1) {
        cj = __ldg(ci + my);
        wv = __ldg(cv + my);
      }
      const int cnt = min(32, e1 - eb);
#pragma unroll 4
      for (int kk = 0; kk < cnt; kk += NG) {  // warp-uniform trip count
        const int k = kk + g;
        const int srcl = k < cnt ? k : 0;
        const int32_t j = __shfl_sync(0xffffffffu, cj, srcl);
        const T w = __shfl_sync(0xffffffffu, wv, srcl);
        if (act && k < cnt) {
          const V xv = __ldg(reinterpret_cast<const V*>(x + (int64_t)j * ldx + coff));
          vfma(acc, w, xv);
        }
      }
      // keep the warp converged for the shuffles of the next batch
      __syncwarp();
    }
#pragma unroll
    for (int o = GS; o < 32; o <<= 1) vshfl_add(acc, o);
    if (g == 0 && act) {
      const V xi = *reinterpret_cast<const V*>(x + (xoff + row) * ldx + coff);
      const T d = deg[row];
      V out = vaxpy_out(d, xi, acc);
      T* yp = y + (int64_t)row * ldy + coff;
      if (coff - c0 + VN <= ncols) {
        *reinterpret_cast<V*>(yp) = out;
      } else {
        for (int q = 0; q < VN && coff - c0 + q < ncols; ++q) yp[q] = vget(out, q);
      }
    }
  }
}

// Batched variant of spmm_vec: each lane gathers U neighbour vectors into
// registers before the FMAs, so U independent L2 loads are in flight per lane
// (the gather is latency-bound: X rows come from L2 in random order). The FMA
// order per (lane, vector) is the same as spmm_vec's.
template <typename T, int GS, int U, int MINB>
__global__ void __launch_bounds__(256, MINB)
spmm_vb(int32_t r0, int32_t r1, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
        const T* __restrict__ cv, const T* __restrict__ deg, const T* __restrict__ x,
        int64_t ldx, int c0, int ncols, T* __restrict__ y, int64_t ldy, int64_t xoff) {
  using V = typename Vec<T>::type;
  constexpr int VN = Vec<T>::N;
  constexpr int NG = 32 / GS;
  const int lane = threadIdx.x & 31;
  const int g = lane / GS, gl = lane % GS;
  const int32_t row = r0 + (int32_t)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (row >= r1) return;
  const int nvec = (ncols + VN - 1) / VN;
  const int32_t e0 = rp[row], e1 = rp[row + 1];
  for (int vbase = 0; vbase < nvec; vbase += GS) {
    const int v = vbase + gl;
    const bool act = v < nvec;
    const int64_t coff = c0 + (int64_t)v * VN;
    const T* xb = x + coff;
    V acc = vzero<V>();
    for (int32_t eb = e0; eb < e1; eb += 32) {
      const int32_t my = eb + lane;
      int32_t cj = 0;
      T wv = T(0);
      if (my < e1) {
        cj = __ldg(ci + my);
        wv = __ldg(cv + my);
      }
      const int cnt = min(32, e1 - eb);
      for (int kk = 0; kk < cnt; kk += NG * U) {  // warp-uniform trip count
        V xv[U];
        T ww[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int k = kk + u * NG + g;
          const int srcl = k < cnt ? k : 0;
          const int32_t j = __shfl_sync(0xffffffffu, cj, srcl);
          const T w = __shfl_sync(0xffffffffu, wv, srcl);
          const bool ok = act && k < cnt;
          ww[u] = ok ? w : T(0);
          xv[u] = ok ? __ldg(reinterpret_cast<const V*>(xb + (int64_t)j * ldx)) : vzero<V>();
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (kk + u * NG + g < cnt) vfma(acc, ww[u], xv[u]);
      }
      __syncwarp();
    }
#pragma unroll
    for (int o = GS; o < 32; o <<= 1) vshfl_add(acc, o);
    if (g == 0 && act) {
      const V xi = *reinterpret_cast<const V*>(x + (xoff + row) * ldx + coff);
      const T d = deg[row];
      V out = vaxpy_out(d, xi, acc);
      T* yp = y + (int64_t)row * ldy + coff;
      if (coff - c0 + VN <= ncols) {
        *reinterpret_cast<V*>(yp) = out;
      } else {
        for (int q = 0; q < VN && coff - c0 + q < ncols; ++q) yp[q] = vget(out, q);
      }
    }
  }
}

// Scalar fallback for unaligned / odd strides.
template <typename T>
__global__ void __launch_bounds__(256)
spmm_scalar(int32_t r0, int32_t r1, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
            const T* __restrict__ cv, const T* __restrict__ deg, const T* __restrict__ x,
            int64_t ldx, int ncols, T* __restrict__ y, int64_t ldy, int64_t xoff) {
  const int lane = threadIdx.x & 31;
  const int32_t row = r0 + (int32_t)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (row >= r1) return;
  const int32_t e0 = rp[row], e1 = rp[row + 1];
  for (int c = lane; c < ((ncols + 31) / 32) * 32; c += 32) {
    T acc = T(0);
    for (int32_t eb = e0; eb < e1; eb += 32) {
      const int32_t my = eb + lane;
      int32_t cj = 0;
      T wv = T(0);
      if (my < e1) { cj = ci[my]; wv = cv[my]; }
      const int cnt = min(32, e1 - eb);
      for (int k = 0; k < cnt; ++k) {
        const int32_t j = __shfl_sync(0xffffffffu, cj, k);
        const T w = __shfl_sync(0xffffffffu, wv, k);
        if (c < ncols) acc += w * x[(int64_t)j * ldx + c];
      }
    }
    if (c < ncols) y[(int64_t)row * ldy + c] = deg[row] * x[(xoff + row) * ldx + c] - acc;
  }
}

template <typename T>
int launch_spmm(int32_t r0, int32_t r1, const int32_t* rp, const int32_t* ci, const T* cv,
                const T* deg, const T* x, int64_t ldx, int ncols, T* y, int64_t ldy,
                cudaStream_t st, int64_t xoff, int64_t x_rows) {
  constexpr int VN = Vec<T>::N;
  const int64_t rows = (int64_t)r1 - r0;
  if (rows <= 0 || ncols <= 0) return SPB_OK;
  const int threads = 256;
  const int64_t blocks = ceil_div(rows * 32, threads);
  const bool aligned = (ldx % VN == 0) && (ldy % VN == 0) &&
                       ((uintptr_t)x % (VN * sizeof(T)) == 0) &&
                       ((uintptr_t)y % (VN * sizeof(T)) == 0);
  if (!aligned) {
    spmm_scalar<T><<<blocks, threads, 0, st>>>(r0, r1, rp, ci, cv, deg, x, ldx, ncols, y, ldy, xoff);
    SPB_LAUNCH_CHECK();
    return SPB_OK;
  }
  // Full-width rows: each gathered neighbour row is one contiguous run (432 B at
  // C3) and the CSR is read once. Measured and rejected (round 2, C3 R block inside
  // the solver's 336-float rows, 1.538 ms full width): L2-sized column panels, 56 /
  // 36 / 28 columns, 1.77 / 2.38 / 2.81 ms (with evict-last hints on X); L2
  // eviction-priority hints on full rows (fractional evict_last on the gathered X,
  // evict_first on the CSR and Y), 1.53-1.70 ms. ncu at C3: 6.49 GB of DRAM reads
  // per launch (L2 hit rate 26 %) at 4.2 TB/s -- the gathers miss a 216 MB X block.
  // More loads or warps in flight do not raise it (C3 / C4 ms: U = 2 gathers per lane,
  // 8 CTAs of 4 warps per SM 1.55 / 13.4; U = 4 1.56 / 12.8; U = 2 at 16 CTAs 1.88 /
  // 16.4; U = 4 at 12 CTAs 1.87 / 15.5; U = 8 4.36 / 33.6): ~4.3 TB/s is what random
  // 448-byte row gathers sustain here; a contiguous X (ld = l instead of the solver's
  // 3 lp) gains 4 %.
  (void)x_rows;
  {
    const int c0 = 0, pc = ncols;
    const int nvec = (pc + VN - 1) / VN;
    // rows of more than 8 vectors: spmm_vb (kU gathers in flight per lane, 128-thread
    // blocks so short rows free their slots early; round 1 with U = 2: -7 % at C2, -9 %
    // at C3 against spmm_vec in the natural order)
    if (nvec > 8) {
      // one gather in flight per lane (U = 1): with the locality order the gathers hit
      // L2 (69 % at C3) and U = 2 / 4 measured slower (C3 apply 0.94 / 1.02 / 1.19 ms,
      // C4 7.57 / 8.17 / 9.26 ms); 128-thread blocks, 8 per SM (64-thread blocks 0.97,
      // 4 per SM 1.08, 12 per SM 0.99 ms at C3; tools/bench_spmm_order.py)
      constexpr int kU = 1, kMinB = 8, kBlock = 128;
      auto kf = nvec <= 16 ? spmm_vb<T, 16, kU, kMinB> : spmm_vb<T, 32, kU, kMinB>;
      const int64_t vblocks = ceil_div(rows * 32, kBlock);
      kf<<<vblocks, kBlock, 0, st>>>(r0, r1, rp, ci, cv, deg, x, ldx, c0, pc, y, ldy, xoff);
      SPB_LAUNCH_CHECK();
      return SPB_OK;
    }
    if (nvec <= 1)
      spmm_vec<T, 1><<<blocks, threads, 0, st>>>(r0, r1, rp, ci, cv, deg, x, ldx, c0, pc, y, ldy, xoff);
    else if (nvec <= 2)
      spmm_vec<T, 2><<<blocks, threads, 0, st>>>(r0, r1, rp, ci, cv, deg, x, ldx, c0, pc, y, ldy, xoff);
    else if (nvec <= 4)
      spmm_vec<T, 4><<<blocks, threads, 0, st>>>(r0, r1, rp, ci, cv, deg, x, ldx, c0, pc, y, ldy, xoff);
    else if (nvec <= 8)
      spmm_vec<T, 8><<<blocks, threads, 0, st>>>(r0, r1, rp, ci, cv, deg, x, ldx, c0, pc, y, ldy, xoff);
    else if (nvec <= 16)
      spmm_vec<T, 16><<<blocks, threads, 0, st>>>(r0, r1, rp, ci, cv, deg, x, ldx, c0, pc, y, ldy, xoff);
    else
      spmm_vec<T, 32><<<blocks, threads, 0, st>>>(r0, r1, rp, ci, cv, deg, x, ldx, c0, pc, y, ldy, xoff);
    SPB_LAUNCH_CHECK();
  }
  return SPB_OK;
}

}  // namespace

int laplacian_spmm(int dtype, int32_t r0, int32_t r1, const int32_t* rp, const int32_t* ci,
                   const void* cv, const void* deg, const void* x, int64_t ldx, int ncols,
                   void* y, int64_t ldy, cudaStream_t st, int64_t xoff, int64_t x_rows) {
  if (dtype == SPB_F32)
    return launch_spmm<float>(r0, r1, rp, ci, (const float*)cv, (const float*)deg,
                              (const float*)x, ldx, ncols, (float*)y, ldy, st, xoff, x_rows);
  return launch_spmm<double>(r0, r1, rp, ci, (const double*)cv, (const double*)deg,
                             (const double*)x, ldx, ncols, (double*)y, ldy, st, xoff, x_rows);
}

}  // namespace spb

extern "C" int spb_laplacian_spmm(int dtype, int32_t row_begin, int32_t row_end,
                                  const int32_t* row_ptr, const int32_t* col, const void* val,
                                  const void* deg, const void* x, int64_t ldx, int32_t ncols,
                                  void* y, int64_t ldy, void* stream) {
  if (dtype != SPB_F32 && dtype != SPB_F64) {
    spb::set_error("unknown dtype %d", dtype);
    return SPB_ERR_DOMAIN;
  }
  if (row_begin < 0 || row_end < row_begin || ncols < 0 || ldx < ncols || ldy < ncols) {
    spb::set_error("spmm shape contract violated");
    return SPB_ERR_CONTRACT;
  }
  return spb::laplacian_spmm(dtype, row_begin, row_end, row_ptr, col, val, deg, x, ldx, ncols, y,
                             ldy, (cudaStream_t)stream, 0, 0);
}
