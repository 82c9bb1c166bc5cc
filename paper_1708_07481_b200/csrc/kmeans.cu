// (e) Optional k-means assignment on the spectral embedding (north star (e);
// SURVEY.md §8(f) row 3). The reference has no k-means (spectral.py:5),
// so this mode is parity-unpinned; the QRCP assignment stays the default.
//
// Lloyd iterations from given initial centroids (the QRCP seed rows by default):
//   assign : argmin_c ||x_i - mu_c||^2 = argmin_c (||mu_c||^2 - 2 x_i . mu_c)
//            float32 embeddings (k <= 192, no row normalisation): the distance GEMM
//            X mu' on the tcgen05 tensor cores (3xTF32, TMA-fed; update_tc.cu)
//            with the argmin fused into its epilogue -- X is read once per Lloyd
//            step and no n x k distance matrix is written; otherwise a thread per
//            row with the centroids and their norms in shared memory; changes are
//            counted for the stop test;
//   update : per-cluster sums as a segmented reduction (float64 atomics into
//            k x d accumulators, then mu = sum / count; empty clusters keep
//            their previous centroid).
#include "dense.cuh"

namespace spb {
namespace {

constexpr int KT = 256;

// coefficients of the distance GEMM: C[t][j] = mu[j][t] (d x k, float64)
__global__ void km_coeffs(const float* __restrict__ mu, int k, int d, double* __restrict__ c) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k * d; e += gridDim.x * blockDim.x) {
    const int t = e / k, j = e % k;
    c[e] = (double)mu[(size_t)j * d + t];
  }
}

template <typename T>
__global__ void __launch_bounds__(KT)
km_assign(const T* __restrict__ X, int64_t ldx, int n, int d, int k, const float* __restrict__ mu,
          const float* __restrict__ mu2, int* __restrict__ labels, int normalize,
          unsigned long long* __restrict__ changed) {
  extern __shared__ float sm[];  // mu (k x d) then mu2 (k)
  float* smu = sm;
  float* smu2 = sm + (size_t)k * d;
  for (int x = threadIdx.x; x < k * d; x += KT) smu[x] = mu[x];
  for (int x = threadIdx.x; x < k; x += KT) smu2[x] = mu2[x];
  __syncthreads();
  const int i = blockIdx.x * KT + threadIdx.x;
  int ch = 0;
  if (i < n) {
    float xr[64];
    float best = INFINITY;
    int lab = 0;
    float scale = 1.0f;
    if (normalize) {
      double s = 0.0;
      for (int t = 0; t < d; ++t) {
        const double v = (double)X[(int64_t)i * ldx + t];
        s += v * v;
      }
      scale = s > 0.0 ? (float)(1.0 / sqrt(s)) : 0.0f;
    }
    for (int c = 0; c < k; ++c) {
      float dot = 0.0f;
      for (int t0 = 0; t0 < d; t0 += 64) {
        const int tn = min(64, d - t0);
        if (c == 0 || d > 64) {
#pragma unroll 8
          for (int t = 0; t < tn; ++t) xr[t] = (float)X[(int64_t)i * ldx + t0 + t] * scale;
        }
        const float* m = smu + (size_t)c * d + t0;
#pragma unroll 8
        for (int t = 0; t < tn; ++t) dot = fmaf(xr[t], m[t], dot);
      }
      const float dist = smu2[c] - 2.0f * dot;
      if (dist < best) {  // strict: lowest cluster index on ties
        best = dist;
        lab = c;
      }
    }
    ch = labels[i] != lab;
    labels[i] = lab;
  }
  const unsigned m = __ballot_sync(0xffffffffu, ch);
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(changed, (unsigned long long)__popc(m));
}

template <typename T>
__global__ void km_accumulate(const T* __restrict__ X, int64_t ldx, int n, int d,
                              const int* __restrict__ labels, int normalize,
                              double* __restrict__ sums, unsigned long long* __restrict__ counts) {
  // warp per row: lanes over dimensions
  const int lane = threadIdx.x & 31;
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (row >= n) return;
  const int c = labels[row];
  double scale = 1.0;
  if (normalize) {
    double s = 0.0;
    for (int t = lane; t < d; t += 32) {
      const double v = (double)X[row * ldx + t];
      s += v * v;
    }
    s = warp_sum(s);
    scale = s > 0.0 ? 1.0 / sqrt(s) : 0.0;
  }
  for (int t = lane; t < d; t += 32) atomicAdd(&sums[(size_t)c * d + t], (double)X[row * ldx + t] * scale);
  if (lane == 0) atomicAdd(&counts[c], 1ull);
}

__global__ void km_finalize(const double* __restrict__ sums, const unsigned long long* __restrict__ counts,
                            int k, int d, float* __restrict__ mu, float* __restrict__ mu2) {
  const int c = blockIdx.x;
  __shared__ double red[32];
  double s2 = 0.0;
  const unsigned long long cnt = counts[c];
  for (int t = threadIdx.x; t < d; t += blockDim.x) {
    float v = mu[(size_t)c * d + t];
    if (cnt > 0) v = (float)(sums[(size_t)c * d + t] / (double)cnt);
    mu[(size_t)c * d + t] = v;
    s2 += (double)v * v;
  }
  s2 = warp_sum(s2);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s2;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    mu2[c] = (float)t;
  }
}

template <typename T>
__global__ void km_init(const T* __restrict__ X, int64_t ldx, int d, int k, const int* __restrict__ seeds,
                        int normalize, float* __restrict__ mu) {
  const int c = blockIdx.x;
  const int64_t r = seeds[c];
  __shared__ double sc;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int t = 0; t < d; ++t) {
      const double v = (double)X[r * ldx + t];
      s += v * v;
    }
    sc = (normalize && s > 0.0) ? 1.0 / sqrt(s) : 1.0;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < d; t += blockDim.x) mu[(size_t)c * d + t] = (float)((double)X[r * ldx + t] * sc);
}

template <typename T>
int kmeans_t(const void* xv, int64_t ldx, int n, int d, int k, const int* seeds, int max_iter,
             int normalize, int* labels, float* mu, float* mu2, double* sums,
             unsigned long long* counts, unsigned long long* changed, double* coef,
             float* cstage, size_t cstage_cap, int* iters_out, cudaStream_t st) {
  const T* X = (const T*)xv;
  km_init<T><<<k, 128, 0, st>>>(X, ldx, d, k, seeds, normalize, mu);
  SPB_CUDA(cudaMemsetAsync(sums, 0, sizeof(double) * (size_t)k * d, st));
  SPB_CUDA(cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * k, st));
  km_finalize<<<k, 128, 0, st>>>(sums, counts, k, d, mu, mu2);  // norms of the initial centroids
  SPB_CUDA(cudaMemsetAsync(labels, 0xff, sizeof(int) * n, st));
  const size_t smem = sizeof(float) * ((size_t)k * d + k);
  // the tensor-core path reads X through a TMA map: 16-byte aligned rows; an
  // unaligned float32 embedding is copied once into padded rows for the Lloyd loop
  const float* Xtc = nullptr;
  int64_t ldtc = ldx;
  float* xpad = nullptr;
  if (sizeof(T) == 4 && !normalize && coef) {
    if ((reinterpret_cast<uintptr_t>(X) & 15) == 0 && (ldx & 3) == 0) {
      Xtc = (const float*)X;
    } else {
      ldtc = round_up(d, 4);
      if (cudaMallocAsync((void**)&xpad, sizeof(float) * (size_t)n * ldtc, st) == cudaSuccess) {
        SPB_CUDA(cudaMemcpy2DAsync(xpad, sizeof(float) * ldtc, X, sizeof(T) * ldx, sizeof(float) * d, n,
                                   cudaMemcpyDeviceToDevice, st));
        Xtc = xpad;
      } else {
        cudaGetLastError();
        xpad = nullptr;
      }
    }
  }
  SPB_CUDA(cudaFuncSetAttribute(km_assign<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)std::max<size_t>(smem, 48 * 1024)));
  int it = 0;
  for (; it < max_iter; ++it) {
    SPB_CUDA(cudaMemsetAsync(changed, 0, sizeof(unsigned long long), st));
    bool tc = false;
    if (sizeof(T) == 4 && !normalize && coef && cstage && Xtc) {
      km_coeffs<<<(int)std::min<int64_t>(ceil_div((int64_t)k * d, 256), 256), 256, 0, st>>>(mu, k, d,
                                                                                          coef);
      UpdParams p{};
      p.nseg = 1;
      p.q = k;
      p.seg[0] = {Xtc, ldtc, coef, k, nullptr, 0, 1.0, d, 1};
      p.cstage = cstage;
      p.cstage_cap = cstage_cap;
      p.argmin_bias = mu2;
      p.argmin_labels = labels;
      p.argmin_changed = changed;
      tc = update_tc(p, n, st);
    }
    if (!tc)
      km_assign<T><<<(int)ceil_div(n, KT), KT, smem, st>>>(X, ldx, n, d, k, mu, mu2, labels,
                                                           normalize, changed);
    SPB_LAUNCH_CHECK();
    unsigned long long h = 0;
    SPB_CUDA(cudaMemcpyAsync(&h, changed, sizeof(h), cudaMemcpyDeviceToHost, st));
    SPB_CUDA(cudaStreamSynchronize(st));
    if (h == 0) break;
    SPB_CUDA(cudaMemsetAsync(sums, 0, sizeof(double) * (size_t)k * d, st));
    SPB_CUDA(cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * k, st));
    // (a shared-memory privatised float64 accumulator measured slower at C4,
    // 2M x 160: 5.6 against 3.8 ms per Lloyd step -- shared float64 atomics)
    km_accumulate<T><<<(int)ceil_div((int64_t)n * 32, 256), 256, 0, st>>>(X, ldx, n, d, labels,
                                                                         normalize, sums, counts);
    km_finalize<<<k, 128, 0, st>>>(sums, counts, k, d, mu, mu2);
    SPB_LAUNCH_CHECK();
  }
  *iters_out = it;
  if (xpad) SPB_CUDA(cudaFreeAsync(xpad, st));
  return SPB_OK;
}

}  // namespace
}  // namespace spb

using namespace spb;

extern "C" size_t spb_kmeans_workspace(int32_t k, int32_t d) {
  Arena a;
  a.dry = true;
  a.take<double>((size_t)k * d);            // sums
  a.take<float>(k);                         // mu2
  a.take<unsigned long long>(k);            // counts
  a.take<unsigned long long>(1);            // changed
  a.take<double>((size_t)k * d);            // distance-GEMM coefficients
  a.take<float>(update_tc_cstage_floats(d, 1, k));  // their TF32 split staging
  return a.used + 1024;
}

extern "C" int spb_kmeans(int dtype, const void* x, int64_t ldx, int32_t n, int32_t d, int32_t k,
                          const int32_t* seeds, int32_t max_iter, int32_t normalize_rows, void* ws,
                          size_t ws_bytes, int32_t* labels_out, float* centroids_out,
                          int32_t* iterations_out, void* stream) {
  if (dtype != SPB_F32 && dtype != SPB_F64) {
    set_error("unknown dtype %d", dtype);
    return SPB_ERR_DOMAIN;
  }
  if (k < 1 || n < k || d < 1 || ldx < d) {
    set_error("kmeans needs n >= k >= 1 and ldx >= d >= 1");
    return SPB_ERR_CONTRACT;
  }
  if ((size_t)k * d * sizeof(float) > 200 * 1024) {
    set_error("kmeans centroids (k*d=%d) exceed shared memory", k * d);
    return SPB_ERR_CONTRACT;
  }
  Arena a;
  a.base = (char*)ws;
  a.cap = ws_bytes;
  double* sums = a.take<double>((size_t)k * d);
  float* mu2 = a.take<float>(k);
  unsigned long long* counts = a.take<unsigned long long>(k);
  unsigned long long* changed = a.take<unsigned long long>(1);
  double* coef = a.take<double>((size_t)k * d);
  const size_t cstage_cap = update_tc_cstage_floats(d, 1, k);
  float* cstage = a.take<float>(cstage_cap);
  if (a.used > ws_bytes) {
    set_error("kmeans workspace too small");
    return SPB_ERR_WORKSPACE;
  }
  int it = 0;
  cudaStream_t st = (cudaStream_t)stream;
  int s = dtype == SPB_F32
              ? kmeans_t<float>(x, ldx, n, d, k, seeds, max_iter, normalize_rows, labels_out,
                                centroids_out, mu2, sums, counts, changed, coef, cstage,
                                cstage_cap, &it, st)
              : kmeans_t<double>(x, ldx, n, d, k, seeds, max_iter, normalize_rows, labels_out,
                                 centroids_out, mu2, sums, counts, changed, nullptr, nullptr, 0,
                                 &it, st);
  *iterations_out = it;
  return s;
}

// ---------------------------------------------------------------------------
// (f.4) Contingency table on the device (metrics.py:65-75): counts[t * kf + f]
// of (truth, found) label pairs, a shared-memory histogram per CTA when the
// table fits (integer atomics: order-independent, so deterministic), global
// 64-bit atomics otherwise.
namespace spb {
namespace {
__global__ void contingency_kernel(const int32_t* __restrict__ t, const int32_t* __restrict__ f,
                                   int64_t n, int kt, int kf, unsigned long long* __restrict__ counts,
                                   int use_smem, int* __restrict__ bad) {
  extern __shared__ unsigned int hist[];
  const int cells = kt * kf;
  if (use_smem) {
    for (int x = threadIdx.x; x < cells; x += blockDim.x) hist[x] = 0u;
    __syncthreads();
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int a = t[i], b = f[i];
    if (a < 0 || a >= kt || b < 0 || b >= kf) {
      atomicOr(bad, 1);
      continue;
    }
    if (use_smem) atomicAdd(&hist[a * kf + b], 1u);
    else atomicAdd(&counts[(int64_t)a * kf + b], 1ull);
  }
  if (use_smem) {
    __syncthreads();
    for (int x = threadIdx.x; x < cells; x += blockDim.x)
      if (hist[x]) atomicAdd(&counts[x], (unsigned long long)hist[x]);
  }
}
}  // namespace
}  // namespace spb

extern "C" int spb_contingency(const int32_t* truth, const int32_t* found, int64_t n, int32_t kt,
                               int32_t kf, int64_t* counts, void* ws, size_t ws_bytes,
                               void* stream) {
  if (n < 0 || kt < 1 || kf < 1) {
    set_error("contingency needs n >= 0 and label ranges >= 1");
    return SPB_ERR_CONTRACT;
  }
  if (ws_bytes < sizeof(int) || !ws) {
    set_error("contingency workspace too small");
    return SPB_ERR_WORKSPACE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  int* bad = (int*)ws;
  SPB_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * (size_t)kt * kf, st));
  SPB_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
  const size_t smem = sizeof(unsigned int) * (size_t)kt * kf;
  const int use_smem = smem <= 48 * 1024;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(std::max<int64_t>(n, 1), 1024),
                                                                 4 * num_sms()));
  contingency_kernel<<<blocks, 256, use_smem ? smem : 0, st>>>(
      truth, found, n, kt, kf, (unsigned long long*)counts, use_smem, bad);
  SPB_LAUNCH_CHECK();
  int hb = 0;
  SPB_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  SPB_CUDA(cudaStreamSynchronize(st));
  if (hb) {
    set_error("label outside [0, k)");
    return SPB_ERR_CONTRACT;
  }
  return SPB_OK;
}
