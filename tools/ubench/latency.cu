// Latency microbenchmarks for the single-CTA / cluster kernels' building blocks.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat latency.cu && /tmp/lat
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_sync(int iters, long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}

__global__ void k_ddiv(int iters, double x, long long* out, double* sink) {
  double a = x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = 1.0 / (a + 1.0);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / iters; sink[0] = a; }
}

__global__ void k_drcp(int iters, double x, long long* out, double* sink) {
  double a = x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = __drcp_rn(a + 1.0);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / iters; sink[0] = a; }
}

__global__ void k_dsqrt(int iters, double x, long long* out, double* sink) {
  double a = x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = sqrt(a + 1.0);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / iters; sink[0] = a; }
}

__global__ void k_smem_chain(int iters, long long* out) {
  __shared__ double s[1024];
  s[threadIdx.x] = threadIdx.x;
  __syncthreads();
  int idx = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double v = s[idx];
    s[idx] = v * 1.0000001 + 1.0;
    idx = (idx + 33) & 1023;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}

__global__ void k_cluster(int iters, long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  long long t1 = clock64();
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  if (threadIdx.x == 0 && r == 0) out[0] = (t1 - t0) / iters;
}


__device__ __forceinline__ void tri_index(int t, int* ti, int* tq) {
  int r = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
  while ((r + 1) * (r + 2) / 2 <= t) ++r;
  while (r * (r + 1) / 2 > t) --r;
  *ti = r;
  *tq = t - r * (r + 1) / 2;
}

// The Cholesky P1 column step (chol_wsync): pivot read, reciprocal, one
// trailing-triangle element per thread, CTA barrier. variant 0: as written;
// 1: tri_index hoisted; 2: hoisted + no division (reciprocal precomputed)
__global__ void k_p1(int reps, int variant, long long* out) {
  extern __shared__ double A[];
  __shared__ double dinv[32];
  const int ld = 147, tid = threadIdx.x;
  for (int x = tid; x < 147 * 147; x += blockDim.x) A[x] = (x % 148 == 0) ? 100.0 : 0.01;
  __syncthreads();
  int hti, htq;
  tri_index(tid, &hti, &htq);
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    const int kb = 32 * (r % 4);
    for (int c = 0; c < 32; ++c) {
      const double dc = A[(kb + c) * ld + kb + c];
      const double rc = variant == 2 ? 0.01 : 1.0 / dc;
      const int rem = 31 - c;
      if (tid < rem * (rem + 1) / 2) {
        int ti, tq;
        if (variant == 0) tri_index(tid, &ti, &tq);
        else { ti = hti; tq = htq; }
        const int i = kb + c + 1 + ti, q = kb + c + 1 + tq;
        A[i * ld + q] = fma(-A[i * ld + kb + c] * rc, A[q * ld + kb + c], A[i * ld + q]);
      }
      if (tid == 0) dinv[c] = rc;
      __syncthreads();
    }
  }
  long long t1 = clock64();
  if (tid == 0) out[0] = (t1 - t0) / (reps * 32);
}


__global__ void k_dfma(int iters, double x, long long* out, double* sink) {
  double a = x, b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / iters; sink[0] = a; }
}

__global__ void k_dfma_tp(int iters, double x, long long* out, double* sink) {
  double a0 = x, a1 = x + 1, a2 = x + 2, a3 = x + 3, a4 = x + 4, a5 = x + 5, a6 = x + 6, a7 = x + 7;
  const double b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) * 100 / iters; }
  sink[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void k_shfl(int iters, double x, long long* out, double* sink) {
  double a = x + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a += __shfl_xor_sync(0xffffffffu, a, 1 + (i & 15));
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / iters; sink[0] = a; }
}

int main() {
  long long* d;
  double* sink;
  cudaMalloc(&d, 64);
  cudaMalloc(&sink, 64);
  long long h;
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock rate attr %d kHz\n", clk);
  for (int nt : {64, 256, 512, 1024}) {
    k_sync<<<1, nt>>>(10000, d);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("__syncthreads %4d threads: %lld cycles\n", nt, h);
  }
  k_ddiv<<<1, 32>>>(10000, 0.5, d, sink); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); printf("dependent 1/x (DDIV): %lld cycles\n", h);
  k_drcp<<<1, 32>>>(10000, 0.5, d, sink); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); printf("dependent __drcp_rn: %lld cycles\n", h);
  k_dsqrt<<<1, 32>>>(10000, 0.5, d, sink); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); printf("dependent sqrt: %lld cycles\n", h);
  k_dfma<<<1, 32>>>(10000, 0.5, d, sink); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); printf("dependent DFMA: %lld cycles\n", h);
  k_shfl<<<1, 32>>>(10000, 0.5, d, sink); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); printf("dependent f64 shfl+DADD: %lld cycles\n", h);
  for (int nt : {32, 128, 256, 512, 1024}) {
    k_dfma_tp<<<1, nt>>>(10000, 0.5, d, sink); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("8 indep DFMA per iter, %4d thr: %.2f cycles/iter\n", nt, h / 100.0);
  }
  for (int nt : {32, 1024}) {
    k_smem_chain<<<1, nt>>>(10000, d); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("smem load->fma->store chain (%d thr): %lld cycles\n", nt, h);
  }
  cudaFuncSetAttribute(k_p1, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int v : {0, 1, 2}) {
    for (int nt : {512, 1024}) {
      k_p1<<<1, nt, 147 * 147 * 8>>>(100, v, d);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("chol P1 column step variant %d, %d thr: %lld cycles (%s)\n", v, nt, h, cudaGetErrorString(e));
    }
  }
  for (int C : {2, 4, 8, 16}) {
    cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int nt : {256, 512}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(C);
      cfg.blockDim = dim3(nt);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      cudaError_t e = cudaLaunchKernelEx(&cfg, k_cluster, 10000, d);
      cudaDeviceSynchronize();
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("cluster barrier C=%2d %d thr: %lld cycles (%s)\n", C, nt, h, cudaGetErrorString(e));
    }
  }
  return 0;
}
