// C-ABI plumbing: error strings, version, casts, block copies, reductions.
#include <cstdarg>
#include <cstring>

#include <mutex>

#include "common.cuh"

namespace spb {

static thread_local char g_err[1024] = {0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

namespace {

template <typename S, typename D>
__global__ void copy_block_k(const S* __restrict__ s, int64_t lds, D* __restrict__ d, int64_t ldd,
                             int64_t rows, int32_t cols) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / cols;
    int32_t c = (int32_t)(i - r * cols);
    d[r * ldd + c] = (D)s[r * lds + c];
  }
}

template <typename S, typename D>
int copy_block_t(const void* s, int64_t lds, void* d, int64_t ldd, int64_t rows, int32_t cols,
                 cudaStream_t st) {
  int64_t total = rows * cols;
  if (total <= 0) return SPB_OK;
  int grid = (int)std::min<int64_t>(ceil_div(total, 256), (int64_t)num_sms() * 8);
  copy_block_k<S, D><<<grid, 256, 0, st>>>((const S*)s, lds, (D*)d, ldd, rows, cols);
  SPB_LAUNCH_CHECK();
  return SPB_OK;
}

__global__ void max_partial(const double* __restrict__ v, int64_t n, double* __restrict__ out) {
  double m = -INFINITY;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, v[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ double sm[32];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = sm[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) r = fmax(r, sm[w]);
    out[blockIdx.x] = r;
  }
}

}  // namespace

int copy_block(int sdt, const void* s, int64_t lds, int ddt, void* d, int64_t ldd, int64_t rows,
               int32_t cols, cudaStream_t st) {
  if (sdt == SPB_F64 && ddt == SPB_F64) return copy_block_t<double, double>(s, lds, d, ldd, rows, cols, st);
  if (sdt == SPB_F64 && ddt == SPB_F32) return copy_block_t<double, float>(s, lds, d, ldd, rows, cols, st);
  if (sdt == SPB_F32 && ddt == SPB_F64) return copy_block_t<float, double>(s, lds, d, ldd, rows, cols, st);
  return copy_block_t<float, float>(s, lds, d, ldd, rows, cols, st);
}

}  // namespace spb

using namespace spb;

extern "C" const char* spb_last_error(void) { return g_err; }

extern "C" int spb_version(void) { return 100; }

extern "C" int spb_device_sm_count(void) { return num_sms(); }

extern "C" int spb_cast(const double* in, int64_t count, int dtype, void* out, void* stream) {
  if (dtype != SPB_F32 && dtype != SPB_F64) {
    set_error("unknown dtype %d", dtype);
    return SPB_ERR_DOMAIN;
  }
  return copy_block(SPB_F64, in, 1, dtype, out, 1, count, 1, (cudaStream_t)stream);
}

extern "C" int spb_copy_block(int src_dtype, const void* src, int64_t lds, int dst_dtype,
                              void* dst, int64_t ldd, int64_t rows, int32_t cols, void* stream) {
  if ((src_dtype != SPB_F32 && src_dtype != SPB_F64) ||
      (dst_dtype != SPB_F32 && dst_dtype != SPB_F64)) {
    set_error("unknown dtype");
    return SPB_ERR_DOMAIN;
  }
  if (lds < cols || ldd < cols || rows < 0) {
    set_error("copy_block shape contract violated");
    return SPB_ERR_CONTRACT;
  }
  return copy_block(src_dtype, src, lds, dst_dtype, dst, ldd, rows, cols, (cudaStream_t)stream);
}

extern "C" int spb_max_f64(const double* v, int64_t count, double* out_host, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (count <= 0) {
    *out_host = -INFINITY;
    return SPB_OK;
  }
  const int blocks = (int)std::min<int64_t>(ceil_div(count, 256), 256);
  // per-device scratch allocated once (a stream-ordered allocation per call
  // occasionally stalled the caller for hundreds of ms while the pool remapped)
  static std::mutex mu;
  static double* scratch[64] = {nullptr};
  int dev = 0;
  SPB_CUDA(cudaGetDevice(&dev));
  double* part = nullptr;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!scratch[dev & 63]) SPB_CUDA(cudaMalloc((void**)&scratch[dev & 63], sizeof(double) * 320));
    part = scratch[dev & 63];
    max_partial<<<blocks, 256, 0, st>>>(v, count, part);
    max_partial<<<1, 256, 0, st>>>(part, blocks, part + blocks);
    SPB_CUDA(cudaMemcpyAsync(out_host, part + blocks, sizeof(double), cudaMemcpyDeviceToHost, st));
    SPB_CUDA(cudaStreamSynchronize(st));
  }
  return SPB_OK;
}
