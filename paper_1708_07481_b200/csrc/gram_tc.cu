// (c) Tall-skinny Gram products on the 5th-generation tensor cores (tcgen05),
// 3xTF32 split, TMA-fed, float64 split-K reduction.
//
//   G[p x q] = U' V,   U: n x p, V: n x q, float32, vertex-major (row stride ld)
//
// This is the Rayleigh-Ritz product [X R P]'[X R P | LX LR LP] of
// lobpcg.py:418 (and the smaller Grams of :228, :366) as one GEMM with
// M = columns of U, N = columns of V, K = n (the vertices).
//
// Per CTA: one 128 x BN output tile over a BK-aligned range of rows (split-K).
// Warp roles (warp-specialised, mbarrier pipeline with KS stages):
//   warp 0  TMA producer: boxes {32 columns x BK rows} of U and V into a staging
//           buffer (vertex-major, as stored in HBM);
//   warps 2-5 splitters: x -> hi = x with the low 13 mantissa bits cleared (exact
//           in TF32), lo = x - hi, written transposed into the K-major canonical
//           (no-swizzle, 8x16B core matrix) operand buffers; fence.proxy.async;
//   warp 1  MMA issuer (one thread): per 8-row K step, three
//           tcgen05.mma.kind::tf32 into one fp32 TMEM accumulator:
//           U_hi'V_lo + U_lo'V_hi + U_hi'V_hi; tcgen05.commit frees the stage;
//   warps 2-5 epilogue: tcgen05.ld 32x32b -> float64 partial tile in global.
// The split-K partials are summed in float64 in a fixed order (sum_splits):
// the fp32 accumulation length is one CTA's row range (n / ksplit rows).
#include <cuda.h>

#include "dense.cuh"

namespace spb {
namespace {

constexpr int TBM = 128;   // UMMA M
constexpr int TBN = 128;   // max UMMA N per tile
constexpr int TBK = 16;    // rows (K) per pipeline stage
constexpr int TKS = 4;     // pipeline stages
constexpr int TBOX = 32;   // columns per TMA box
constexpr int kStageA = TBM * TBK * 4;  // bytes of one A-sized buffer (8 KB)
constexpr int kStageB = TBN * TBK * 4;  // bytes of one B-sized buffer (8 KB)
// stage: [staging A][staging B][A hi][A lo][B hi][B lo]
constexpr int kStageBytes = 3 * (kStageA + kStageB);
constexpr int kSmemBytes = TKS * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// K-major, no swizzle ("interleave") canonical layout: 8 rows x 16 bytes core
// matrices; SBO = byte stride between 8-row groups (M/N), LBO = byte stride
// between the 16-byte K halves of an 8-element (tf32) K step.
__device__ __forceinline__ uint64_t umma_desc_k_interleave(uint32_t saddr, uint32_t lbo,
                                                           uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
  return d;                // layout type 0 = SWIZZLE_NONE
}
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

struct TcJob {
  int q;       // columns of V for this job
  int out_c;   // output column offset
  int ntiles;  // ceil(q / TBN)
};

struct TcParams {
  TcJob job[2];
  int njobs;
  int p;           // columns of U (rows of G)
  int mtiles;
  int tiles;       // mtiles * sum(ntiles)
  int64_t n;       // rows (K)
  int64_t kchunk;  // rows per split (multiple of TBK)
  int ldo;         // partial leading dimension
  int64_t split_stride;
};

__global__ void __launch_bounds__(192, 1)
gram_tc_kernel(const __grid_constant__ CUtensorMap mapU, const __grid_constant__ CUtensorMap mapV0,
               const __grid_constant__ CUtensorMap mapV1, TcParams P, double* __restrict__ part) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)dsm + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(base + TKS * kStageBytes);
  uint64_t* split = full + TKS;
  uint64_t* empty = split + TKS;
  uint64_t* accb = empty + TKS;
  uint32_t* tmem_slot = (uint32_t*)(accb + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // tile decode
  int t = blockIdx.x;
  const int mt = t % P.mtiles;
  t /= P.mtiles;
  int j = 0;
  while (j + 1 < P.njobs && t >= P.job[j].ntiles) {
    t -= P.job[j].ntiles;
    ++j;
  }
  const TcJob jb = P.job[j];
  const int m0 = mt * TBM, n0 = t * TBN;
  const int nvalid = min(TBN, jb.q - n0);
  const int nmma = (nvalid + 31) / 32 * 32;  // UMMA N (multiple of 32 <= 256)
  const int nbox = nmma / TBOX;
  const CUtensorMap* mapV = j == 0 ? &mapV0 : &mapV1;
  const int64_t k0 = (int64_t)blockIdx.y * P.kchunk;
  const int64_t k1 = min(P.n, k0 + P.kchunk);
  const int nk = (int)((k1 - k0 + TBK - 1) / TBK);

  if (threadIdx.x == 0) {
    for (int s = 0; s < TKS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&split[s], 128);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accb, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0 && nk > 0) {
      const uint32_t bytes = (uint32_t)(kStageA + nbox * TBOX * TBK * 4);
      for (int kc = 0; kc < nk; ++kc) {
        const int s = kc % TKS, u = kc / TKS;
        if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
        uint8_t* st = base + s * kStageBytes;
        mbar_expect_tx(&full[s], bytes);
        const int row = (int)(k0 + (int64_t)kc * TBK);
#pragma unroll
        for (int g = 0; g < TBM / TBOX; ++g)
          tma_load_2d(st + g * TBOX * TBK * 4, &mapU, &full[s], m0 + g * TBOX, row);
        for (int g = 0; g < nbox; ++g)
          tma_load_2d(st + kStageA + g * TBOX * TBK * 4, mapV, &full[s], n0 + g * TBOX, row);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && nk > 0) {
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) |  // F32 acc, TF32 A/B, K-major
                             ((uint32_t)(nmma >> 3) << 17) | ((uint32_t)(TBM >> 4) << 24);
      const uint32_t sbo = 128;                   // 8 rows x 16 B core matrix
      const uint32_t lbo_a = (TBM / 8) * 128;     // between 4-element K chunks
      const uint32_t lbo_b = (TBN / 8) * 128;
      for (int kc = 0; kc < nk; ++kc) {
        const int s = kc % TKS, u = kc / TKS;
        mbar_wait(&split[s], u & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        uint8_t* st = base + s * kStageBytes + kStageA + kStageB;
        const uint32_t ahi = smem_u32(st), alo = smem_u32(st + kStageA);
        const uint32_t bhi = smem_u32(st + 2 * kStageA), blo = smem_u32(st + 2 * kStageA + kStageB);
#pragma unroll
        for (int kk = 0; kk < TBK / 8; ++kk) {
          const uint64_t dah = umma_desc_k_interleave(ahi + kk * 2 * lbo_a, lbo_a, sbo);
          const uint64_t dal = umma_desc_k_interleave(alo + kk * 2 * lbo_a, lbo_a, sbo);
          const uint64_t dbh = umma_desc_k_interleave(bhi + kk * 2 * lbo_b, lbo_b, sbo);
          const uint64_t dbl = umma_desc_k_interleave(blo + kk * 2 * lbo_b, lbo_b, sbo);
          const uint32_t acc0 = (kc | kk) ? 1u : 0u;
          umma_tf32(tmem, dah, dbl, idesc, acc0);  // small terms first
          umma_tf32(tmem, dal, dbh, idesc, 1u);
          umma_tf32(tmem, dah, dbh, idesc, 1u);
        }
        umma_commit(&empty[s]);
      }
      umma_commit(accb);
    }
  } else {
    // warps 2..5: split, then epilogue
    const int st_tid = threadIdx.x - 64;  // 0..127
    // staging (k, c) of box g -> operand row m = 32 g + c, K index k:
    // K-major interleave offset (floats) = (k / 4) * (rows * 4) + (m / 8) * 32 + (m % 8) * 4 + k % 4
    const int total = (TBM + nmma) * TBK;
    for (int kc = 0; kc < nk; ++kc) {
      const int s = kc % TKS, u = kc / TKS;
      mbar_wait(&full[s], u & 1);
      uint8_t* st = base + s * kStageBytes;
      const float* stg = (const float*)st;
      float* ahi = (float*)(st + kStageA + kStageB);
      float* alo = ahi + TBM * TBK;
      float* bhi = alo + TBM * TBK;
      float* blo = bhi + TBN * TBK;
      for (int i = st_tid; i < total; i += 128) {
        const bool isA = i < TBM * TBK;
        const int e = isA ? i : i - TBM * TBK;
        const int g = e / (TBOX * TBK), k = (e / TBOX) % TBK, c = e % TBOX;
        const int mrow = g * TBOX + c;
        const int rows = isA ? TBM : TBN;
        const float x = isA ? stg[e] : stg[TBM * TBK + e];
        const float h = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
        const int off = (k >> 2) * (rows * 4) + (mrow >> 3) * 32 + (mrow & 7) * 4 + (k & 3);
        if (isA) {
          ahi[off] = h;
          alo[off] = x - h;
        } else {
          bhi[off] = h;
          blo[off] = x - h;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&split[s]);
    }
    // epilogue
    if (nk > 0) {
      mbar_wait(accb, 0);
      asm volatile("tcgen05.fence::after_thread_sync;");
    }
    const int quarter = warp & 3;
    const int row = m0 + quarter * 32 + lane;
    double* out = part + (int64_t)blockIdx.y * P.split_stride;
    for (int c0 = 0; c0 < nmma; c0 += 32) {
      uint32_t r[32];
      if (nk > 0) {
        const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, "
            "%10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, "
            "%27, %28, %29, %30, %31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
              "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
              "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
              "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
              "=r"(r[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      } else {
#pragma unroll
        for (int q = 0; q < 32; ++q) r[q] = 0u;
      }
      if (row < P.p) {
        double* orow = out + (int64_t)row * P.ldo + jb.out_c + n0 + c0;
#pragma unroll
        for (int q = 0; q < 32; ++q)
          if (c0 + q < nvalid) orow[q] = (double)__uint_as_float(r[q]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  }
}

__global__ void sum_splits_tc(const double* __restrict__ part, int ksplit, int64_t stride, int rows,
                              int cols, int ldp, double* __restrict__ out, int ldo) {
  const int64_t total = (int64_t)rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / cols), c = (int)(e % cols);
    double s = 0.0;
    for (int k = 0; k < ksplit; ++k) s += part[k * stride + (int64_t)r * ldp + c];
    out[(int64_t)r * ldo + c] = s;
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

int make_map(CUtensorMap* m, const void* ptr, int64_t rows, int cols, int64_t ld) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return SPB_ERR_CUDA;
  }
  if (((uintptr_t)ptr & 15) || ((ld * 4) & 15)) {
    set_error("TMA needs 16-byte aligned base and row pitch");
    return SPB_ERR_CONTRACT;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {TBOX, TBK};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return SPB_ERR_CUDA;
  }
  return SPB_OK;
}

}  // namespace

bool gram_tc_supported() {
  static int ok = -1;
  if (ok < 0) {
    int dev = 0, maj = 0, min_ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&min_, cudaDevAttrComputeCapabilityMinor, dev);
    ok = (maj == 10 && min_ == 0 && encode_fn() != nullptr) ? 1 : 0;
  }
  return ok == 1;
}

size_t gram_tc_partial_doubles(int64_t n, int p, int qtot) {
  const int tiles = (int)ceil_div(p, TBM) * (int)ceil_div(qtot, TBN) + 2;
  int64_t ks = ceil_div(num_sms(), tiles);
  ks = std::max<int64_t>(1, std::min<int64_t>(ks, ceil_div(n, 256)));
  return (size_t)ks * p * qtot;
}

// out[p x (q0 + q1)] (ld ldo) = U' [V0 | V1]; float32 operands.
int gram_tc(const float* U, int64_t ldu, int p, const float* V0, int64_t ldv0, int q0,
            const float* V1, int64_t ldv1, int q1, int64_t n, double* partial, size_t partial_cap,
            double* out, int ldo, cudaStream_t st) {
  if (p <= 0 || q0 <= 0) return SPB_OK;
  static std::atomic<uint64_t> attr{0};
  if (!done_on_device(attr)) {
    SPB_CUDA(cudaFuncSetAttribute(gram_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kSmemBytes));
    mark_on_device(attr);
  }
  CUtensorMap mu, mv0, mv1;
  SPB_TRY(make_map(&mu, U, n, p, ldu));
  SPB_TRY(make_map(&mv0, V0, n, q0, ldv0));
  if (V1 && q1 > 0) SPB_TRY(make_map(&mv1, V1, n, q1, ldv1));
  else mv1 = mv0;
  TcParams P{};
  P.njobs = (V1 && q1 > 0) ? 2 : 1;
  P.job[0] = {q0, 0, (int)ceil_div(q0, TBN)};
  if (P.njobs == 2) P.job[1] = {q1, q0, (int)ceil_div(q1, TBN)};
  P.p = p;
  P.mtiles = (int)ceil_div(p, TBM);
  P.tiles = P.mtiles * (P.job[0].ntiles + (P.njobs == 2 ? P.job[1].ntiles : 0));
  P.n = n;
  const int qtot = q0 + (P.njobs == 2 ? q1 : 0);
  int64_t ks = ceil_div(num_sms(), P.tiles);
  ks = std::max<int64_t>(1, std::min<int64_t>(ks, ceil_div(n, 256)));
  while (ks > 1 && (size_t)ks * p * qtot > partial_cap) --ks;
  if ((size_t)ks * p * qtot > partial_cap) {
    set_error("gram_tc partial workspace too small");
    return SPB_ERR_WORKSPACE;
  }
  P.kchunk = round_up(ceil_div(std::max<int64_t>(n, 1), ks), TBK);
  ks = ceil_div(std::max<int64_t>(n, 1), P.kchunk);
  P.ldo = qtot;
  P.split_stride = (int64_t)p * qtot;
  dim3 grid(P.tiles, (unsigned)ks);
  gram_tc_kernel<<<grid, 192, kSmemBytes, st>>>(mu, mv0, mv1, P, partial);
  SPB_LAUNCH_CHECK();
  const int64_t total = (int64_t)p * qtot;
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), 1024));
  sum_splits_tc<<<g, 256, 0, st>>>(partial, (int)ks, P.split_stride, p, qtot, qtot, out, ldo);
  SPB_LAUNCH_CHECK();
  return SPB_OK;
}

}  // namespace spb

using namespace spb;

namespace spb {
size_t gram_oz_ws_bytes(int64_t n, int p, int q);
int gram_oz(const float* U, int64_t ldu, int p, const float* V, int64_t ldv, int q, int64_t n,
            void* ws, size_t ws_bytes, double* out, int ldo, cudaStream_t st);
}  // namespace spb

extern "C" int spb_gram(int dtype, int mode, const void* u, int64_t ldu, int32_t p, const void* v,
                        int64_t ldv, int32_t q, int64_t n, double* out, int64_t ldo, void* ws,
                        size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (p < 0 || q < 0 || n < 0 || ldu < p || ldv < q || ldo < q) {
    set_error("gram shape contract violated");
    return SPB_ERR_CONTRACT;
  }
  double* part = (double*)ws;
  const size_t cap = ws_bytes / sizeof(double);
  if (mode == 2) {
    if (dtype != SPB_F32) {
      set_error("Ozaki tensor-core Gram needs float32 storage");
      return SPB_ERR_DOMAIN;
    }
    if (!gram_tc_supported()) {
      set_error("tensor-core Gram needs an sm_100 device");
      return SPB_ERR_CUDA;
    }
    return gram_oz((const float*)u, ldu, p, (const float*)v, ldv, q, n, ws, ws_bytes, out, (int)ldo, st);
  }
  if (mode == 1) {
    if (dtype != SPB_F32) {
      set_error("tensor-core Gram needs float32 storage");
      return SPB_ERR_DOMAIN;
    }
    if (!gram_tc_supported()) {
      set_error("tensor-core Gram needs an sm_100 device");
      return SPB_ERR_CUDA;
    }
    return gram_tc((const float*)u, ldu, p, (const float*)v, ldv, q, nullptr, 0, 0, n, part, cap,
                   out, (int)ldo, st);
  }
  GramBatch b{};
  b.njobs = 1;
  b.job[0] = {u, v, ldu, ldv, p, q, 0, 0};
  b.tile_start[0] = 0;
  b.tile_start[1] = (int)(ceil_div(p, 64) * ceil_div(q, 64));
  return gram_batched(dtype, b, n, p, q, part, cap, out, (int)ldo, st);
}

extern "C" size_t spb_gram_workspace(int32_t p, int32_t q, int64_t n) {
  size_t a = gram_tc_partial_doubles(n, p, q);
  size_t b = gram_partial_doubles(n, (int)(ceil_div(p, 64) * ceil_div(q, 64)), p, q, nullptr);
  const size_t c = gram_oz_ws_bytes(n, p, q) / sizeof(double) + 1;
  return (std::max(std::max(a, b), c) + 64) * sizeof(double);
}
