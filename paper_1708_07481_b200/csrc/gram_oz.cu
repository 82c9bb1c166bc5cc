// (c) Tall-skinny Gram products on the 5th-generation tensor cores with the
// Ozaki splitting: float64-accurate G = U'V from int8 tcgen05 MMAs.
//
//   G[p x q] = U' V,   U: n x p, V: n x q (float32, vertex-major, row stride ld)
//
// Every column c of U (and of V) gets a power-of-two scale 2^e_c > 2 max|x|; the
// scaled entries r in (-1/2, 1/2) are written as S = 6 signed digits in [-64, 64]
// (round to nearest), r = sum_t a_t 2^(-7t) + eps, |eps| <= 2^-43 (exact digit
// extraction in fp32).
// Then G_cd = 2^(e_c + e_d) sum_{t+u <= S+1} 2^(-7(t+u)) (A_t' B_u)_cd: 21 int8
// GEMMs with exact int32 accumulation, grouped by the level t+u into six TMEM
// accumulators, converted to fp64 and combined smallest level first. The
// per-product truncation error is O(2^-42) relative to the column maxima, far
// below the fp32 storage rounding of the operands.
//
// Four digits (10 MMAs, 128-wide tiles: 1.8 -> 1.45 ms per C3 Rayleigh-Ritz Gram
// pair, ~5e-9 relative) were measured in round 2 and rejected: the float32 C3 solve
// then stops after 23 iterations instead of the reference's 25 (its residual sits 5 %
// above the threshold at iteration 23), while five digits reproduce 25.
//
// Operands are pre-packed by oz_pack into the UMMA canonical K-major layout
// (core matrices of 8 columns x 16 bytes of K), the digits interleaved per group:
//   [kblock (32 rows)][column group (8 cols)][digit][k half][8 cols][16 rows]
// so a CTA's operand tile for one 32-row k-block -- all digits of its column
// groups -- is ONE contiguous bulk copy (digit plane t of a group at +256 t;
// 8-column groups OZ_S * 256 bytes apart = the descriptors' stride). Ten bulk
// copies per k-block (one per digit and operand) had cost ~20 % of the kernel.
//
// Per CTA: a 128 x 80 output tile over a range of k-blocks (split-K, at most
// 16384 rows so the int32 sums cannot overflow). Warp 0 issues the bulk copies
// (mbarrier pipeline, OZ_KS stages), warp 1 one thread issues the 21 MMAs per
// k-block, warps 2-5 the epilogue (tcgen05.ld -> fp64 partial tile); the split-K
// partials are reduced in a fixed order (sum_splits).
#include "dense.cuh"

namespace spb {

int oz_sum_splits(const double* part, int ks, int64_t stride, int rows, int cols, double* out,
                  int ldo, cudaStream_t st);

namespace {

constexpr int OZ_S = 5;          // digits per value (2^-35 of the column maxima)
constexpr int OZ_M = 128;        // UMMA M (columns of U per tile)
constexpr int OZ_N = 96;         // UMMA N (columns of V per tile); OZ_S * OZ_N <= 512 TMEM columns
constexpr int OZ_KB = 32;        // rows per k-block (one UMMA K step for 8-bit operands)
constexpr int OZ_KS = 4;         // pipeline stages (5, 6 measured equal)
constexpr int OZ_MAXROWS = 16384;  // rows per CTA: 6 pairs x 127^2 x 16384 < 2^31
constexpr int kOzA = OZ_S * (OZ_M / 8) * 256;  // bytes of the A planes per stage (24 KB)
constexpr int kOzB = OZ_S * (OZ_N / 8) * 256;  // bytes of the B planes per stage (15 KB)
constexpr int kOzStage = kOzA + kOzB;
constexpr int kOzSmem = OZ_KS * kOzStage + 1024 + 256;

__device__ __forceinline__ uint32_t s_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void oz_mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(bar)), "r"(count));
}
__device__ __forceinline__ void oz_mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void oz_mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "OZW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra OZW_%=;\n}" ::"r"(s_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          s_u32(dst)),
      "l"(src), "r"(bytes), "r"(s_u32(bar))
      : "memory");
}
__device__ __forceinline__ uint64_t oz_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (Blackwell); layout SWIZZLE_NONE
  return d;
}
__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
// one lane of a converged warp (elect.sync)
__device__ __forceinline__ bool oz_elect() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void oz_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   s_u32(bar))
               : "memory");
}

// Column maxima |x| (as float bits; non-negative floats order like their bits).
// Column scale exponent: 2^e > 2 max|x| (the scaled entries lie in (-1/2, 1/2), so the
// round-to-nearest digits below stay within [-64, 64]).
__device__ __forceinline__ int oz_exp(unsigned cm) {
  const float mx = __uint_as_float(cm);
  int e = 0;
  if (mx > 0.f) frexpf(mx, &e);  // mx < 2^e
  return e + 1;
}

__global__ void oz_colmax(const float* __restrict__ X, int64_t ldx, int64_t n, int cols,
                          unsigned* __restrict__ cmax) {
  const int c = blockIdx.y * 32 + (threadIdx.x & 31);
  if (c >= cols) return;
  unsigned m = 0;
  const int64_t step = (int64_t)gridDim.x * (blockDim.x >> 5);
#pragma unroll 8
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += step)
    m = max(m, __float_as_uint(fabsf(__ldg(X + r * ldx + c))));
  atomicMax(&cmax[c], m);
}

// Same with 16-byte loads: a warp covers 128 consecutive columns of a row.
// Up to two operands in one launch (blockIdx.z), e.g. the Rayleigh-Ritz B and LB.
struct OzSrc {
  const float* X;
  int64_t ldx;
  unsigned* cmax;
  int8_t* planes;
};
struct OzSrc2 {
  OzSrc s[2];
};

__global__ void oz_colmax4(const OzSrc2 P2, int64_t n, int cols) {
  const float* __restrict__ X = P2.s[blockIdx.z].X;
  const int64_t ldx = P2.s[blockIdx.z].ldx;
  unsigned* __restrict__ cmax = P2.s[blockIdx.z].cmax;
  __shared__ uint4 wm[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.y * 128 + lane * 4;
  unsigned m0 = 0, m1 = 0, m2 = 0, m3 = 0;
  if (c < cols) {
    const int64_t step = (int64_t)gridDim.x * (blockDim.x >> 5);
#pragma unroll 8
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; r < n; r += step) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(X + r * ldx + c));
      m0 = max(m0, __float_as_uint(fabsf(v.x)));
      m1 = max(m1, __float_as_uint(fabsf(v.y)));
      m2 = max(m2, __float_as_uint(fabsf(v.z)));
      m3 = max(m3, __float_as_uint(fabsf(v.w)));
    }
  }
  wm[warp][lane] = make_uint4(m0, m1, m2, m3);
  __syncthreads();
  // one atomic per column per CTA (8x fewer on the same addresses)
  if (warp == 0 && c < cols) {
    for (int q = 1; q < 8; ++q) {
      const uint4 o = wm[q][lane];
      m0 = max(m0, o.x);
      m1 = max(m1, o.y);
      m2 = max(m2, o.z);
      m3 = max(m3, o.w);
    }
    atomicMax(&cmax[c], m0);
    if (c + 1 < cols) atomicMax(&cmax[c + 1], m1);
    if (c + 2 < cols) atomicMax(&cmax[c + 2], m2);
    if (c + 3 < cols) atomicMax(&cmax[c + 3], m3);
  }
}

// Digits of x / 2^e_c into the packed planes (see the header comment). One
// thread per (k-block, k half, column): 16 consecutive rows of one column, the
// lanes of a warp on 32 consecutive columns (coalesced row reads); the 16 digit
// bytes of each plane are packed in registers and stored as one 16-byte vector
// (a warp's stores form contiguous 128-byte runs).
__global__ void __launch_bounds__(256)
oz_pack(const OzSrc2 P2, int64_t n, int cols, int ncg, int64_t nkb, int stride) {
  const float* __restrict__ X = P2.s[blockIdx.z].X;
  const int64_t ldx = P2.s[blockIdx.z].ldx;
  const unsigned* __restrict__ cmax = P2.s[blockIdx.z].cmax;
  int8_t* __restrict__ planes = P2.s[blockIdx.z].planes;
  const int cpad = ncg * 8;
  const int64_t total = nkb * 2 * cpad;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(t % cpad);
    const int64_t kh = t / cpad;
    const int h = (int)(kh & 1);
    const int64_t kb = kh >> 1;
    const int e = c < cols ? oz_exp(cmax[c]) : 0;
    const float sc = ldexpf(1.0f, -e);  // exact power of two (normal range)
    float xv[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int64_t r = kb * OZ_KB + h * 16 + i;
      xv[i] = (c < cols && r < n) ? __ldg(X + r * ldx + c) : 0.f;
    }
    uint32_t w[OZ_S][4];
#pragma unroll
    for (int sd = 0; sd < OZ_S; ++sd)
#pragma unroll
      for (int q = 0; q < 4; ++q) w[sd][q] = 0u;
    // digits by round-to-nearest through the 1.5 * 2^23 magic constant: the digit is
    // the low byte of t's bit pattern (two's complement), no float -> int conversion
    // (the F2I pipe runs at a quarter of the FP32 rate and bound this kernel)
    constexpr float kMagic = 12582912.0f;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float v = xv[i] * sc;  // exact: power-of-two scaling, |v| < 1/2
#pragma unroll
      for (int sd = 0; sd < OZ_S; ++sd) {
        const float y = v * 128.f;   // exact, |y| < 64 (+ rounding carry of the level above)
        const float t = y + kMagic;  // round(y) in the low mantissa bits
        const float a = t - kMagic;  // exact
        v = y - a;                   // exact, |v| <= 1/2
        w[sd][i >> 2] |= (__float_as_uint(t) & 0xffu) << (8 * (i & 3));
      }
    }
    // stride: column groups per k-block of the buffer (> ncg when packing a view)
    const int64_t off = ((kb * stride + (c >> 3)) * OZ_S * 2 + h) * 128 + (c & 7) * 16;
#pragma unroll
    for (int sd = 0; sd < OZ_S; ++sd)
      *reinterpret_cast<uint4*>(planes + off + sd * 256) = make_uint4(w[sd][0], w[sd][1], w[sd][2], w[sd][3]);
  }
}

// One Gram of a launch: out = A' B from two packed operands.
struct OzJob {
  const int8_t* PA;
  const int8_t* PB;
  const unsigned* cmaxA;
  const unsigned* cmaxB;
  int64_t planeA, planeB;  // bytes per plane
  int ncgA, ncgB;          // column groups of the operands
  int strideA, strideB;    // column groups per k-block of the buffers they live in
  int p, q;                // output rows (A columns), columns (B columns)
  double* part;            // split-K partials, ks x p x q
};

constexpr int kOzMaxTiles = 96;

struct OzParams {
  OzJob job[2];
  uint8_t tm[kOzMaxTiles], tn[kOzMaxTiles], tj[kOzMaxTiles];  // active (m tile, n tile, job)
  int64_t nkb;       // k-blocks
  int64_t kbchunk;   // k-blocks per split
};

__global__ void __launch_bounds__(192, 1)
gram_oz_kernel(const __grid_constant__ OzParams P) {
  extern __shared__ __align__(1024) uint8_t osm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)osm + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(base + OZ_KS * kOzStage);
  uint64_t* empty = full + OZ_KS;
  uint64_t* accb = empty + OZ_KS;
  uint32_t* tmem_slot = (uint32_t*)(accb + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const OzJob& J = P.job[P.tj[blockIdx.x]];
  const int8_t* __restrict__ PA = J.PA;
  const int8_t* __restrict__ PB = J.PB;
  const int m0 = P.tm[blockIdx.x] * OZ_M, n0 = P.tn[blockIdx.x] * OZ_N;
  const int64_t kb0 = (int64_t)blockIdx.y * P.kbchunk;
  const int64_t kb1 = min(P.nkb, kb0 + P.kbchunk);
  const int nk = kb1 > kb0 ? (int)(kb1 - kb0) : 0;
  const int gA = m0 / 8, gB = n0 / 8;
  const int cgA = min(OZ_M / 8, J.ncgA - gA);  // column groups present in this tile
  const int cgB = min(OZ_N / 8, J.ncgB - gB);
  // UMMA N of this tile: the last column tile of a narrow Gram (C3's 108 = 96 + 12
  // columns) runs N = 16 instead of 96 (N: multiple of 16 for M = 128)
  const int ntile = min(OZ_N, (J.q - n0 + 15) & ~15);

  if (threadIdx.x == 0) {
    for (int s = 0; s < OZ_KS; ++s) {
      oz_mbar_init(&full[s], 1);
      oz_mbar_init(&empty[s], 1);
    }
    oz_mbar_init(accb, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     s_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // zero the operand buffers once: column groups absent from a tile stay zero
  for (int i = threadIdx.x; i < OZ_KS * kOzStage / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(base)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0 && nk > 0) {
      const uint32_t bytesA = (uint32_t)cgA * OZ_S * 256, bytesB = (uint32_t)cgB * OZ_S * 256;
      for (int kc = 0; kc < nk; ++kc) {
        const int s = kc % OZ_KS, u = kc / OZ_KS;
        if (u > 0) oz_mbar_wait(&empty[s], (u - 1) & 1);
        uint8_t* st = base + s * kOzStage;
        oz_mbar_expect(&full[s], bytesA + bytesB);
        const int64_t kb = kb0 + kc;
        bulk_g2s(st, PA + (kb * J.strideA + gA) * OZ_S * 256, bytesA, &full[s]);
        bulk_g2s(st + kOzA, PB + (kb * J.strideB + gB) * OZ_S * 256, bytesB, &full[s]);
      }
    }
  } else if (warp == 1) {
    // the whole warp walks the pipeline (converged: descriptors and TMEM addresses
    // stay in uniform registers); one elected lane issues the MMAs and commits
    if (nk > 0) {
      const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) |  // S32 acc, s8 A/B, K-major
                             ((uint32_t)(ntile >> 3) << 17) | ((uint32_t)(OZ_M >> 4) << 24);
      const uint64_t dA0 = oz_desc(s_u32(base), 128, OZ_S * 256);
      const uint64_t dB0 = oz_desc(s_u32(base + kOzA), 128, OZ_S * 256);
      for (int kc = 0; kc < nk; ++kc) {
        const int s = kc % OZ_KS, u = kc / OZ_KS;
        oz_mbar_wait(&full[s], u & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        // descriptor start addresses advance in 16-byte units (no carry out of the
        // 14-bit field: every shared-memory address is < 256 KB)
        const uint64_t ds = (uint64_t)((s * kOzStage) >> 4);
        if (oz_elect()) {
          // level L = t + u - 2 accumulates digit pairs (t, u), t + u <= S + 1
#pragma unroll
          for (int t = 1; t <= OZ_S; ++t)
#pragma unroll
            for (int uu = 1; uu <= OZ_S; ++uu) {
              if (t + uu > OZ_S + 1) continue;
              const int L = t + uu - 2;
              const uint64_t da = dA0 + ds + (uint64_t)(((t - 1) * 256) >> 4);
              const uint64_t db = dB0 + ds + (uint64_t)(((uu - 1) * 256) >> 4);
              // first write of level L in this CTA: the (1, L+1) pair at kc == 0
              const uint32_t acc = (kc > 0 || t > 1) ? 1u : 0u;
              umma_i8(tmem + (uint32_t)(L * OZ_N), da, db, idesc, acc);
            }
          oz_commit(&empty[s]);
        }
        __syncwarp();
      }
      if (oz_elect()) oz_commit(accb);
      __syncwarp();
    }
  } else {
    // epilogue: warps 2..5 -> TMEM lanes 32*(warp & 3) .. +31 = tile rows
    if (nk > 0) {
      oz_mbar_wait(accb, 0);
      asm volatile("tcgen05.fence::after_thread_sync;");
    }
    const int quarter = warp & 3;
    const int row = m0 + quarter * 32 + lane;
    const int eA = row < J.p ? oz_exp(J.cmaxA[row]) : 0;
    double* out = J.part + (int64_t)blockIdx.y * J.p * J.q;
    for (int c0 = 0; c0 < ntile; c0 += 16) {
      double acc[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = 0.0;
      if (nk > 0) {
#pragma unroll
        for (int L = OZ_S - 1; L >= 0; --L) {  // smallest level first
          uint32_t r[16];
          const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(L * OZ_N + c0);
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, "
              "%10, %11, %12, %13, %14, %15}, [%16];"
              : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),
                "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
              : "r"(taddr));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          const double sc = ldexp(1.0, -7 * (L + 2));
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[i] = fma((double)(int)r[i], sc, acc[i]);
        }
      }
      if (row < J.p) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int col = n0 + c0 + i;
          if (col < J.q) {
            out[(int64_t)row * J.q + col] = ldexp(acc[i], eA + oz_exp(J.cmaxB[col]));
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

}  // namespace

// One operand in the packed digit layout (planes + per-column max bits).
struct OzOperand {
  int8_t* planes = nullptr;
  unsigned* cmax = nullptr;
  int cols = 0, ncg = 0;
  int stride = 0;  // column groups per k-block of the buffer (== ncg unless a view)
  int64_t n = 0, nkb = 0, plane_bytes = 0;
};

size_t oz_operand_bytes(int64_t n, int cols) {
  const int64_t nkb = ceil_div(std::max<int64_t>(n, 1), OZ_KB);
  // rounded to 1 KB: the next operand's planes are bulk-copy sources (16-byte aligned)
  const size_t b = (size_t)OZ_S * nkb * ceil_div(cols, 8) * 256 + sizeof(unsigned) * (size_t)cols;
  return (b + 1023) / 1024 * 1024;
}

// Where an operand of n x cols lives inside mem (no launch).
void oz_describe(int64_t n, int cols, void* mem, OzOperand* op) {
  op->cols = cols;
  op->n = n;
  op->nkb = ceil_div(std::max<int64_t>(n, 1), OZ_KB);
  op->ncg = (int)ceil_div(cols, 8);
  op->stride = op->ncg;
  op->plane_bytes = op->nkb * op->ncg * 256;
  op->planes = (int8_t*)mem;
  op->cmax = (unsigned*)(op->planes + OZ_S * op->plane_bytes);
}

// Columns [col0, col0 + cols) of a packed operand (col0 a multiple of 8) as an
// operand of their own: same planes, the parent's k-block stride.
OzOperand oz_view(const OzOperand& W, int col0, int cols) {
  OzOperand v = W;
  v.planes = W.planes + (size_t)(col0 / 8) * OZ_S * 256;
  v.cmax = W.cmax + col0;
  v.cols = cols;
  v.ncg = (int)ceil_div(cols, 8);
  return v;
}

// Column maxima and digit planes of nop (1 or 2) described operands (whole buffers
// or views of the same shape: equal cols / ncg / stride) from the float32 blocks X[i]
// (n x cols, row stride ld[i]): one colmax launch and one pack launch for all.
int oz_fill_n(int nop, const float* const* X, const int64_t* ld, const OzOperand* op,
              cudaStream_t st) {
  OzSrc2 P2{};
  bool vec = true;
  const int64_t n = op[0].n;
  const int cols = op[0].cols;
  for (int i = 0; i < nop; ++i) {
    SPB_CUDA(cudaMemsetAsync(op[i].cmax, 0, sizeof(unsigned) * (size_t)cols, st));
    P2.s[i] = {X[i], ld[i], op[i].cmax, op[i].planes};
    vec = vec && (reinterpret_cast<uintptr_t>(X[i]) & 15) == 0 && (ld[i] & 3) == 0;
  }
  if (vec) {
    oz_colmax4<<<dim3((unsigned)std::min<int64_t>(ceil_div(n, 64), 2 * num_sms()),
                      (unsigned)ceil_div(cols, 128), (unsigned)nop),
                 256, 0, st>>>(P2, n, cols);
  } else {
    const int gx = (int)std::min<int64_t>(ceil_div(n, 8), 4 * num_sms());
    for (int i = 0; i < nop; ++i)
      oz_colmax<<<dim3(gx, (unsigned)ceil_div(cols, 32)), 256, 0, st>>>(X[i], ld[i], n, cols,
                                                                         op[i].cmax);
  }
  const int64_t t = op[0].nkb * 2 * op[0].ncg * 8;
  oz_pack<<<dim3((unsigned)std::min<int64_t>(ceil_div(t, 256), 16 * num_sms()), 1, (unsigned)nop), 256,
            0, st>>>(P2, n, cols, op[0].ncg, op[0].nkb, op[0].stride);
  SPB_LAUNCH_CHECK();
  return SPB_OK;
}

// The same for whole operands laid out in mem[i].
int oz_prepare_n(int nop, const float* const* X, const int64_t* ld, int64_t n, int cols,
                 void* const* mem, OzOperand* op, cudaStream_t st) {
  for (int i = 0; i < nop; ++i) oz_describe(n, cols, mem[i], &op[i]);
  return oz_fill_n(nop, X, ld, op, st);
}

int oz_prepare(const float* X, int64_t ldx, int64_t n, int cols, void* mem, OzOperand* op,
               cudaStream_t st) {
  const float* xs[1] = {X};
  const int64_t ls[1] = {ldx};
  void* ms[1] = {mem};
  return oz_prepare_n(1, xs, ls, n, cols, ms, op, st);
}

// Split-K factor of a launch with `tiles` output tiles over nkb k-blocks: at most
// OZ_MAXROWS rows per split (exact int32 sums), at least two CTAs per SM, and
// among the next few candidates the one with the fewest idle CTA slots in the
// last wave (one CTA per SM).
// sms: the SMs the launch can count on (fewer than the device's when a cluster kernel
// runs beside it on another stream).
int64_t oz_splits(int64_t nkb, int tiles, int sms = 0) {
  if (sms <= 0) sms = num_sms();
  const int64_t lo = std::max<int64_t>(ceil_div(2 * sms, tiles), ceil_div(nkb, OZ_MAXROWS / OZ_KB));
  int64_t best = std::min<int64_t>(lo, nkb);
  double best_eff = 0.0;
  for (int64_t ks = best; ks <= std::min<int64_t>(nkb, lo + 16); ++ks) {
    const int64_t kb = ceil_div(nkb, ks), kse = ceil_div(nkb, kb);  // effective splits
    const int64_t units = (int64_t)tiles * kse;
    const double eff = (double)units / (double)(ceil_div(units, sms) * sms);
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = ks;
    }
  }
  return best;
}

size_t gram_oz_partial_doubles(int64_t n, int p, int q) {
  const int tiles = (int)(ceil_div(p, OZ_M) * ceil_div(q, OZ_N));
  const int64_t nkb = ceil_div(std::max<int64_t>(n, 1), OZ_KB);
  // the Rayleigh-Ritz launch runs two jobs (G_B upper tiles + G_A) in one grid
  int64_t ks = std::max(oz_splits(nkb, tiles), oz_splits(nkb, 2 * tiles));
  ks = std::max<int64_t>(ks, ceil_div(2 * num_sms(), tiles));
  if (p == q) {  // G_B alone (upper tiles only) when the two Grams go out as two launches
    int ut = 0;
    for (int nt = 0; nt < (int)ceil_div(q, OZ_N); ++nt)
      for (int mt = 0; mt < (int)ceil_div(p, OZ_M); ++mt) ut += (nt + 1) * OZ_N > mt * OZ_M;
    ks = std::max(ks, oz_splits(nkb, ut));
  }
  ks = std::min<int64_t>(ks + 16, nkb);
  return (size_t)std::max<int64_t>(ks, 1) * p * q;
}

// outs[j][A_j.cols x B_j.cols] (ld ldo) = A_j' B_j for one or two jobs in ONE launch
// (all k-blocks of every job split the same way); upper[j]: B_j == A_j, only tiles
// reaching the diagonal are computed. partial: per job gram_oz_partial_doubles.
int oz_gemm_jobs(int njobs, const OzOperand* const* A, const OzOperand* const* B, const bool* upper,
                 double* const* partial, size_t partial_cap, double* const* out, int ldo,
                 cudaStream_t st, int sms = 0) {
  static std::atomic<uint64_t> attr{0};
  if (!done_on_device(attr)) {
    SPB_CUDA(cudaFuncSetAttribute(gram_oz_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kOzSmem));
    mark_on_device(attr);
  }
  OzParams P{};
  int tiles = 0;
  for (int j = 0; j < njobs; ++j) {
    const int p = A[j]->cols, q = B[j]->cols;
    if (p <= 0 || q <= 0) continue;
    OzJob& J = P.job[j];
    J.PA = A[j]->planes;
    J.PB = B[j]->planes;
    J.cmaxA = A[j]->cmax;
    J.cmaxB = B[j]->cmax;
    J.planeA = A[j]->plane_bytes;
    J.planeB = B[j]->plane_bytes;
    J.ncgA = A[j]->ncg;
    J.ncgB = B[j]->ncg;
    J.strideA = A[j]->stride;
    J.strideB = B[j]->stride;
    J.p = p;
    J.q = q;
    J.part = partial[j];
    const int mtiles = (int)ceil_div(p, OZ_M), ntiles = (int)ceil_div(q, OZ_N);
    for (int nt = 0; nt < ntiles; ++nt)
      for (int mt = 0; mt < mtiles; ++mt) {
        if (upper[j] && (nt + 1) * OZ_N <= mt * OZ_M) continue;  // wholly below the diagonal
        if (tiles == kOzMaxTiles) {
          set_error("Ozaki Gram: more than %d output tiles", kOzMaxTiles);
          return SPB_ERR_CONTRACT;
        }
        P.tm[tiles] = (uint8_t)mt;
        P.tn[tiles] = (uint8_t)nt;
        P.tj[tiles] = (uint8_t)j;
        ++tiles;
      }
  }
  if (tiles == 0) return SPB_OK;
  const int64_t nkb = A[0]->nkb;
  int64_t ks = oz_splits(nkb, tiles, sms);
  size_t need = 0;
  for (int j = 0; j < njobs; ++j) need = std::max(need, (size_t)P.job[j].p * P.job[j].q);
  while (ks > 1 && (size_t)ks * need > partial_cap) --ks;
  P.nkb = nkb;
  P.kbchunk = ceil_div(nkb, ks);
  ks = ceil_div(nkb, P.kbchunk);
  if ((size_t)ks * need > partial_cap || P.kbchunk * OZ_KB > OZ_MAXROWS) {
    set_error("Ozaki Gram partial workspace too small");
    return SPB_ERR_WORKSPACE;
  }
  gram_oz_kernel<<<dim3(tiles, (unsigned)ks), 192, kOzSmem, st>>>(P);
  SPB_LAUNCH_CHECK();
  for (int j = 0; j < njobs; ++j)
    if (P.job[j].p > 0 && P.job[j].q > 0)
      SPB_TRY(oz_sum_splits(P.job[j].part, (int)ks, (int64_t)P.job[j].p * P.job[j].q, P.job[j].p,
                            P.job[j].q, out[j], ldo, st));
  return SPB_OK;
}

// out[A.cols x B.cols] (ld ldo) = A' B from two prepared operands.
int oz_gemm(const OzOperand& A, const OzOperand& B, double* partial, size_t partial_cap,
            double* out, int ldo, cudaStream_t st, bool upper = false, int sms = 0) {
  const OzOperand* a[1] = {&A};
  const OzOperand* b[1] = {&B};
  double* pp[1] = {partial};
  double* oo[1] = {out};
  return oz_gemm_jobs(1, a, b, &upper, pp, partial_cap, oo, ldo, st, sms);
}

// Workspace of gram_oz: both operands' digit planes, then the split-K partials.
size_t gram_oz_ws_bytes(int64_t n, int p, int q) {
  return oz_operand_bytes(n, p) + oz_operand_bytes(n, q) +
         2 * gram_oz_partial_doubles(n, p, q) * sizeof(double) + 2048;
}

// out[p x q] (ld ldo) = U' V with float32 operands, float64-accurate; ws is caller
// memory of gram_oz_ws_bytes(n, p, q) bytes (no allocation here).
int gram_oz(const float* U, int64_t ldu, int p, const float* V, int64_t ldv, int q, int64_t n,
            void* ws, size_t ws_bytes, double* out, int ldo, cudaStream_t st) {
  if (p <= 0 || q <= 0) return SPB_OK;
  const size_t ba = oz_operand_bytes(n, p), bb = oz_operand_bytes(n, q);
  if (ws_bytes < gram_oz_ws_bytes(n, p, q)) {
    set_error("Ozaki Gram workspace too small (%zu < %zu bytes)", ws_bytes, gram_oz_ws_bytes(n, p, q));
    return SPB_ERR_WORKSPACE;
  }
  uint8_t* scr = (uint8_t*)ws;
  double* partial = (double*)(scr + ba + bb);
  const size_t partial_cap = (ws_bytes - ba - bb) / sizeof(double);
  OzOperand A, B;
  if (U == V && ldu == ldv && p == q) {  // U'U: one operand, packed once
    SPB_TRY(oz_prepare(U, ldu, n, p, scr, &A, st));
    return oz_gemm(A, A, partial, partial_cap, out, ldo, st);
  }
  if (p == q) {  // both operands in one column-maxima and one packing launch
    const float* xs[2] = {U, V};
    const int64_t ls[2] = {ldu, ldv};
    void* ms[2] = {scr, scr + ba};
    OzOperand ops[2];
    SPB_TRY(oz_prepare_n(2, xs, ls, n, p, ms, ops, st));
    return oz_gemm(ops[0], ops[1], partial, partial_cap, out, ldo, st);
  }
  SPB_TRY(oz_prepare(U, ldu, n, p, scr, &A, st));
  SPB_TRY(oz_prepare(V, ldv, n, q, scr + ba, &B, st));
  return oz_gemm(A, B, partial, partial_cap, out, ldo, st);
}

// out[(c1 + q) x q] (ld ldo) = W' W[:, c1 : c1 + q] for W = the first c1 + q columns of
// a float32 block (row stride ld, c1 a multiple of 8), packed once: rows [0, c1) are
// X'R and rows [c1, c1 + q) are R'R when W = [X | R] (lobpcg.cu, project_orth).
// rr_cols > 0: W is packed in place inside the Rayleigh-Ritz B operand of rr_cols
// columns that gram_oz_rr will use on the same ws (its k-block stride), so the planes
// and column scales of the leading c1 columns (X) are already there for it
// (gram_oz_rr's keep_cols).
int gram_oz_xr(const float* W, int64_t ld, int64_t n, int c1, int q, void* ws, size_t ws_bytes,
               double* out, int ldo, cudaStream_t st, int rr_cols) {
  const int cols = c1 + q;
  uint8_t* scr = (uint8_t*)ws;
  OzOperand Wop;
  size_t poff;  // split-K partials behind the operand area
  if (rr_cols > 0) {
    if (rr_cols < cols || ws_bytes < gram_oz_ws_bytes(n, rr_cols, rr_cols)) {
      set_error("Ozaki [X R]'R Gram: Rayleigh-Ritz operand narrower than [X R]");
      return SPB_ERR_CONTRACT;
    }
    OzOperand RR;
    oz_describe(n, rr_cols, scr, &RR);
    Wop = oz_view(RR, 0, cols);
    poff = 2 * oz_operand_bytes(n, rr_cols);
  } else {
    oz_describe(n, cols, scr, &Wop);
    poff = oz_operand_bytes(n, cols);
  }
  if ((c1 & 7) || ws_bytes < poff + gram_oz_partial_doubles(n, cols, q) * sizeof(double)) {
    set_error("Ozaki [X R]'R Gram: bad split or workspace too small");
    return SPB_ERR_WORKSPACE;
  }
  SPB_TRY(oz_fill_n(1, &W, &ld, &Wop, st));
  const OzOperand R = oz_view(Wop, c1, q);
  return oz_gemm(Wop, R, (double*)(scr + poff), (ws_bytes - poff) / sizeof(double), out, ldo, st);
}

// The Rayleigh-Ritz Grams of the solver: Gb = B'B (upper triangle valid, ld ldo) and
// Ga = B'LB (ld ldo), B and LB n x cols (row stride ld), each operand packed once;
// ws: gram_oz_ws_bytes(n, cols, cols) bytes of the solver's workspace.
// phase 0: both Grams in one launch. Phases 1-4 split it for the caller's stream
// overlap (lobpcg.cu, rr_grams_body), in this order on the same ws: 1 packs B, 2
// launches Gb, 3 packs LB (may run beside 2 on another stream), 4 launches Ga.
// keep_cols (phase 1; a multiple of 8): the leading keep_cols columns of B were packed
// into this operand by gram_oz_xr(..., rr_cols = cols) and are unchanged since.
int gram_oz_rr(const float* B, const float* LB, int64_t ld, int64_t n, int cols, double* Ga,
               double* Gb, int ldo, void* ws, size_t ws_bytes, cudaStream_t st, int phase,
               int keep_cols) {
  const size_t bo = oz_operand_bytes(n, cols);
  if (ws_bytes < gram_oz_ws_bytes(n, cols, cols)) {
    set_error("Ozaki Gram workspace too small");
    return SPB_ERR_WORKSPACE;
  }
  uint8_t* scr = (uint8_t*)ws;
  double* part = (double*)(scr + 2 * bo);
  const size_t pc = (ws_bytes - 2 * bo) / sizeof(double) / 2;
  OzOperand ops[2];
  if (phase == 0) {
    const float* xs[2] = {B, LB};
    const int64_t ls[2] = {ld, ld};
    void* ms[2] = {scr, scr + bo};
    SPB_TRY(oz_prepare_n(2, xs, ls, n, cols, ms, ops, st));
  } else {
    oz_describe(n, cols, scr, &ops[0]);
    oz_describe(n, cols, scr + bo, &ops[1]);
    if (phase == 1) {
      if (keep_cols <= 0 || keep_cols >= cols || (keep_cols & 7))
        return oz_prepare(B, ld, n, cols, scr, &ops[0], st);
      const OzOperand rest = oz_view(ops[0], keep_cols, cols - keep_cols);
      const float* src = B + keep_cols;
      return oz_fill_n(1, &src, &ld, &rest, st);
    }
    if (phase == 2) return oz_gemm(ops[0], ops[0], part, pc, Gb, ldo, st, true);
    if (phase == 3) return oz_prepare(LB, ld, n, cols, scr + bo, &ops[1], st);
    // the G_B factorisation's 16-CTA cluster runs beside this launch (lobpcg.cu)
    return oz_gemm(ops[0], ops[1], part + pc, pc, Ga, ldo, st, false, num_sms() - 16);
  }
  const OzOperand& OB = ops[0];
  const OzOperand& OL = ops[1];
  // G_B (upper tiles, read as such) and G_A in one launch: one grid, one tail
  const OzOperand* a[2] = {&OB, &OB};
  const OzOperand* b[2] = {&OB, &OL};
  const bool up[2] = {true, false};
  double* pp[2] = {part, part + pc};
  double* oo[2] = {Gb, Ga};
  return oz_gemm_jobs(2, a, b, up, pp, pc, oo, ldo, st);
}

}  // namespace spb
