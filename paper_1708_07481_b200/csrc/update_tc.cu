// (c) Block update on the 5th-generation tensor cores: 3xTF32 split, TMA-fed.
//
//   acc = init + sum_s A_s (scale_s C_s),  written to seg.out after every
//   segment with emit set (the running sum, as block_update's other kernels).
//
// This is the LOBPCG basis update X' = X Cx + R Cr + P Cp, P' = R Cr + P Cp of
// lobpcg.py:436-439 (and the in-place right-multiplications of :228, :366) as a
// GEMM with M = 128 rows (vertices) per CTA, N = q (block width, padded to 16),
// K = the segment widths. The float32 operands are split as x = hi + lo with
// hi = x rounded to the nearest TF32 value and lo = (x - hi) rounded likewise
// (split error 2^-24 |x|); three tcgen05.mma.kind::tf32 per K step (hi*lo +
// lo*hi + hi*hi) into one fp32 TMEM accumulator give float32-accurate products.
//
// Warp roles (320 threads):
//   warp 0    TMA producer: {32 columns x 128 rows} boxes of A_s, 128-byte
//             swizzled, plus one bulk copy of the pre-split coefficient chunk
//             (hi | lo, same swizzled K-major layout, staged once per launch by
//             tc_stage_coeffs);
//   warp 1    MMA issuer (one thread); each 32-deep chunk into one of two TMEM
//             regions (double-buffered);
//   warps 2-5 splitters: hi written in place over the staged tile, lo into its
//             own buffer (elementwise, so the swizzled layout is preserved);
//   warps 6-9 epilogue (6-13 when q > 128, two warps per lane quarter, each
//             owning half of the columns): per chunk, tcgen05.ld the region and add it into
//             float32 registers (round-to-nearest: the tensor cores' own
//             accumulation, which is not, then spans 12 MMAs only); at every
//             emit, store the running sum (+ init) as float32 rows.
#include <cuda.h>

#include <cstdlib>

#include "dense.cuh"

namespace spb {
namespace {

constexpr int UTM = 128;             // rows per CTA (UMMA M)
constexpr int UTK = 32;              // K per chunk (one 128-byte swizzle atom of fp32)
// chunks per TMEM accumulation group: the tensor cores' fp32 accumulation is not
// round-to-nearest (biased), so its error grows with the MMAs it spans; 2 (64-deep,
// 24 MMAs, half the epilogue round trips) measurably moved float32 trajectories
// (C3 stopped after 23 instead of the reference's 25 iterations), 1 keeps 12
constexpr int kUtCpg = 1;
constexpr int UTS_MAX = 4;           // pipeline stages (runtime: 2 when two CTAs fit per SM)
constexpr int kUtA = UTM * UTK * 4;  // A tile bytes (16 KB)
constexpr int kUtThreads = 320;  // 6 + 4 EW warps; EW = 1 (q <= 128)
constexpr int kUtThreadsW = 448; // EW = 2 (q <= 192: each epilogue warp owns half the columns)

__device__ __forceinline__ uint32_t ut_smem(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void ut_mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(ut_smem(bar)), "r"(count));
}
__device__ __forceinline__ void ut_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ut_smem(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void ut_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ut_smem(bar)) : "memory");
}
__device__ __forceinline__ void ut_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "UTW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra UTW_%=;\n}" ::"r"(ut_smem(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void ut_tma2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                         int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(ut_smem(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(ut_smem(bar))
      : "memory");
}
__device__ __forceinline__ void ut_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          ut_smem(dst)),
      "l"(src), "r"(bytes), "r"(ut_smem(bar))
      : "memory");
}
// K-major, 128-byte swizzle: 8-row x 128-byte atoms, SBO = 1024 B between atoms
// along M/N; a K step of 8 tf32 advances the start address by 32 bytes.
__device__ __forceinline__ uint64_t ut_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                   // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;         // SBO
  d |= (uint64_t)1 << 46;                   // descriptor version (Blackwell)
  d |= (uint64_t)2 << 61;                   // layout: SWIZZLE_128B
  return d;
}
__device__ __forceinline__ void ut_mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
// one lane of a converged warp (elect.sync)
__device__ __forceinline__ bool ut_elect() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void ut_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   ut_smem(bar))
               : "memory");
}
// A from tensor memory (the split operands written by the splitter warps with
// tcgen05.st), B from shared memory.
__device__ __forceinline__ void ut_mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                          uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void ut_tmem_st32(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31, %32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
      "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]),
      "f"(v[16]), "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]),
      "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}

// Round to the nearest TF32 value (a float32 container with 13 zero low bits).
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// x = hi + lo with both parts TF32 values rounded to nearest: the split error is
// 2^-24 |x| (the lo part's own rounding), not the 2^-22 of truncated parts.
__device__ __forceinline__ void tf32_split(float x, float& hi, float& lo) {
  hi = tf32_rna(x);
  lo = tf32_rna(x - hi);  // x - hi is exact in float32
}

struct UtSeg {
  int chunks;      // ceil(w / UTK)
  int emit;
  float* out;
  int64_t ldo;
};

struct UtParams {
  UtSeg seg[3];
  int nseg;
  int q, npad;              // output columns, UMMA N (multiple of 16)
  int nemit;
  const float* init;
  int64_t ldi;
  const float* coef;        // staged chunks: [chunk][hi | lo][npad rows x 128 B, swizzled]
  // chunk groups (per tile, chunk index j < nk): a group of up to UT_CPG chunks of one
  // segment accumulates in one TMEM region before the epilogue adds it into registers
  uint8_t gstart[32], gend[32];
  int64_t n;
  uint32_t tmem_cols;
  int stages;
  const float* argmin_bias;          // argmin epilogue (see UpdParams)
  int* argmin_labels;
  unsigned long long* argmin_changed;
  int tma_store;        // emits go out as TMA tensor stores from swizzled smem staging
  uint32_t stg_off;     // staging offset from the aligned smem base: [EW][2][128 rows][128 B]
};

// Orderable 64-bit key of (distance, column): unsigned compare = (dist, col) lexicographic.
__device__ __forceinline__ unsigned long long ut_argkey(float d, int j) {
  const uint32_t b = __float_as_uint(d);
  const uint32_t o = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  return ((unsigned long long)o << 32) | (uint32_t)j;
}

// Coefficient chunks: element (output column j, k) of chunk c of segment s is
// scale_s C_s[32 c + k][j], stored at the 128-byte-swizzled K-major position.
__global__ void tc_stage_coeffs(UpdParams P, int npad, float* __restrict__ dst) {
  int cbase = 0;
  for (int s = 0; s < P.nseg; ++s) {
    const UpdSeg sg = P.seg[s];
    const int chunks = (sg.w + UTK - 1) / UTK;
    const int total = chunks * npad * UTK;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
      const int c = e / (npad * UTK), r = e % (npad * UTK);
      const int j = r / UTK, k = r % UTK;
      const int kg = c * UTK + k;
      float x = 0.0f;
      if (kg < sg.w && j < P.q) x = (float)(sg.scale * sg.C[(int64_t)kg * sg.ldc + j]);
      float h, l;
      tf32_split(x, h, l);
      const int off = (j >> 3) * 256 + (j & 7) * 32 + (((k >> 2) ^ (j & 7)) << 2) + (k & 3);
      float* chunk = dst + (size_t)(cbase + c) * 2 * npad * UTK;
      chunk[off] = h;
      chunk[npad * UTK + off] = l;
    }
    cbase += chunks;
  }
}

// ATM (A in tensor memory, npad <= 128): the splitters read their row of the TMA'd
// A tile, split it and store hi / lo into per-stage TMEM columns (256 + 64 s ...),
// so a stage is only [A raw][B hi|lo] in shared memory -- four stages instead of
// three -- and the MMAs read A from TMEM instead of shared memory.
template <int NPMAX, int EW, bool ATM = false>
__global__ void __launch_bounds__(EW == 1 ? kUtThreads : kUtThreadsW, 1)
update_tc_kernel(const __grid_constant__ CUtensorMap map0, const __grid_constant__ CUtensorMap map1,
                 const __grid_constant__ CUtensorMap map2, const __grid_constant__ CUtensorMap omap0,
                 const __grid_constant__ CUtensorMap omap1, const __grid_constant__ CUtensorMap omap2,
                 UtParams P) {
  extern __shared__ __align__(1024) uint8_t usm_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)usm_raw + 1023) & ~(uintptr_t)1023);
  const int kB = 2 * P.npad * UTK * 4;              // coefficient chunk bytes (hi | lo)
  // [A hi (staged in place)][A lo][B hi|lo], or with ATM [A raw][B hi|lo]
  const int kStage = (ATM ? 1 : 2) * kUtA + kB;
  const int kBoff = (ATM ? 1 : 2) * kUtA;          // B offset inside a stage
  const int UTS = P.stages;
  uint64_t* full = (uint64_t*)(base + UTS * kStage);
  uint64_t* split = full + UTS_MAX;
  uint64_t* empty = split + UTS_MAX;
  uint64_t* rdone = empty + UTS_MAX;                // [2] chunk partial ready in TMEM
  uint64_t* rfree = rdone + 2;                      // [2] region read by the epilogue
  uint32_t* tmem_slot = (uint32_t*)(rfree + 2);
  // argmin keys [tile parity][column half][row]
  unsigned long long* akeys = (unsigned long long*)(base + UTS * kStage + 256);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = (int)((P.n + UTM - 1) / UTM);
  // persistent: tiles blockIdx.x, blockIdx.x + gridDim.x, ...; chunk counters
  // run on across tiles so the stage ring and TMEM regions never drain
  int nk = 0;
  for (int s = 0; s < P.nseg; ++s) nk += P.seg[s].chunks;

  if (threadIdx.x == 0) {
    for (int s = 0; s < UTS; ++s) {
      ut_mbar_init(&full[s], 1);
      ut_mbar_init(&split[s], 128);
      ut_mbar_init(&empty[s], 1);
    }
    for (int e = 0; e < 2; ++e) {
      ut_mbar_init(&rdone[e], 1);
      ut_mbar_init(&rfree[e], 128 * EW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     ut_smem(tmem_slot)),
                 "r"(P.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int st = 0, u = 0;  // stage ring position (no integer division in the loops)
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int kc = 0;
        for (int s = 0; s < P.nseg; ++s) {
          const CUtensorMap* map = s == 0 ? &map0 : (s == 1 ? &map1 : &map2);
          for (int c = 0; c < P.seg[s].chunks; ++c, ++kc) {
            if (u > 0) ut_wait(&empty[st], (u - 1) & 1);
            uint8_t* sb = base + st * kStage;
            ut_expect(&full[st], (uint32_t)(kUtA + kB));
            ut_tma2d(sb, map, &full[st], c * UTK, tile * UTM);
            ut_bulk(sb + kBoff, P.coef + (size_t)kc * 2 * P.npad * UTK, (uint32_t)kB, &full[st]);
            if (++st == UTS) { st = 0; ++u; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // the whole warp walks the pipeline (converged: descriptors and TMEM addresses
    // stay in uniform registers); one elected lane issues the MMAs and commits
    {
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) |  // F32 acc, TF32 A/B, K-major
                             ((uint32_t)(P.npad >> 3) << 17) | ((uint32_t)(UTM >> 4) << 24);
      const int total = ((ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x) * nk;
      const uint64_t dbase = ut_desc_sw128(ut_smem(base + kBoff));  // stage 0's B hi
      const uint32_t blo_off = (uint32_t)(P.npad * UTK * 4) >> 4;
      int G = 0, rg = 0;  // chunk group counter / its TMEM region (double-buffered)
      int st = 0, u = 0, j = 0;  // stage ring position, chunk index within the tile
      for (int kc = 0; kc < total; ++kc) {
        const bool first = P.gstart[j] != 0;
        if (first) {
          rg = G & 1;
          if (G >= 2) ut_wait(&rfree[rg], ((G >> 1) - 1) & 1);
        }
        ut_wait(&split[st], u & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        // descriptor start addresses advance in 16-byte units (no carry: smem < 256 KB)
        const uint64_t dbh0 = dbase + (uint64_t)(((uint32_t)st * (uint32_t)kStage) >> 4);
        const uint64_t dbl0 = dbh0 + blo_off;
        const uint32_t dacc = tmem + (uint32_t)(rg * P.npad);
        if (ut_elect()) {
          if constexpr (ATM) {
            const uint32_t ta = tmem + 256u + (uint32_t)st * 64u;  // hi at +0, lo at +32
#pragma unroll
            for (int kk = 0; kk < UTK / 8; ++kk) {
              const uint64_t dbh = dbh0 + (uint64_t)(kk * 2), dbl = dbl0 + (uint64_t)(kk * 2);
              ut_mma_ts(dacc, ta + kk * 8, dbl, idesc, (kk == 0 && first) ? 0u : 1u);
              ut_mma_ts(dacc, ta + 32 + kk * 8, dbh, idesc, 1u);
              ut_mma_ts(dacc, ta + kk * 8, dbh, idesc, 1u);
            }
          } else {
            const uint64_t dah0 = ut_desc_sw128(ut_smem(base)) +
                                  (uint64_t)(((uint32_t)st * (uint32_t)kStage) >> 4);
            const uint64_t dal0 = dah0 + (uint64_t)(kUtA >> 4);
#pragma unroll
            for (int kk = 0; kk < UTK / 8; ++kk) {
              const uint64_t o = (uint64_t)(kk * 2);  // 32 bytes per K step of 8 tf32
              ut_mma(dacc, dah0 + o, dbl0 + o, idesc, (kk == 0 && first) ? 0u : 1u);  // small terms first
              ut_mma(dacc, dal0 + o, dbh0 + o, idesc, 1u);
              ut_mma(dacc, dah0 + o, dbh0 + o, idesc, 1u);
            }
          }
          ut_commit(&empty[st]);
          if (P.gend[j]) ut_commit(&rdone[rg]);
        }
        __syncwarp();
        if (P.gend[j]) ++G;
        if (++st == UTS) { st = 0; ++u; }
        if (++j == nk) j = 0;
      }
    }
  } else if (warp < 6) {
    // splitters: hi in place, lo to its own buffer (elementwise: layout preserved)
    const int t = threadIdx.x - 64;
    const int total = ((ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x) * nk;
    int st = 0, u = 0;  // stage ring position (no integer division in the loop)
    for (int kc = 0; kc < total; ++kc, st = (st + 1 == UTS) ? 0 : st + 1, u += (st == 0)) {
      ut_wait(&full[st], u & 1);
      if constexpr (ATM) {
        // this thread's row of the 128B-swizzled tile: 16-byte chunk c of row r sits at
        // position c ^ (r & 7) (conflict-free: 8 rows cover all banks)
        const int r = 32 * (warp & 3) + lane;
        const uint32_t row_s = ut_smem(base + st * kStage + r * 128);  // explicit ld.shared
        float hi[32], lo[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          float4 x;
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
                       : "r"(row_s + (uint32_t)((c ^ (r & 7)) * 16)));
          tf32_split(x.x, hi[4 * c], lo[4 * c]);
          tf32_split(x.y, hi[4 * c + 1], lo[4 * c + 1]);
          tf32_split(x.z, hi[4 * c + 2], lo[4 * c + 2]);
          tf32_split(x.w, hi[4 * c + 3], lo[4 * c + 3]);
        }
        const uint32_t ta = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + 256u + (uint32_t)st * 64u;
        ut_tmem_st32(ta, hi);
        ut_tmem_st32(ta + 32, lo);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;");
        ut_arrive(&split[st]);
        continue;
      }
      // explicit shared-space accesses (generic pointers derived from the aligned
      // dynamic-smem base compiled to generic LD/ST: lg_throttle stalls in ncu)
      const uint32_t a_s = ut_smem(base + st * kStage), lo_s = a_s + kUtA;
#pragma unroll
      for (int i = 0; i < kUtA / 16 / 128; ++i) {
        const uint32_t e = (uint32_t)(i * 128 + t) * 16u;
        float4 x, h, l;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w) : "r"(a_s + e));
        tf32_split(x.x, h.x, l.x);
        tf32_split(x.y, h.y, l.y);
        tf32_split(x.z, h.z, l.z);
        tf32_split(x.w, h.w, l.w);
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a_s + e), "f"(h.x), "f"(h.y),
                     "f"(h.z), "f"(h.w) : "memory");
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(lo_s + e), "f"(l.x), "f"(l.y),
                     "f"(l.z), "f"(l.w) : "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      ut_arrive(&split[st]);
    }
  } else {
    // epilogue: warps 6..9 -> TMEM lane quarter (warp & 3) = tile rows. Every
    // chunk group's partial product (UT_CPG x 32 deep) is added into float32
    // registers (round-to-nearest), so the tensor cores' own accumulation covers
    // at most 24 MMAs; the running sum is written at every emit.
    constexpr int NH = NPMAX / EW;         // columns per epilogue warp
    const int quarter = warp & 3;
    const int cb = ((warp - 6) >> 2) * NH;  // first column of this warp
    int G = 0, npass = 0;
    const int half = (warp - 6) >> 2;
    const bool issuer = (warp & 3) == 2 && lane == 0;  // first warp of this column half
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row = (int64_t)tile * UTM + quarter * 32 + lane;
    int j = 0;  // chunk index within the tile
    float acc[NH];
#pragma unroll
    for (int i = 0; i < NH; ++i) acc[i] = 0.0f;
    if (P.init && row < P.n) {
      const float* irow = P.init + row * P.ldi + cb;
      const bool vec = (reinterpret_cast<uintptr_t>(irow) & 15) == 0;
#pragma unroll
      for (int c0 = 0; c0 < NH; c0 += 4) {
        if (vec && cb + c0 + 4 <= P.q) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(irow + c0));
          acc[c0] = v.x;
          acc[c0 + 1] = v.y;
          acc[c0 + 2] = v.z;
          acc[c0 + 3] = v.w;
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (cb + c0 + i < P.q) acc[c0 + i] = irow[c0 + i];
        }
      }
    }
    // the next tile's rows of init: into L2 while this tile's chunks stream through
    if (P.init && tile + (int)gridDim.x < ntiles) {
      const int64_t nrow = row + (int64_t)gridDim.x * UTM;
      if (nrow < P.n) {
        const char* p = reinterpret_cast<const char*>(P.init + nrow * P.ldi + cb);
        for (int b = 0; b < NH * 4; b += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + b));
      }
    }
    for (int s = 0; s < P.nseg; ++s) {
      for (int c = 0; c < P.seg[s].chunks; ++c, ++j) {
        if (!P.gend[j]) continue;  // the group accumulates on in TMEM
        const int rg = G & 1;
        ut_wait(&rdone[rg], (G >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int c0 = 0; c0 < NH; c0 += 16) {
          if (cb + c0 < P.npad) {
            uint32_t r[16];
            const uint32_t taddr =
                tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(rg * P.npad + cb + c0);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, "
                "%10, %11, %12, %13, %14, %15}, [%16];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                  "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),
                  "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[c0 + i] += __uint_as_float(r[i]);
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        ut_arrive(&rfree[rg]);
        ++G;
      }
      if (P.argmin_labels && s == P.nseg - 1) {
        // k-means assignment: argmin over this warp's columns, then (EW = 2) over the
        // two column halves through shared memory, double-buffered by tile parity
        float best = INFINITY;
        int bj = 0;
#pragma unroll
        for (int i = 0; i < NH; ++i) {
          if (cb + i < P.q) {
            const float dist = fmaf(-2.0f, acc[i], P.argmin_bias[cb + i]);
            if (dist < best) {  // strict: lowest column on ties
              best = dist;
              bj = cb + i;
            }
          }
        }
        const int par = ((tile - (int)blockIdx.x) / (int)gridDim.x) & 1;
        const int half = (warp - 6) >> 2;
        int lab = bj;
        if (EW == 2) {
          akeys[(par * 2 + half) * UTM + quarter * 32 + lane] = ut_argkey(best, bj);
          asm volatile("bar.sync 1, %0;" ::"r"(32 * 4 * EW) : "memory");
          const unsigned long long k0 = akeys[(par * 2) * UTM + quarter * 32 + lane];
          const unsigned long long k1 = akeys[(par * 2 + 1) * UTM + quarter * 32 + lane];
          lab = (int)(uint32_t)(k0 <= k1 ? k0 : k1);
        }
        if (half == 0) {
          int moved = 0;
          if (row < P.n) {
            moved = P.argmin_labels[row] != lab;
            P.argmin_labels[row] = lab;
          }
          const unsigned m = __ballot_sync(0xffffffffu, moved);
          if (lane == 0 && m) atomicAdd(P.argmin_changed, (unsigned long long)__popc(m));
        }
      } else if (P.seg[s].emit && P.tma_store) {
        // 32-column slices of the 128-row tile: each thread writes its row into the
        // 128B-swizzled staging buffer (conflict-free), then one thread stores the slice
        // with a TMA tensor store (rows >= n and columns >= q are clipped by the map);
        // two buffers per column half, the previous store's smem read awaited by the
        // issuer before the barrier that releases the next writes
        const CUtensorMap* om = s == 0 ? &omap0 : (s == 1 ? &omap1 : &omap2);
        const int r = quarter * 32 + lane;
        const int ncol = P.q - cb;
#pragma unroll
        for (int c0 = 0; c0 < NH; c0 += 32) {
          if (c0 < ncol) {
            const uint32_t buf = ut_smem(base + P.stg_off) + (uint32_t)((half * 2 + (npass & 1)) * 16384);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const uint32_t a = buf + (uint32_t)(r * 128 + ((k ^ (r & 7)) << 4));
              asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(acc[c0 + 4 * k]),
                           "f"(acc[c0 + 4 * k + 1]), "f"(acc[c0 + 4 * k + 2]), "f"(acc[c0 + 4 * k + 3])
                           : "memory");
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (issuer) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            asm volatile("bar.sync %0, 128;" ::"r"(2 + half) : "memory");
            if (issuer) {
              asm volatile(
                  "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(om),
                  "r"(cb + c0), "r"(tile * UTM), "r"(buf)
                  : "memory");
              asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            ++npass;
          }
        }
      } else if (P.seg[s].emit && row < P.n) {
        float* orow = P.seg[s].out + row * P.seg[s].ldo + cb;
        const bool vec = (reinterpret_cast<uintptr_t>(orow) & 15) == 0;
#pragma unroll
        for (int c0 = 0; c0 < NH; c0 += 4) {
          if (vec && cb + c0 + 4 <= P.q)
            *reinterpret_cast<float4*>(orow + c0) =
                make_float4(acc[c0], acc[c0 + 1], acc[c0 + 2], acc[c0 + 3]);
          else
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (cb + c0 + i < P.q) orow[c0 + i] = acc[c0 + i];
        }
      }
    }
    }  // tile
    if (issuer && P.tma_store) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(P.tmem_cols));
  }
}

typedef CUresult (*UtEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                               const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                               const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

UtEncodeFn ut_encode() {
  static UtEncodeFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (UtEncodeFn)p;
  }
  return fn;
}

// {cols (K, inner) x rows} float32 view with row pitch ld, 32 x 128 boxes, 128B swizzle
bool ut_map(CUtensorMap* m, const void* ptr, int64_t rows, int cols, int64_t ld) {
  UtEncodeFn fn = ut_encode();
  if (!fn) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  const cuuint32_t box[2] = {(cuuint32_t)UTK, (cuuint32_t)UTM};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// {q (inner) x rows} float32 output view with row pitch ld: 32 x 128 boxes (one
// 128-byte swizzle span per row), the epilogue's staging layout
bool ut_map_out(CUtensorMap* m, const void* ptr, int64_t rows, int cols, int64_t ld) {
  UtEncodeFn fn = ut_encode();
  if (!fn) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  const cuuint32_t box[2] = {32u, (cuuint32_t)UTM};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

size_t update_tc_cstage_floats(int w_total, int nseg, int q) {
  const int npad = (q + 15) / 16 * 16;
  return (size_t)((w_total + UTK - 1) / UTK + nseg) * 2 * npad * UTK;
}

// Float32 block update on the tensor cores; returns false (nothing launched)
// when the shape is outside the kernel's envelope, so the caller falls back.
bool update_tc(const UpdParams& p, int64_t n, cudaStream_t st) {
  if (p.nseg < 1 || p.nseg > 3 || p.q < 1 || p.q > 256 || n < 1 || n > INT32_MAX) return false;
  const int npad = (p.q + 15) / 16 * 16;
  int nemit = 0, chunks = 0, wtot = 0;
  for (int s = 0; s < p.nseg; ++s) {
    const UpdSeg& g = p.seg[s];
    if (g.w < 1) return false;
    if ((reinterpret_cast<uintptr_t>(g.A) & 15) || (g.lda & 3)) return false;
    nemit += g.emit ? 1 : 0;
    chunks += (g.w + UTK - 1) / UTK;
    wtot += g.w;
  }
  if (nemit < 1 || !p.seg[p.nseg - 1].emit || npad > 192) return false;
  uint32_t cols = 32;
  while (cols < (uint32_t)(2 * npad)) cols <<= 1;
  const size_t need = (size_t)chunks * 2 * npad * UTK;
  if (!p.cstage || need > p.cstage_cap || need > update_tc_cstage_floats(wtot, p.nseg, p.q) ||
      (reinterpret_cast<uintptr_t>(p.cstage) & 15))
    return false;
  CUtensorMap maps[3], omaps[3];
  for (int s = 0; s < 3; ++s) {
    const UpdSeg& g = p.seg[s < p.nseg ? s : 0];
    if (!ut_map(&maps[s], g.A, n, g.w, g.lda)) return false;
  }
  // output maps for the TMA-store epilogue (emitting segments only)
  bool omaps_ok = true;
  for (int s = 0; s < 3; ++s) {
    const UpdSeg& g = p.seg[s < p.nseg ? s : p.nseg - 1];
    const UpdSeg& e = g.emit ? g : p.seg[p.nseg - 1];
    if ((reinterpret_cast<uintptr_t>(e.out) & 15) || (e.ldo & 3) ||
        !ut_map_out(&omaps[s], e.out, n, p.q, e.ldo))
      omaps_ok = false;
  }
  UtParams P{};
  for (int s = 0; s < p.nseg; ++s) {
    P.seg[s].chunks = (p.seg[s].w + UTK - 1) / UTK;
    P.seg[s].emit = p.seg[s].emit;
    P.seg[s].out = (float*)p.seg[s].out;
    P.seg[s].ldo = p.seg[s].ldo;
  }
  P.nseg = p.nseg;
  {
    int j = 0;
    for (int s = 0; s < p.nseg; ++s)
      for (int c = 0; c < P.seg[s].chunks; ++c, ++j) {
        P.gstart[j] = (c % kUtCpg) == 0;
        P.gend[j] = (c % kUtCpg) == kUtCpg - 1 || c == P.seg[s].chunks - 1;
      }
    if (j > 32) return false;
  }
  P.q = p.q;
  P.npad = npad;
  P.nemit = nemit;
  P.init = (const float*)p.init;
  P.ldi = p.ldi;
  P.coef = p.cstage;
  P.argmin_bias = p.argmin_bias;
  P.argmin_labels = p.argmin_labels;
  P.argmin_changed = p.argmin_changed;
  P.n = n;
  // A in tensor memory for 64 < npad <= 128 (C3's l = 108): 2 x npad accumulator
  // columns + 4 stages x 64 split-operand columns fit the 512 TMEM columns
  // (C3 update time 36.9 -> 34.1 ms per partition against the shared-memory A path)
  const bool atm = npad > 64 && npad <= 128;
  if (atm) cols = 512;
  P.tmem_cols = cols;
  const int kB = 2 * npad * UTK * 4;
  const size_t kStage = (atm ? 1 : 2) * kUtA + kB;
  // two stages when two CTAs fit per SM (one CTA's epilogue overlaps the other's
  // MMAs), else three
  constexpr size_t kExtra = 1024 + 256 + 4 * UTM * 8;  // alignment, barriers, argmin keys
  int stages = 2 * (2 * kStage + kExtra) <= 227 * 1024 ? 2 : 3;
  if ((size_t)stages * kStage + kExtra > 227 * 1024) stages = 2;
  if (atm) stages = 4;
  P.stages = stages;
  size_t smem = (size_t)stages * kStage + kExtra;
  // TMA-store epilogue when its staging ([EW][2][16 KB], 1 KB aligned) fits beside the
  // stages without costing a stage or a second CTA per SM: the C3 (A in TMEM) and
  // C4 (two epilogue warp groups) shapes; row-wise st.global of 448-704-byte rows
  // otherwise (one 16-byte piece of 32 rows per warp store: LSU-bound at tile ends)
  const int ew = npad > 128 ? 2 : 1;
  const size_t stg_off = round_up((size_t)stages * kStage + 256 + 4 * UTM * 8, 1024);
  const size_t smem_tma = stg_off + (size_t)ew * 2 * 16384 + 1024;
  if (omaps_ok && !p.argmin_labels && (atm || ew == 2) && smem_tma <= 227 * 1024) {
    P.tma_store = 1;
    P.stg_off = (uint32_t)stg_off;
    smem = std::max(smem, smem_tma);
  }
  static std::atomic<uint64_t> attr{0};
  if (!done_on_device(attr)) {
    cudaFuncSetAttribute(update_tc_kernel<64, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(update_tc_kernel<128, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(update_tc_kernel<192, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(update_tc_kernel<128, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    mark_on_device(attr);
  }
  if (smem > 227 * 1024) return false;
  tc_stage_coeffs<<<64, 256, 0, st>>>(p, npad, p.cstage);
  const int per_sm = !atm && 2 * (smem + 2048) <= 228 * 1024 ? 2 : 1;
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(n, UTM), (int64_t)per_sm * num_sms());
  if (atm)
    update_tc_kernel<128, 1, true><<<grid, kUtThreads, smem, st>>>(maps[0], maps[1], maps[2], omaps[0],
                                                                   omaps[1], omaps[2], P);
  else if (npad <= 64)
    update_tc_kernel<64, 1><<<grid, kUtThreads, smem, st>>>(maps[0], maps[1], maps[2], omaps[0],
                                                            omaps[1], omaps[2], P);
  else if (npad <= 128)
    update_tc_kernel<128, 1><<<grid, kUtThreads, smem, st>>>(maps[0], maps[1], maps[2], omaps[0],
                                                             omaps[1], omaps[2], P);
  else
    update_tc_kernel<192, 2><<<grid, kUtThreadsW, smem, st>>>(maps[0], maps[1], maps[2], omaps[0],
                                                              omaps[1], omaps[2], P);
  return true;
}

}  // namespace spb
