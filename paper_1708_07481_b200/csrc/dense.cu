// (c) Tall-skinny dense products of the LOBPCG body, CUDA-core path.
//
// * gram_batched  — G = U' V for a batch of column blocks (the Rayleigh-Ritz
//   Grams [X R P]'[LX LR LP] and [X R P]'[X R P] of lobpcg.py:418, the
//   projection X'R of :366 and the CholQR Gram of :228). Split-K over rows,
//   products and accumulation in float64 (fp32 inputs multiply exactly in
//   fp64), per-split partials reduced in a fixed order => deterministic.
// * block_update  — out = init + sum_s A_s C_s with emit points, row-local and
//   therefore safe in place: X' = [X R P] C and P' = [R P] C[l:] share one
//   accumulator (lobpcg.py:436-439), R -= X (X'R) (:366-369), R <- R inv (:237).
// * column_reduce — residual R = LX - X diag(theta) fused with its column norms
//   (lobpcg.py:338-341), plain column sums of squares (P norms :382) and sums
//   (mean removal :259-260); per-block partials, fixed-order final reduction.
// * gather / scale columns — soft-lock compaction (_move_columns :250-256) and
//   P normalisation (:391-393).
#include <cstdlib>

#include "dense.cuh"

namespace spb {
namespace {

constexpr int GT = 64;
constexpr int GK = 32;

// Gram on the FP64 tensor pipe: mma.sync m8n8k4 f64 (DMMA). 64x64 output tile
// per CTA, 4 warps as 2x2 of 32x32 (4x4 DMMA tiles each). Operands are widened
// to fp64 once, when a 32-row chunk is staged in shared memory (rows padded to
// 68 doubles so the four k-rows of a fragment load hit disjoint bank groups);
// the next chunk's global loads are in registers while the current one
// multiplies. fp32 inputs multiply exactly in fp64, so the result matches the
// CUDA-core path up to fp64 summation order.
constexpr int DK = 32;   // rows per staged chunk
constexpr int DLD = 68;  // padded row length (doubles)
constexpr size_t kDmmaSmem = sizeof(double) * 2 * 2 * DK * DLD;

template <typename T>
__global__ void __launch_bounds__(128, 3)
gram_dmma(GramBatch b, int64_t n, int64_t kchunk, int ldo, int64_t split_stride,
          double* __restrict__ part) {
  extern __shared__ double dsm[];
  double* Us = dsm;                 // [2][DK][DLD]
  double* Vs = dsm + 2 * DK * DLD;  // [2][DK][DLD]
  const int tile = blockIdx.x;
  int j = 0;
  while (j + 1 < b.njobs && tile >= b.tile_start[j + 1]) ++j;
  const GramJob jb = b.job[j];
  const int local = tile - b.tile_start[j];
  const int tq_count = (jb.q + GT - 1) / GT;
  const int tp = local / tq_count, tq = local % tq_count;
  const int p0 = tp * GT, q0 = tq * GT;
  const int64_t k0 = (int64_t)blockIdx.y * kchunk;
  const int64_t k1 = min(n, k0 + kchunk);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  const T* U = (const T*)jb.U;
  const T* V = (const T*)jb.V;
  constexpr int PER = DK * GT / 128;  // 16 per operand
  T ru[PER], rv[PER];
  const bool ufull = p0 + GT <= jb.p, vfull = q0 + GT <= jb.q;
  auto load = [&](int64_t kb) {
#pragma unroll
    for (int t = 0; t < PER; ++t) {
      const int e = tid + 128 * t;
      const int r = e / GT, c = e % GT;
      const int64_t k = kb + r;
      const bool kin = k < k1;
      ru[t] = (kin && (ufull || p0 + c < jb.p)) ? U[k * jb.ldu + p0 + c] : T(0);
      rv[t] = (kin && (vfull || q0 + c < jb.q)) ? V[k * jb.ldv + q0 + c] : T(0);
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int t = 0; t < PER; ++t) {
      const int e = tid + 128 * t;
      const int r = e / GT, c = e % GT;
      Us[(buf * DK + r) * DLD + c] = (double)ru[t];
      Vs[(buf * DK + r) * DLD + c] = (double)rv[t];
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;
  const int fr = lane & 3, fc = lane >> 2;  // fragment k-row, m/n index
  int buf = 0;
  if (k0 < k1) {
    load(k0);
    store(0);
  }
  __syncthreads();
  for (int64_t kb = k0; kb < k1; kb += DK) {
    const bool more = kb + DK < k1;
    if (more) load(kb + DK);
    const double* ub = Us + buf * DK * DLD + wm * 32 + fc;
    const double* vb = Vs + buf * DK * DLD + wn * 32 + fc;
#pragma unroll
    for (int k4 = 0; k4 < DK; k4 += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        af[t] = ub[(k4 + fr) * DLD + t * 8];
        bf[t] = vb[(k4 + fr) * DLD + t * 8];
      }
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
          asm volatile(
              "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
              : "+d"(acc[mt][nt][0]), "+d"(acc[mt][nt][1])
              : "d"(af[mt]), "d"(bf[nt]));
    }
    if (more) store(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
  double* out = part + (int64_t)blockIdx.y * split_stride;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int i = p0 + wm * 32 + mt * 8 + fc;
    if (i >= jb.p) continue;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = q0 + wn * 32 + nt * 8 + fr * 2 + h;
        if (c < jb.q) out[(int64_t)(jb.out_r + i) * ldo + jb.out_c + c] = acc[mt][nt][h];
      }
  }
}

// Same DMMA Gram with a configurable CTA tile, so the tile matches the block
// widths of the solver (l = 108 at C3 -> 112x112 tiles instead of 2x2 tiles of
// 64 = 1.4x wasted MMAs). Warp grid WM x WN, each warp
// MT x NT m8n8 tiles; DKT rows per staged chunk; row pitch TM+4 / TN+4 doubles
// (== 4 mod 16: the four k-rows of a fragment load hit disjoint bank groups).
template <typename T, int MT, int NT, int WM, int WN, int DKT>
__global__ void __launch_bounds__(32 * WM * WN)
gram_dmma_t(GramBatch b, int64_t n, int64_t kchunk, int ldo, int64_t split_stride,
            double* __restrict__ part) {
  constexpr int TM = WM * MT * 8, TN = WN * NT * 8, NTHR = 32 * WM * WN;
  constexpr int LDM = TM + 4, LDN = TN + 4;
  constexpr int PERU = (DKT * TM + NTHR - 1) / NTHR, PERV = (DKT * TN + NTHR - 1) / NTHR;
  extern __shared__ double dsm[];
  double* Us = dsm;                  // [2][DKT][LDM]
  double* Vs = dsm + 2 * DKT * LDM;  // [2][DKT][LDN]
  const int tile = blockIdx.x;
  int j = 0;
  while (j + 1 < b.njobs && tile >= b.tile_start[j + 1]) ++j;
  const GramJob jb = b.job[j];
  const int local = tile - b.tile_start[j];
  const int tq_count = (jb.q + TN - 1) / TN;
  const int tp = local / tq_count, tq = local % tq_count;
  const int p0 = tp * TM, q0 = tq * TN;
  const int64_t k0 = (int64_t)blockIdx.y * kchunk;
  const int64_t k1 = min(n, k0 + kchunk);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;
  const T* U = (const T*)jb.U;
  const T* V = (const T*)jb.V;
  T ru[PERU], rv[PERV];
  double acc[MT][NT][2];
#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int c = 0; c < NT; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;
  const int fr = lane & 3, fc = lane >> 2;
  int buf = 0;
#define SPB_GT_LOAD(KB)                                                                     \
  {                                                                                         \
    _Pragma("unroll") for (int t = 0; t < PERU; ++t) {                                      \
      const int e = tid + NTHR * t;                                                         \
      const int r = e / TM, c = e % TM;                                                     \
      const int64_t k = (KB) + r;                                                           \
      ru[t] = (e < DKT * TM && k < k1 && p0 + c < jb.p) ? U[k * jb.ldu + p0 + c] : T(0);     \
    }                                                                                       \
    _Pragma("unroll") for (int t = 0; t < PERV; ++t) {                                      \
      const int e = tid + NTHR * t;                                                         \
      const int r = e / TN, c = e % TN;                                                     \
      const int64_t k = (KB) + r;                                                           \
      rv[t] = (e < DKT * TN && k < k1 && q0 + c < jb.q) ? V[k * jb.ldv + q0 + c] : T(0);     \
    }                                                                                       \
  }
#define SPB_GT_STORE(BUF)                                                                   \
  {                                                                                         \
    _Pragma("unroll") for (int t = 0; t < PERU; ++t) {                                      \
      const int e = tid + NTHR * t;                                                         \
      if (e < DKT * TM) Us[((BUF) * DKT + e / TM) * LDM + e % TM] = (double)ru[t];           \
    }                                                                                       \
    _Pragma("unroll") for (int t = 0; t < PERV; ++t) {                                      \
      const int e = tid + NTHR * t;                                                         \
      if (e < DKT * TN) Vs[((BUF) * DKT + e / TN) * LDN + e % TN] = (double)rv[t];           \
    }                                                                                       \
  }
  if (k0 < k1) {
    SPB_GT_LOAD(k0);
    SPB_GT_STORE(0);
  }
  __syncthreads();
  for (int64_t kb = k0; kb < k1; kb += DKT) {
    const bool more = kb + DKT < k1;
    if (more) SPB_GT_LOAD(kb + DKT);
    const double* ub = Us + buf * DKT * LDM + wm * (MT * 8) + fc;
    const double* vb = Vs + buf * DKT * LDN + wn * (NT * 8) + fc;
#pragma unroll
    for (int k4 = 0; k4 < DKT; k4 += 4) {
      double af[MT], bf[NT];
#pragma unroll
      for (int t = 0; t < MT; ++t) af[t] = ub[(k4 + fr) * LDM + t * 8];
#pragma unroll
      for (int t = 0; t < NT; ++t) bf[t] = vb[(k4 + fr) * LDN + t * 8];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
          asm volatile(
              "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
              : "+d"(acc[mt][nt][0]), "+d"(acc[mt][nt][1])
              : "d"(af[mt]), "d"(bf[nt]));
    }
    if (more) SPB_GT_STORE(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
  double* out = part + (int64_t)blockIdx.y * split_stride;
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int i = p0 + wm * (MT * 8) + mt * 8 + fc;
    if (i >= jb.p) continue;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = q0 + wn * (NT * 8) + nt * 8 + fr * 2 + h;
        if (c < jb.q) out[(int64_t)(jb.out_r + i) * ldo + jb.out_c + c] = acc[mt][nt][h];
      }
  }
#undef SPB_GT_LOAD
#undef SPB_GT_STORE
}

// Launch one tile configuration: recompute the batch's tile starts for its
// tile shape and pick the split-K so tiles * ks fills the GPU.
template <typename T, int MT, int NT, int WM, int WN, int DKT>
int launch_gram_cfg(GramBatch bb, int64_t n, int out_rows, int out_cols, double* partial,
                    size_t partial_cap, int ctas_per_sm, int* ks_out, cudaStream_t st) {
  constexpr int TM = WM * MT * 8, TN = WN * NT * 8, NTHR = 32 * WM * WN;
  constexpr size_t smem = sizeof(double) * 2 * DKT * ((size_t)(TM + 4) + (TN + 4));
  int tiles = 0;
  for (int j = 0; j < bb.njobs; ++j) {
    bb.tile_start[j] = tiles;
    tiles += (int)(ceil_div(bb.job[j].p, TM) * ceil_div(bb.job[j].q, TN));
  }
  bb.tile_start[bb.njobs] = tiles;
  int64_t ks = std::max<int64_t>(1, (int64_t)ctas_per_sm * num_sms() / std::max(tiles, 1));
  constexpr int minrows = 128;  // rows per split at least
  ks = std::min<int64_t>(ks, ceil_div(n, minrows));
  ks = std::max<int64_t>(ks, 1);
  while (ks > 1 && (size_t)ks * out_rows * out_cols > partial_cap) --ks;
  if ((size_t)ks * out_rows * out_cols > partial_cap) {
    set_error("gram partial workspace too small");
    return SPB_ERR_WORKSPACE;
  }
  const int64_t kchunk = round_up(ceil_div(std::max<int64_t>(n, 1), ks), DKT);
  static std::atomic<uint64_t> attr{0};
  if (!done_on_device(attr)) {
    SPB_CUDA(cudaFuncSetAttribute(gram_dmma_t<T, MT, NT, WM, WN, DKT>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    mark_on_device(attr);
  }
  dim3 grid(tiles, (unsigned)ks);
  gram_dmma_t<T, MT, NT, WM, WN, DKT><<<grid, NTHR, smem, st>>>(
      bb, n, kchunk, out_cols, (int64_t)out_rows * out_cols, partial);
  SPB_LAUNCH_CHECK();
  *ks_out = (int)ks;
  return SPB_OK;
}

// Tile shape for a batch: 112 x 112 when every job is 65..112 wide (C3's
// l = 108 blocks: 1.075x padding instead of 1.4x with 64-tiles), else 64.
// (A 176-wide tile for C4 needs more accumulator registers than a warp grid
// of <= 32 warps can hold; 64-tiles pad 176 -> 192, 1.19x.)
int gram_tile_for(const GramBatch& b) {
  int wmin = 1 << 30, wmax = 0;
  for (int j = 0; j < b.njobs; ++j) {
    wmax = std::max(wmax, std::max(b.job[j].p, b.job[j].q));
    wmin = std::min(wmin, std::max(b.job[j].p, b.job[j].q));
  }
  if (wmax > 64 && wmax <= 112 && wmin > 64) return 112;
  // C4's l = 176 blocks: 2 x 2 tiles of 88 pad nothing (64-tiles: 192 = 1.19x)
  if (wmax > 112 && wmax <= 176 && wmin > 88) return 88;
  // C2's l = 49 blocks: 56 x 56 tiles pad 1.31x instead of 1.71x with 64-tiles
  if (wmax > 32 && wmax <= 56) return 56;
  return 64;
}

// Fixed-order reduction of the split-K partials: a CTA owns 32 consecutive
// outputs (one per lane, coalesced); its 8 warps each sum a contiguous range of
// splits and the 8 warp sums are added in warp order (deterministic).
__global__ void __launch_bounds__(256)
sum_splits(const double* __restrict__ part, int ksplit, int64_t split_stride, int rows, int cols,
           int ldp, double* __restrict__ out, int ldo) {
  __shared__ double ws[8][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t total = (int64_t)rows * cols;
  const int kc = (ksplit + 7) / 8;
  const int k0 = warp * kc, k1 = min(ksplit, k0 + kc);
  for (int64_t base = (int64_t)blockIdx.x * 32; base < total; base += (int64_t)gridDim.x * 32) {
    const int64_t e = base + lane;
    double s = 0.0;
    if (e < total) {
      const int r = (int)(e / cols), c = (int)(e % cols);
      const double* p = part + (int64_t)r * ldp + c;
#pragma unroll 4
      for (int k = k0; k < k1; ++k) s += p[(int64_t)k * split_stride];
    }
    ws[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && e < total) {
      double t = ws[0][lane];
#pragma unroll
      for (int w = 1; w < 8; ++w) t += ws[w][lane];
      const int r = (int)(e / cols), c = (int)(e % cols);
      out[(int64_t)r * ldo + c] = t;
    }
    __syncthreads();
  }
}

int sum_splits_grid(int64_t total) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 32), (int64_t)num_sms() * 16));
}

int choose_ksplit(int64_t n, int tiles) {
  // one full wave of the DMMA Gram (3 CTAs per SM): tiles * ks <= 3 * SMs; the
  // per-SM work is the same for fewer, longer splits, but the fixed-order
  // reduction reads ks partial tiles (2 and 4 CTAs per SM measured slower)
  const int target = 3 * num_sms();
  int64_t ks = std::max<int64_t>(1, target / std::max(tiles, 1));
  constexpr int minrows = 128;  // rows per split at least
  ks = std::min<int64_t>(ks, ceil_div(n, minrows));
  return (int)std::max<int64_t>(ks, 1);
}

// ----------------------------------------------------------------------------
// Block update: (8 * RPT) rows x q columns per CTA (q <= 32 * QV <= 256);
// 256 threads as 8 row groups x 32 column lanes, each thread RPT rows x QV
// columns (templated so no predicated-off FMAs are issued).
constexpr int UQ = 256;  // max columns

template <typename T, int QV, int RPT>
__global__ void __launch_bounds__(256)
update_kernel(UpdParams P, int64_t n) {
  constexpr int UR = 8 * RPT;
  constexpr int UK = sizeof(T) == 4 ? 32 : 16;  // k chunk (static smem <= 48 KB)
  __shared__ T As[UK][UR + 1];                  // k-major: As[k][row]
  __shared__ T Cs[UK][32 * QV];
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * UR;
  const int q = P.q;
  T acc[RPT][QV];
#pragma unroll
  for (int a = 0; a < RPT; ++a)
#pragma unroll
    for (int c = 0; c < QV; ++c) {
      T v = T(0);
      const int64_t r = r0 + ty * RPT + a;
      const int col = tx + 32 * c;
      if (P.init && col < q && r < n) v = ((const T*)P.init)[r * P.ldi + col];
      acc[a][c] = v;
    }
  for (int s = 0; s < P.nseg; ++s) {
    const UpdSeg sg = P.seg[s];
    const T* A = (const T*)sg.A;
    for (int k0 = 0; k0 < sg.w; k0 += UK) {
      const int kc = min(UK, sg.w - k0);
      for (int e = tid; e < UR * UK; e += 256) {
        const int r = e / UK, k = e % UK;
        const int64_t gr = r0 + r;
        As[k][r] = (gr < n && k < kc) ? A[gr * sg.lda + k0 + k] : T(0);
      }
      for (int e = tid; e < UK * 32 * QV; e += 256) {
        const int k = e / (32 * QV), c = e % (32 * QV);
        Cs[k][c] = (k < kc && c < q) ? (T)(sg.scale * sg.C[(int64_t)(k0 + k) * sg.ldc + c]) : T(0);
      }
      __syncthreads();
#pragma unroll 4
      for (int k = 0; k < kc; ++k) {
        T a[RPT], cv[QV];
#pragma unroll
        for (int i = 0; i < RPT; ++i) a[i] = As[k][ty * RPT + i];
#pragma unroll
        for (int c = 0; c < QV; ++c) cv[c] = Cs[k][tx + 32 * c];
#pragma unroll
        for (int i = 0; i < RPT; ++i)
#pragma unroll
          for (int c = 0; c < QV; ++c) acc[i][c] = fma(a[i], cv[c], acc[i][c]);
      }
      __syncthreads();
    }
    if (sg.emit) {
      T* O = (T*)sg.out;
#pragma unroll
      for (int a = 0; a < RPT; ++a) {
        const int64_t r = r0 + ty * RPT + a;
        if (r >= n) continue;
#pragma unroll
        for (int c = 0; c < QV; ++c) {
          const int col = tx + 32 * c;
          if (col < q) O[r * sg.ldo + col] = acc[a][c];
        }
      }
    }
  }
}

// fp32 block update with an 8x8 register tile per thread: CTA = RG row groups x
// NCG column groups (8 rows interleaved by RG, 8 contiguous columns each), so a
// k-step costs 2.5 shared float4 loads per 64 FMAs. The coefficients are first
// rounded to fp32 (exactly as update_kernel does) into a staging buffer laid out
// per 16-row k tile as [k][half][column group][4], so both operands arrive by
// cp.async (A zero-filled past n / w) through a 3-stage pipeline with one
// barrier per tile and the column-group reads are bank-conflict free. The
// per-element FMA order is update_kernel's, so results are identical.
constexpr int UKT = 16;       // k per stage
constexpr int UAP = UKT + 4;  // padded A row (floats)
constexpr int UNS = 3;        // pipeline stages

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

int update_cols(int q) { return q <= 32 ? 32 : q <= 64 ? 64 : q <= 128 ? 128 : q <= 192 ? 192 : 256; }

// cst[s] = fp32(scale_s * C_s) in the tile layout above, zero padded.
__global__ void stage_coeffs(UpdParams P, int cols) {
  const int ncg = cols / 8;
  int off = 0;
  for (int s = 0; s < P.nseg; ++s) {
    const UpdSeg sg = P.seg[s];
    const int wr = (int)round_up(sg.w, UKT);
    float* dst = P.cstage + off;
    const int total = wr * cols;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
      const int k = e / cols, r = e % cols;
      const int h = r / (4 * ncg), cg = (r / 4) % ncg, x = r % 4;
      const int c = cg * 8 + h * 4 + x;
      float v = 0.0f;
      if (k < sg.w && c < P.q) v = (float)(sg.scale * sg.C[(int64_t)k * sg.ldc + c]);
      dst[e] = v;
    }
    off += total;
  }
}

template <int NCG, int RG>
__global__ void __launch_bounds__(NCG * RG, NCG * RG <= 128 ? 4 : 2)
update_f32(UpdParams P, int64_t n) {
  constexpr int NT = NCG * RG, ROWS = RG * 8, COLS = NCG * 8;
  extern __shared__ __align__(16) float usm[];
  float* As = usm;                          // [UNS][ROWS][UAP]
  float* Cs = usm + UNS * ROWS * UAP;       // [UNS][UKT][COLS]
  const int tid = threadIdx.x, cg = tid % NCG, rg = tid / NCG;
  const int64_t r0 = (int64_t)blockIdx.x * ROWS;
  const int q = P.q;
  const int c0 = cg * 8;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t r = r0 + rg + RG * i;
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const int col = c0 + jj;
      acc[i][jj] = (P.init && col < q && r < n) ? ((const float*)P.init)[r * P.ldi + col] : 0.0f;
    }
  }
  int coff = 0;
  for (int s = 0; s < P.nseg; ++s) {
    const UpdSeg sg = P.seg[s];
    const float* A = (const float*)sg.A;
    const float* Cg = P.cstage + coff;
    const int ntiles = (sg.w + UKT - 1) / UKT;
    coff += ntiles * UKT * COLS;
    auto stage = [&](int t) {
      if (t < ntiles) {
        const int buf = t % UNS;
        const int k0 = t * UKT;
        for (int e = tid; e < ROWS * (UKT / 4); e += NT) {
          const int r = e / (UKT / 4), ch = e % (UKT / 4);
          const int64_t gr = r0 + r;
          const int k = k0 + ch * 4;
          int bytes = 0;
          if (gr < n && k < sg.w) bytes = min(4, sg.w - k) * 4;
          const float* src = bytes ? A + gr * sg.lda + k : A;
          cp_async16(As + (buf * ROWS + r) * UAP + ch * 4, src, bytes);
        }
        const float* cs = Cg + (size_t)t * UKT * COLS;
        for (int e = tid; e < UKT * COLS / 4; e += NT)
          cp_async16(Cs + buf * UKT * COLS + e * 4, cs + e * 4, 16);
      }
      cp_async_commit();
    };
    for (int t = 0; t < UNS - 1; ++t) stage(t);
    for (int t = 0; t < ntiles; ++t) {
      cp_async_wait<UNS - 2>();
      __syncthreads();
      stage(t + UNS - 1);
      const int buf = t % UNS;
      const float* Ab = As + buf * ROWS * UAP;
      const float* Cb = Cs + buf * UKT * COLS;
#pragma unroll
      for (int kk = 0; kk < UKT; kk += 4) {
        float4 a4[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) a4[i] = *reinterpret_cast<const float4*>(Ab + (rg + RG * i) * UAP + kk);
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) {
          const float4 cA = *reinterpret_cast<const float4*>(Cb + (kk + k4) * COLS + cg * 4);
          const float4 cB = *reinterpret_cast<const float4*>(Cb + (kk + k4) * COLS + (NCG + cg) * 4);
          const float cv[8] = {cA.x, cA.y, cA.z, cA.w, cB.x, cB.y, cB.z, cB.w};
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float a = k4 == 0 ? a4[i].x : (k4 == 1 ? a4[i].y : (k4 == 2 ? a4[i].z : a4[i].w));
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) acc[i][jj] = fmaf(a, cv[jj], acc[i][jj]);
          }
        }
      }
    }
    cp_async_wait<0>();
    __syncthreads();  // buffers free before the next segment's prologue
    if (sg.emit) {
      float* O = (float*)sg.out;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t r = r0 + rg + RG * i;
        if (r >= n) continue;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const int col = c0 + jj;
          if (col < q) O[r * sg.ldo + col] = acc[i][jj];
        }
      }
    }
  }
}

template <int NCG, int RG>
void launch_update_f32(const UpdParams& p, int64_t n, cudaStream_t st) {
  constexpr int ROWS = RG * 8, COLS = NCG * 8;
  const size_t smem = sizeof(float) * (UNS * ROWS * UAP + UNS * UKT * COLS);
  static std::atomic<uint64_t> attr{0};
  if (!done_on_device(attr)) {
    cudaFuncSetAttribute(update_f32<NCG, RG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    mark_on_device(attr);
  }
  stage_coeffs<<<32, 256, 0, st>>>(p, COLS);
  update_f32<NCG, RG><<<(unsigned)ceil_div(n, ROWS), NCG * RG, smem, st>>>(p, n);
}

bool update_f32_ok(const UpdParams& p) {
  if (!p.cstage) return false;
  size_t need = 0;
  for (int s = 0; s < p.nseg; ++s) {
    const UpdSeg& g = p.seg[s];
    if ((reinterpret_cast<uintptr_t>(g.A) & 15) || (g.lda & 3)) return false;
    need += (size_t)round_up(g.w, UKT) * update_cols(p.q);
  }
  return need <= p.cstage_cap && (reinterpret_cast<uintptr_t>(p.cstage) & 15) == 0;
}

template <typename T, int QV>
void launch_update_qv(const UpdParams& p, int64_t n, cudaStream_t st) {
  constexpr int RPT = QV <= 2 ? 8 : (QV <= 4 ? 4 : 2);
  const int64_t blocks = ceil_div(n, 8 * RPT);
  update_kernel<T, QV, RPT><<<blocks, 256, 0, st>>>(p, n);
}

static int g_update_mode = -1;  // spb_block_update's override (-1: default)

template <typename T>
void launch_update(const UpdParams& p, int64_t n, cudaStream_t st) {
  // float32: 3xTF32 on the tensor cores (update_tc.cu) unless spb_block_update
  // asked for the FMA kernel (mode 0)
  const bool tc = g_update_mode != 0;
  if (sizeof(T) == 4 && tc && update_tc(p, n, st)) return;
  // (narrow blocks, q <= 64 at C1/C2: the generic kernel below measured faster than
  // update_f32's 8-row-group variants)
  if (sizeof(T) == 4 && p.q > 64 && update_f32_ok(p)) {
    if (p.q <= 128) launch_update_f32<16, 8>(p, n, st);
    else if (p.q <= 192) launch_update_f32<24, 8>(p, n, st);
    else launch_update_f32<32, 8>(p, n, st);
    return;
  }
  const int qv = (p.q + 31) / 32;
  switch (qv) {
    case 1: launch_update_qv<T, 1>(p, n, st); break;
    case 2: launch_update_qv<T, 2>(p, n, st); break;
    case 3: launch_update_qv<T, 3>(p, n, st); break;
    case 4: launch_update_qv<T, 4>(p, n, st); break;
    case 5: launch_update_qv<T, 5>(p, n, st); break;
    case 6: launch_update_qv<T, 6>(p, n, st); break;
    default: launch_update_qv<T, 8>(p, n, st); break;
  }
}

// ----------------------------------------------------------------------------
// Column reductions: each CTA covers a contiguous row range; thread layout
// (ry, cx) with cx over columns (warp-coalesced along a row), ry over rows.
constexpr int CRB = 256;

template <typename T>
__global__ void __launch_bounds__(CRB)
colreduce_kernel(int kind, const T* __restrict__ A, int64_t lda, int cols, int64_t n,
                 int64_t rows_per_block, const T* __restrict__ X, int64_t ldx,
                 const double* __restrict__ theta, T* __restrict__ R, int64_t ldr,
                 double* __restrict__ part) {
  extern __shared__ double sred[];  // [ry][cw]
  const int cw = min(((cols + 31) / 32) * 32, CRB);
  const int nry = CRB / cw;
  const int tid = threadIdx.x;
  const int cx = tid % cw, ry = tid / cw;
  const int64_t rb = (int64_t)blockIdx.x * rows_per_block;
  const int64_t re = min(n, rb + rows_per_block);
  for (int c0 = 0; c0 < cols; c0 += cw) {
    const int c = c0 + cx;
    double s = 0.0;
    if (ry < nry && c < cols) {
      T th = T(0);
      if (kind == CR_RESIDUAL) th = (T)theta[c];
#pragma unroll 4
      for (int64_t r = rb + ry; r < re; r += nry) {
        T v = A[r * lda + c];
        if (kind == CR_RESIDUAL) {
          v = v - X[r * ldx + c] * th;
          R[r * ldr + c] = v;
        }
        const double dv = (double)v;
        s += (kind == CR_SUM) ? dv : dv * dv;
      }
    }
    if (ry < nry) sred[ry * cw + cx] = s;
    __syncthreads();
    if (ry == 0 && c < cols) {
      double t = 0.0;
      for (int y = 0; y < nry; ++y) t += sred[y * cw + cx];
      part[(int64_t)blockIdx.x * cols + c] = t;
    }
    __syncthreads();
  }
}

// float32, 16-byte rows: the same reduction with float4 loads (a thread owns four
// adjacent columns; 256 / ceil(cols/4 -> 32) row groups per CTA), for the wide blocks
// of C3 / C4 where the scalar kernel had too few bytes in flight for HBM.
__global__ void __launch_bounds__(256)
colreduce4_kernel(int kind, const float* __restrict__ A, int64_t lda, int cols, int64_t n,
                  int64_t rows_per_block, const float* __restrict__ X, int64_t ldx,
                  const double* __restrict__ theta, float* __restrict__ R, int64_t ldr,
                  double* __restrict__ part) {
  extern __shared__ double sred[];  // [ry][cw * 4]
  const int c4 = (cols + 3) / 4;
  const int cw = ((c4 + 31) / 32) * 32;  // <= 256 (cols <= 1024)
  const int nry = 256 / cw;
  const int tid = threadIdx.x;
  const int cx = tid % cw, ry = tid / cw;
  const int c = cx * 4;
  const int64_t rb = (int64_t)blockIdx.x * rows_per_block;
  const int64_t re = min(n, rb + rows_per_block);
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if (ry < nry && c < cols) {
    float t0 = 0.f, t1 = 0.f, t2 = 0.f, t3 = 0.f;
    if (kind == CR_RESIDUAL) {
      t0 = (float)theta[c];
      t1 = c + 1 < cols ? (float)theta[c + 1] : 0.f;
      t2 = c + 2 < cols ? (float)theta[c + 2] : 0.f;
      t3 = c + 3 < cols ? (float)theta[c + 3] : 0.f;
    }
#pragma unroll 4
    for (int64_t r = rb + ry; r < re; r += nry) {
      float4 v = *reinterpret_cast<const float4*>(A + r * lda + c);
      if (kind == CR_RESIDUAL) {
        const float4 x = *reinterpret_cast<const float4*>(X + r * ldx + c);
        v.x = v.x - x.x * t0;
        v.y = v.y - x.y * t1;
        v.z = v.z - x.z * t2;
        v.w = v.w - x.w * t3;
        *reinterpret_cast<float4*>(R + r * ldr + c) = v;
      }
      if (kind == CR_SUM) {
        s0 += (double)v.x; s1 += (double)v.y; s2 += (double)v.z; s3 += (double)v.w;
      } else {
        s0 += (double)v.x * v.x; s1 += (double)v.y * v.y; s2 += (double)v.z * v.z; s3 += (double)v.w * v.w;
      }
    }
  }
  if (ry < nry) {
    double* q = sred + (ry * cw + cx) * 4;
    q[0] = s0; q[1] = s1; q[2] = s2; q[3] = s3;
  }
  __syncthreads();
  for (int cc = tid; cc < cols; cc += 256) {
    double t = 0.0;
    for (int y = 0; y < nry; ++y) t += sred[(y * cw + cc / 4) * 4 + (cc & 3)];
    part[(int64_t)blockIdx.x * cols + cc] = t;
  }
}

// float32 column scaling with float4 rows (no 64-bit division per element).
__global__ void scale_cols4_kernel(float* __restrict__ A, int64_t lda, int n, const double* __restrict__ s,
                                   int count) {
  const int c4 = (count + 3) / 4;
  const int total = n * c4;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int r = e / c4, c = (e - r * c4) * 4;
    float4* p = reinterpret_cast<float4*>(A + (int64_t)r * lda + c);
    float4 v = *p;
    v.x = (float)((double)v.x * s[c]);
    if (c + 1 < count) v.y = (float)((double)v.y * s[c + 1]);
    if (c + 2 < count) v.z = (float)((double)v.z * s[c + 2]);
    if (c + 3 < count) v.w = (float)((double)v.w * s[c + 3]);
    *p = v;
  }
}

// One warp per column: lane-strided partial sums then a fixed shuffle tree
// (deterministic: same order every call).
__global__ void colreduce_final(const double* __restrict__ part, int blocks, int cols,
                                double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= cols) return;
  double s = 0.0;
  for (int b = lane; b < blocks; b += 32) s += part[(int64_t)b * cols + c];
  s = warp_sum(s);
  if (lane == 0) out[c] = s;
}

int colreduce_blocks(int64_t n) {
  // 8 CTAs of 256 threads per SM: enough loads in flight for HBM bandwidth
  return (int)std::max<int64_t>(1, std::min<int64_t>(8 * num_sms(), ceil_div(n, 64)));
}

// ----------------------------------------------------------------------------
template <typename T>
__global__ void gather_cols_kernel(T* __restrict__ A, int64_t lda, int64_t n,
                                   const int* __restrict__ idx, int count) {
  // one warp per row: read all selected values, then write (left-moving, in place)
  const int lane = threadIdx.x & 31;
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (row >= n) return;
  T* a = A + row * lda;
  T v[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int j = lane + 32 * t;
    v[t] = j < count ? a[idx[j]] : T(0);
  }
  __syncwarp();
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int j = lane + 32 * t;
    if (j < count) a[j] = v[t];
  }
}

template <typename T>
__global__ void scale_cols_kernel(T* __restrict__ A, int64_t lda, int64_t n,
                                  const double* __restrict__ s, int count) {
  const int64_t total = n * count;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / count;
    const int c = (int)(e - r * count);
    A[r * lda + c] = (T)((double)A[r * lda + c] * s[c]);
  }
}

template <typename T>
__global__ void sub_means_kernel(T* __restrict__ A, int64_t lda, int64_t n, int cols,
                                 const double* __restrict__ sums, double ndiv) {
  const int64_t total = n * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols;
    const int c = (int)(e - r * cols);
    A[r * lda + c] = (T)((double)A[r * lda + c] - sums[c] / ndiv);
  }
}

int grid_1d(int64_t total) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), (int64_t)num_sms() * 8));
}

}  // namespace

size_t gram_partial_doubles(int64_t n, int tiles, int out_rows, int out_cols, int* ksplit_out) {
  int ks = choose_ksplit(n, tiles);
  if (ksplit_out) *ksplit_out = ks;
  return (size_t)ks * out_rows * out_cols;
}

int gram_batched(int dtype, const GramBatch& b, int64_t n, int out_rows, int out_cols,
                 double* partial, size_t partial_cap, double* out, int ldo, cudaStream_t st) {
  const int tiles = b.tile_start[b.njobs];
  if (tiles == 0) return SPB_OK;
  int ks = choose_ksplit(n, tiles);
  while (ks > 1 && (size_t)ks * out_rows * out_cols > partial_cap) --ks;
  if ((size_t)ks * out_rows * out_cols > partial_cap) {
    set_error("gram partial workspace too small");
    return SPB_ERR_WORKSPACE;
  }
  const int64_t kchunk = round_up(ceil_div(std::max<int64_t>(n, 1), ks), GK);
  const int64_t stride = (int64_t)out_rows * out_cols;
  dim3 grid(tiles, ks);
  if (n > 0 && gram_tile_for(b) == 56) {
    // 56 x 56: 7 warps of 8 x 56 (1 x 7 m8n8 tiles each), two CTAs per SM in the split
    constexpr int cps = 2;
    const int rc =
        dtype == SPB_F32
            ? launch_gram_cfg<float, 1, 7, 7, 1, 32>(b, n, out_rows, out_cols, partial, partial_cap,
                                                     cps, &ks, st)
            : launch_gram_cfg<double, 1, 7, 7, 1, 32>(b, n, out_rows, out_cols, partial, partial_cap,
                                                      cps, &ks, st);
    if (rc != SPB_OK) return rc;
  } else if (n > 0 && gram_tile_for(b) == 88) {
    // 88 x 88: 11 warps of 8 x 88 (1 x 11 m8n8 tiles each)
    const int rc =
        dtype == SPB_F32
            ? launch_gram_cfg<float, 1, 11, 11, 1, 32>(b, n, out_rows, out_cols, partial, partial_cap,
                                                       1, &ks, st)
            : launch_gram_cfg<double, 1, 11, 11, 1, 32>(b, n, out_rows, out_cols, partial,
                                                        partial_cap, 1, &ks, st);
    if (rc != SPB_OK) return rc;
  } else if (n > 0 && gram_tile_for(b) != 64) {
    // 112 x 112: 7 x 2 warps of 16 x 56 (2 x 7 m8n8 tiles each)
    const int rc =
        dtype == SPB_F32
            ? launch_gram_cfg<float, 2, 7, 7, 2, 16>(b, n, out_rows, out_cols, partial, partial_cap, 1,
                                                     &ks, st)
            : launch_gram_cfg<double, 2, 7, 7, 2, 16>(b, n, out_rows, out_cols, partial, partial_cap,
                                                      1, &ks, st);
    if (rc != SPB_OK) return rc;
  } else if (n > 0) {
    static std::atomic<uint64_t> attr{0};
    if (!done_on_device(attr)) {
      SPB_CUDA(cudaFuncSetAttribute(gram_dmma<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)kDmmaSmem));
      SPB_CUDA(cudaFuncSetAttribute(gram_dmma<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)kDmmaSmem));
      mark_on_device(attr);
    }
    if (dtype == SPB_F32)
      gram_dmma<float><<<grid, 128, kDmmaSmem, st>>>(b, n, kchunk, out_cols, stride, partial);
    else
      gram_dmma<double><<<grid, 128, kDmmaSmem, st>>>(b, n, kchunk, out_cols, stride, partial);
    SPB_LAUNCH_CHECK();
  } else {
    SPB_CUDA(cudaMemsetAsync(partial, 0, sizeof(double) * stride, st));
    ks = 1;
  }
  sum_splits<<<sum_splits_grid(stride), 256, 0, st>>>(partial, ks, stride, out_rows, out_cols,
                                                        out_cols, out, ldo);
  SPB_LAUNCH_CHECK();
  return SPB_OK;
}

int block_update(int dtype, const UpdParams& p, int64_t n, cudaStream_t st) {
  if (p.q > UQ) {
    set_error("block update supports at most %d columns (got %d)", UQ, p.q);
    return SPB_ERR_CONTRACT;
  }
  if (n <= 0 || p.q <= 0) return SPB_OK;
  if (dtype == SPB_F32)
    launch_update<float>(p, n, st);
  else
    launch_update<double>(p, n, st);
  SPB_LAUNCH_CHECK();
  return SPB_OK;
}

int oz_sum_splits(const double* part, int ks, int64_t stride, int rows, int cols, double* out,
                  int ldo, cudaStream_t st) {
  sum_splits<<<sum_splits_grid(stride), 256, 0, st>>>(part, ks, stride, rows, cols, cols, out, ldo);
  SPB_LAUNCH_CHECK();
  return SPB_OK;
}

size_t update_cstage_floats(int w_total, int nseg) {
  return std::max((size_t)(w_total + nseg * UKT) * 256, update_tc_cstage_floats(w_total, nseg, 256));
}

size_t colreduce_partial_doubles(int64_t n, int cols) {
  return (size_t)colreduce_blocks(n) * std::max(cols, 1);
}

int column_reduce(int dtype, int kind, const void* A, int64_t lda, int cols, int64_t n,
                  const void* X, int64_t ldx, const double* theta, void* R, int64_t ldr,
                  double* partial, double* out, cudaStream_t st) {
  if (cols <= 0) return SPB_OK;
  const int blocks = colreduce_blocks(n);
  const int64_t rpb = ceil_div(std::max<int64_t>(n, 1), blocks);
  const size_t smem = sizeof(double) * CRB;
  const bool v4 = dtype == SPB_F32 && cols >= 64 && cols <= 1024 && (lda & 3) == 0 &&
                  (reinterpret_cast<uintptr_t>(A) & 15) == 0 &&
                  (kind != CR_RESIDUAL || ((ldx & 3) == 0 && (ldr & 3) == 0 &&
                                           (reinterpret_cast<uintptr_t>(X) & 15) == 0 &&
                                           (reinterpret_cast<uintptr_t>(R) & 15) == 0));
  if (v4)
    colreduce4_kernel<<<blocks, 256, sizeof(double) * 256 * 4, st>>>(
        kind, (const float*)A, lda, cols, n, rpb, (const float*)X, ldx, theta, (float*)R, ldr,
        partial);
  else if (dtype == SPB_F32)
    colreduce_kernel<float><<<blocks, CRB, smem, st>>>(kind, (const float*)A, lda, cols, n, rpb,
                                                       (const float*)X, ldx, theta, (float*)R,
                                                       ldr, partial);
  else
    colreduce_kernel<double><<<blocks, CRB, smem, st>>>(kind, (const double*)A, lda, cols, n,
                                                        rpb, (const double*)X, ldx, theta,
                                                        (double*)R, ldr, partial);
  colreduce_final<<<(int)ceil_div((int64_t)cols * 32, 256), 256, 0, st>>>(partial, blocks, cols, out);
  SPB_LAUNCH_CHECK();
  return SPB_OK;
}

int gather_columns(int dtype, void* A, int64_t lda, int64_t n, const int* idx, int count,
                   cudaStream_t st) {
  if (count > 256) {
    set_error("column gather supports at most 256 columns");
    return SPB_ERR_CONTRACT;
  }
  if (n <= 0 || count <= 0) return SPB_OK;
  const int64_t blocks = ceil_div(n * 32, 256);
  if (dtype == SPB_F32)
    gather_cols_kernel<float><<<blocks, 256, 0, st>>>((float*)A, lda, n, idx, count);
  else
    gather_cols_kernel<double><<<blocks, 256, 0, st>>>((double*)A, lda, n, idx, count);
  SPB_LAUNCH_CHECK();
  return SPB_OK;
}

int scale_columns(int dtype, void* A, int64_t lda, int64_t n, const double* s, int count,
                  cudaStream_t st) {
  if (n <= 0 || count <= 0) return SPB_OK;
  if (dtype == SPB_F32 && (lda & 3) == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0 &&
      n * ((count + 3) / 4) < INT32_MAX)
    scale_cols4_kernel<<<grid_1d(n * ((count + 3) / 4)), 256, 0, st>>>((float*)A, lda, (int)n, s,
                                                                          count);
  else if (dtype == SPB_F32)
    scale_cols_kernel<float><<<grid_1d(n * count), 256, 0, st>>>((float*)A, lda, n, s, count);
  else
    scale_cols_kernel<double><<<grid_1d(n * count), 256, 0, st>>>((double*)A, lda, n, s, count);
  SPB_LAUNCH_CHECK();
  return SPB_OK;
}

int subtract_column_means(int dtype, void* A, int64_t lda, int64_t n, int cols,
                          const double* sums, cudaStream_t st, double n_div) {
  if (n <= 0 || cols <= 0) return SPB_OK;
  const double nd = n_div > 0 ? n_div : (double)n;
  if (dtype == SPB_F32)
    sub_means_kernel<float><<<grid_1d(n * cols), 256, 0, st>>>((float*)A, lda, n, cols, sums, nd);
  else
    sub_means_kernel<double><<<grid_1d(n * cols), 256, 0, st>>>((double*)A, lda, n, cols, sums, nd);
  SPB_LAUNCH_CHECK();
  return SPB_OK;
}

// Dense operator Y = A X (DenseOperator, lobpcg.py:132-151): float64 storage only.
int dense_apply(const double* Adense, int64_t n, const void* X, int64_t ldx, int cols, void* Y,
                int64_t ldy, int dtype, double* scratch, cudaStream_t st) {
  if (dtype != SPB_F64) {
    set_error("dense operators need float64 storage");
    return SPB_ERR_DOMAIN;
  }
  (void)scratch;
  UpdParams p{};
  p.nseg = 1;
  p.q = cols;
  p.seg[0].A = Adense;
  p.seg[0].lda = n;
  p.seg[0].w = (int)n;
  p.seg[0].C = (const double*)X;
  p.seg[0].ldc = ldx;
  p.seg[0].emit = 1;
  p.seg[0].scale = 1.0;
  p.seg[0].out = Y;
  p.seg[0].ldo = ldy;
  return block_update(SPB_F64, p, n, st);
}

}  // namespace spb

extern "C" size_t spb_block_update_workspace(int32_t w, int32_t q) {
  (void)q;
  return sizeof(float) * spb::update_cstage_floats(std::max(w, 1), 1) + 256;
}

extern "C" int spb_block_update(int dtype, int mode, const void* a, int64_t lda, int32_t w,
                                const double* c, int64_t ldc, int32_t q, double scale,
                                const void* init, int64_t ldi, void* out, int64_t ldo, int64_t n,
                                void* ws, size_t ws_bytes, void* stream) {
  using namespace spb;
  if (dtype != SPB_F32 && dtype != SPB_F64) {
    set_error("unknown dtype %d", dtype);
    return SPB_ERR_DOMAIN;
  }
  if (w < 1 || q < 1 || q > 256 || n < 0 || lda < w || ldc < q || ldo < q || (init && ldi < q)) {
    set_error("block update shape contract violated");
    return SPB_ERR_CONTRACT;
  }
  if (mode == 1 && dtype != SPB_F32) {
    set_error("tensor-core update needs float32 storage");
    return SPB_ERR_DOMAIN;
  }
  if (ws_bytes < spb_block_update_workspace(w, q)) {
    set_error("block update workspace too small");
    return SPB_ERR_WORKSPACE;
  }
  if (n == 0) return SPB_OK;
  UpdParams p{};
  p.nseg = 1;
  p.q = q;
  p.init = init;
  p.ldi = ldi;
  p.seg[0] = {a, lda, c, ldc, out, ldo, scale, w, 1};
  p.cstage = (float*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  p.cstage_cap = (ws_bytes - 256) / sizeof(float);
  const int saved = g_update_mode;
  g_update_mode = mode;
  const int rc = block_update(dtype, p, n, (cudaStream_t)stream);
  g_update_mode = saved;
  if (rc != SPB_OK) return rc;
  SPB_LAUNCH_CHECK();
  return SPB_OK;
}
