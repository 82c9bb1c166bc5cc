// (a) Edge list -> CSR (directed A or symmetrised W = A + A') + degrees.
//
// Replaces graph.py:106-145 (_coerce_edges/from_edges: self-loops dropped,
// duplicates summed, columns sorted), graph.py:220-236 (symmetrize: W = A + A',
// zero sums dropped as scipy's canonical csr binop does) and graph.py:239-250
// (degrees: bincount over rows + bincount over columns, each in CSR order).
//
// Pipeline (all device, no atomics on the data path => deterministic):
//   1. validate endpoints / weights                       (flags)
//   2. emit (key = row<<b | col, payload = 2*arc + dir)   fixed slots 2e, 2e+1;
//      self-loops emit a sentinel key that sorts last
//   3. stable LSD radix sort of (key, payload), 8-bit digits, ceil(2b/8) passes
//   4. segment heads; per group sequential sums of the forward (A_ij) and the
//      reverse (A_ji) weights in arc order; keep flag (W != 0 for SYMMETRIZED)
//   5. exclusive scan of keep flags -> output slots; scatter col / val / row
//   6. row_ptr from the row of each output entry; degrees per row as
//      (sum_j A_ij in column order) + (sum_j A_ji in column order)
#include "common.cuh"
#include "radix.cuh"
#include "scan.cuh"

namespace spb {
namespace {


struct BuildFlags {
  int bad_endpoint;
  int bad_weight;
  unsigned long long self_loops;
};

__global__ void validate_edges(const int64_t* __restrict__ src, const int64_t* __restrict__ dst,
                               const double* __restrict__ w, int64_t m, int64_t n,
                               BuildFlags* flags) {
  int bad_e = 0, bad_w = 0;
  unsigned loops = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = src[e], d = dst[e];
    bad_e |= (s < 0) | (s >= n) | (d < 0) | (d >= n);
    loops += (s == d);
    if (w) bad_w |= (w[e] < 0.0);
  }
  bad_e = __any_sync(0xffffffffu, bad_e);
  bad_w = __any_sync(0xffffffffu, bad_w);
  loops = warp_sum(loops);
  if ((threadIdx.x & 31) == 0) {
    if (bad_e) atomicOr(&flags->bad_endpoint, 1);
    if (bad_w) atomicOr(&flags->bad_weight, 1);
    if (loops) atomicAdd(&flags->self_loops, (unsigned long long)loops);
  }
}

__global__ void emit_entries(const int64_t* __restrict__ src, const int64_t* __restrict__ dst,
                             int64_t m, int b, int two_sided, uint64_t* __restrict__ keys,
                             uint32_t* __restrict__ pay) {
  const uint64_t sentinel = ((uint64_t(1) << (2 * b)) - 1);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t s = (uint64_t)src[e], d = (uint64_t)dst[e];
    bool loop = (s == d);
    if (two_sided) {
      keys[2 * e] = loop ? sentinel : ((s << b) | d);
      keys[2 * e + 1] = loop ? sentinel : ((d << b) | s);
      pay[2 * e] = (uint32_t)(2 * e);
      pay[2 * e + 1] = (uint32_t)(2 * e + 1);
    } else {
      keys[e] = loop ? sentinel : ((s << b) | d);
      pay[e] = (uint32_t)(2 * e);
    }
  }
}

// Group sums: head of each (row, col) group sums forward / reverse weights in
// payload (= input arc) order. keep[i] = 1 iff i is a head that is emitted.
__global__ void group_reduce(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ pay,
                             int64_t valid, const double* __restrict__ w, int drop_zero,
                             int* __restrict__ keep, double* __restrict__ fsum,
                             double* __restrict__ rsum, uint8_t* __restrict__ has) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < valid;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = keys[i];
    bool head = (i == 0) || (keys[i - 1] != k);
    int flag = 0;
    if (head) {
      double f = 0.0, r = 0.0;
      int hf = 0, hr = 0;
      for (int64_t j = i; j < valid && keys[j] == k; ++j) {
        uint32_t p = pay[j];
        double x = w ? w[p >> 1] : 1.0;
        if (p & 1u) {
          r = hr ? r + x : x;
          hr = 1;
        } else {
          f = hf ? f + x : x;
          hf = 1;
        }
      }
      double tot = hf ? (hr ? f + r : f) : r;
      flag = drop_zero ? (tot != 0.0) : 1;
      fsum[i] = f;
      rsum[i] = r;
      has[i] = (uint8_t)(hf | (hr << 1));
    }
    keep[i] = flag;
  }
}

__global__ void scatter_entries(const uint64_t* __restrict__ keys, int64_t valid, int b,
                                const int* __restrict__ keep, const int* __restrict__ slot,
                                const double* __restrict__ fsum, const double* __restrict__ rsum,
                                const uint8_t* __restrict__ has, int32_t* __restrict__ col,
                                double* __restrict__ val, int32_t* __restrict__ orow,
                                double* __restrict__ ofs, double* __restrict__ ors,
                                uint8_t* __restrict__ ohas) {
  const uint64_t mask = (uint64_t(1) << b) - 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < valid;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (!keep[i]) continue;
    int s = slot[i];
    uint64_t k = keys[i];
    uint8_t h = has[i];
    double f = fsum[i], r = rsum[i];
    col[s] = (int32_t)(k & mask);
    orow[s] = (int32_t)(k >> b);
    val[s] = (h & 1) ? ((h & 2) ? f + r : f) : r;
    ofs[s] = f;
    ors[s] = r;
    ohas[s] = h;
  }
}

__global__ void fill_row_ptr(const int32_t* __restrict__ orow, int64_t nnz, int32_t n,
                             int32_t* __restrict__ row_ptr) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j <= nnz;
       j += (int64_t)gridDim.x * blockDim.x) {
    int32_t r = j < nnz ? orow[j] : n;
    int32_t rp = j > 0 ? orow[j - 1] : -1;
    for (int32_t q = rp + 1; q <= r; ++q) row_ptr[q] = (int32_t)j;
  }
}

// d_i = (sum_j A_ij) + (sum_j A_ji), both accumulated in column order, exactly
// as bincount(rows, w) + bincount(cols, w) over the CSR of A (graph.py:246-249).
__global__ void row_degrees(const int32_t* __restrict__ row_ptr, const double* __restrict__ ofs,
                            const double* __restrict__ ors, const uint8_t* __restrict__ ohas,
                            int32_t n, int with_reverse, double* __restrict__ deg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double a = 0.0, c = 0.0;
    for (int32_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
      uint8_t h = ohas[e];
      if (h & 1) a += ofs[e];
      if (h & 2) c += ors[e];
    }
    deg[i] = with_reverse ? a + c : a;
  }
}

// Row-shard build (multi-GPU): only the entries of W whose row is
// in [r0, r1) are kept -- the forward arc s->d when r0 <= s < r1 and the reverse
// d->s when r0 <= d < r1 -- compacted in emission order (slot 2e, 2e+1), so every
// (row, col) group is summed in the same order as in the whole-graph build and
// the local rows are bit-identical to it. Rows are local (row - r0); columns are
// remapped to the all-gathered layout rank(col) * n_max + (col - bounds[rank]).
__device__ __forceinline__ uint64_t gathered_col(int64_t c, const int32_t* __restrict__ bounds,
                                                 int nranks, int32_t n_max) {
  int lo = 0, hi = nranks;  // owner: bounds[lo] <= c < bounds[lo + 1]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (bounds[mid] <= c) lo = mid; else hi = mid;
  }
  return (uint64_t)lo * (uint64_t)n_max + (uint64_t)(c - bounds[lo]);
}

__global__ void rows_flags(const int64_t* __restrict__ src, const int64_t* __restrict__ dst,
                           int64_t m, int64_t r0, int64_t r1, int* __restrict__ flag) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = src[e], b = dst[e];
    const bool loop = a == b;
    flag[2 * e] = !loop && a >= r0 && a < r1;
    flag[2 * e + 1] = !loop && b >= r0 && b < r1;
  }
}

__global__ void rows_emit(const int64_t* __restrict__ src, const int64_t* __restrict__ dst,
                          int64_t m, int64_t r0, const int32_t* __restrict__ bounds, int nranks,
                          int32_t n_max, int b, const int* __restrict__ flag,
                          const int* __restrict__ slot, uint64_t* __restrict__ keys,
                          uint32_t* __restrict__ pay) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = src[e], c = dst[e];
    if (flag[2 * e]) {
      const int s = slot[2 * e];
      keys[s] = ((uint64_t)(a - r0) << b) | gathered_col(c, bounds, nranks, n_max);
      pay[s] = (uint32_t)(2 * e);
    }
    if (flag[2 * e + 1]) {
      const int s = slot[2 * e + 1];
      keys[s] = ((uint64_t)(c - r0) << b) | gathered_col(a, bounds, nranks, n_max);
      pay[s] = (uint32_t)(2 * e + 1);
    }
  }
}

// ---------------------------------------------------------------------------
// Bucket build (default): no global sort. Entries are counted per row (integer
// atomics), scattered into their row's bucket (atomic cursor: arbitrary order
// inside the bucket), then every row is sorted in shared memory by (col, payload)
// -- payload = emission index 2e / 2e+1, so duplicate (row, col) entries come out
// in the same order as the stable radix sort and every sum below is bit-identical
// to the radix path's -- reduced, and compacted. Rows of more than kBkMaxRow
// entries fall back to the radix path.
constexpr int kBkMaxRow = 1024;   // entries per row sorted in shared memory
constexpr int kBkRank = 96;       // rows up to this many entries: rank sort (3 keys per lane), else bitonic
constexpr int kBkSmall = 256;     // rows up to this many entries: 2 KB per warp (bk_rows)
constexpr int kBkWarps = 8;       // rows (warps) per CTA of bk_rows

struct BkSpec {
  int two_sided;                  // reverse entries (SYMMETRIZED)
  int64_t r0, r1;                 // rows kept (row-shard build), else [0, n)
  const int32_t* bounds;          // non-null: columns remapped to the gathered layout
  int nranks;
  int32_t n_max;
};

__device__ __forceinline__ uint32_t bk_col(const BkSpec& S, int64_t c) {
  if (!S.bounds) return (uint32_t)c;
  int lo = 0, hi = S.nranks;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (S.bounds[mid] <= c) lo = mid; else hi = mid;
  }
  return (uint32_t)((int64_t)lo * S.n_max + (c - S.bounds[lo]));
}

__global__ void bk_count(const int64_t* __restrict__ src, const int64_t* __restrict__ dst, int64_t m,
                         BkSpec S, int* __restrict__ cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = src[e], b = dst[e];
    if (a == b) continue;
    if (a >= S.r0 && a < S.r1) atomicAdd(&cnt[a - S.r0], 1);
    if (S.two_sided && b >= S.r0 && b < S.r1) atomicAdd(&cnt[b - S.r0], 1);
  }
}

__global__ void bk_max(const int* __restrict__ cnt, int64_t n, int* __restrict__ out) {
  int mx = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    mx = max(mx, cnt[i]);
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
}

__global__ void bk_scatter(const int64_t* __restrict__ src, const int64_t* __restrict__ dst, int64_t m,
                           BkSpec S, int* __restrict__ cursor, uint64_t* __restrict__ keys) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = src[e], b = dst[e];
    if (a == b) continue;
    if (a >= S.r0 && a < S.r1) {
      const int p = atomicAdd(&cursor[a - S.r0], 1);
      keys[p] = ((uint64_t)bk_col(S, b) << 32) | (uint32_t)(2 * e);
    }
    if (S.two_sided && b >= S.r0 && b < S.r1) {
      const int p = atomicAdd(&cursor[b - S.r0], 1);
      keys[p] = ((uint64_t)bk_col(S, a) << 32) | (uint32_t)(2 * e + 1);
    }
  }
}

// Warp per row: sort the bucket, sum each (row, col) group in payload order
// (forward and reverse weights apart, as group_reduce), keep non-zero sums
// (SYMMETRIZED), write the row's unique entries at the start of its bucket and its
// degree (forward sums then reverse sums, each in column order, as row_degrees).
// One row (one warp): b is this warp's shared buffer of CAP keys; rows with cnt in
// (lo, CAP] are processed, others skipped (handled by the other launch).
template <int CAP>
__device__ __forceinline__ void bk_row(int64_t row, int lo, uint64_t* b, const int* __restrict__ off,
                                       const uint64_t* __restrict__ keys, const double* __restrict__ w,
                                       int drop_zero, int with_reverse, int32_t* __restrict__ tcol,
                                       double* __restrict__ tval, int* __restrict__ ucnt,
                                       double* __restrict__ deg) {
  const int lane = threadIdx.x & 31;
    const int o0 = off[row], cnt = off[row + 1] - o0;
    if (cnt <= lo || cnt > CAP) return;
    if (cnt <= kBkRank) {
      // short rows (most of them): rank sort -- every key's position is the number of
      // smaller keys (keys are unique: the payload is), read by broadcast from the
      // second half of the buffer
      uint64_t* in = b + CAP / 2;
      for (int i = lane; i < cnt; i += 32) in[i] = keys[o0 + i];
      __syncwarp();
      // up to three keys per lane ranked in one pass over the row (kBkRank <= 96)
      const uint64_t k0 = lane < cnt ? in[lane] : ~0ull;
      const uint64_t k1 = lane + 32 < cnt ? in[lane + 32] : ~0ull;
      const uint64_t k2 = lane + 64 < cnt ? in[lane + 64] : ~0ull;
      int r0 = 0, r1 = 0, r2 = 0;
      for (int t = 0; t < cnt; ++t) {
        const uint64_t v = in[t];
        r0 += v < k0;
        r1 += v < k1;
        r2 += v < k2;
      }
      if (lane < cnt) b[r0] = k0;
      if (lane + 32 < cnt) b[r1] = k1;
      if (lane + 64 < cnt) b[r2] = k2;
      __syncwarp();
    } else {
      int P = 1;
      while (P < cnt) P <<= 1;
      for (int i = lane; i < P; i += 32) b[i] = i < cnt ? keys[o0 + i] : ~0ull;
      __syncwarp();
      for (int k = 2; k <= P; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
          for (int i = lane; i < P; i += 32) {
            const int ixj = i ^ j;
            if (ixj > i) {
              const uint64_t x = b[i], y = b[ixj];
              if ((x > y) == ((i & k) == 0)) {
                b[i] = y;
                b[ixj] = x;
              }
            }
          }
          __syncwarp();
        }
    }
    int u0 = 0;
    double a = 0.0, c = 0.0;
    for (int base = 0; base < cnt; base += 32) {
      const int i = base + lane;
      bool head = false, keep = false;
      double f = 0.0, r = 0.0;
      int hf = 0, hr = 0;
      uint32_t col = 0;
      if (i < cnt) {
        col = (uint32_t)(b[i] >> 32);
        head = i == 0 || (uint32_t)(b[i - 1] >> 32) != col;
        if (head) {
          for (int j = i; j < cnt && (uint32_t)(b[j] >> 32) == col; ++j) {
            const uint32_t p = (uint32_t)b[j];
            const double x = w ? w[p >> 1] : 1.0;
            if (p & 1u) {
              r = hr ? r + x : x;
              hr = 1;
            } else {
              f = hf ? f + x : x;
              hf = 1;
            }
          }
          const double tot = hf ? (hr ? f + r : f) : r;
          keep = drop_zero ? tot != 0.0 : true;
        }
      }
      const unsigned km = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        const int u = u0 + __popc(km & ((1u << lane) - 1u));
        tcol[o0 + u] = (int32_t)col;
        tval[o0 + u] = hf ? (hr ? f + r : f) : r;
      }
      // degree: forward then reverse group sums in column order (lane order here)
      const double fk = (keep && hf) ? f : 0.0, rk = (keep && hr) ? r : 0.0;
      if (!w) {
        // unit weights: every sum is an exact integer, so lane-local partials and a
        // tree reduction give the same bits as the ordered sum
        a += fk;
        c += rk;
      } else if (deg) {
        const bool fh = keep && hf, rh = keep && hr;
        const unsigned fm = __ballot_sync(0xffffffffu, fh), rm = __ballot_sync(0xffffffffu, rh);
        for (int t = 0; t < 32; ++t) {
          const double ft = __shfl_sync(0xffffffffu, fk, t), rt = __shfl_sync(0xffffffffu, rk, t);
          if ((fm >> t) & 1u) a += ft;
          if ((rm >> t) & 1u) c += rt;
        }
      }
      u0 += __popc(km);
    }
    if (!w && deg) {
      a = warp_sum(a);
      c = warp_sum(c);
    }
    if (lane == 0) {
      ucnt[row] = u0;
      if (deg) deg[row] = with_reverse ? a + c : a;
    }
    __syncwarp();
}

// Rows of at most kBkSmall entries, 2 KB of shared memory per warp (full occupancy).
__global__ void __launch_bounds__(32 * kBkWarps)
bk_rows(const int* __restrict__ off, int32_t nrows, const uint64_t* __restrict__ keys,
        const double* __restrict__ w, int drop_zero, int with_reverse, int32_t* __restrict__ tcol,
        double* __restrict__ tval, int* __restrict__ ucnt, double* __restrict__ deg) {
  __shared__ uint64_t buf[kBkWarps][kBkSmall];
  const int wid = threadIdx.x >> 5;
  for (int64_t row = (int64_t)blockIdx.x * kBkWarps + wid; row < nrows;
       row += (int64_t)gridDim.x * kBkWarps)
    bk_row<kBkSmall>(row, -1, buf[wid], off, keys, w, drop_zero, with_reverse, tcol, tval, ucnt, deg);
}

// The few longer rows (kBkSmall < cnt <= kBkMaxRow): one warp per CTA, 8 KB.
__global__ void __launch_bounds__(32)
bk_rows_big(const int* __restrict__ off, int32_t nrows, const uint64_t* __restrict__ keys,
            const double* __restrict__ w, int drop_zero, int with_reverse, int32_t* __restrict__ tcol,
            double* __restrict__ tval, int* __restrict__ ucnt, double* __restrict__ deg) {
  __shared__ uint64_t buf[kBkMaxRow];
  for (int64_t row = blockIdx.x; row < nrows; row += gridDim.x)
    bk_row<kBkMaxRow>(row, kBkSmall, buf, off, keys, w, drop_zero, with_reverse, tcol, tval, ucnt,
                      deg);
}

__global__ void bk_copy(const int* __restrict__ off, const int32_t* __restrict__ row_ptr,
                        int32_t nrows, const int32_t* __restrict__ tcol, const double* __restrict__ tval,
                        int32_t* __restrict__ col, double* __restrict__ val) {
  const int lane = threadIdx.x & 31;
  for (int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; row < nrows;
       row += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int o0 = off[row], d0 = row_ptr[row], cnt = row_ptr[row + 1] - d0;
    for (int i = lane; i < cnt; i += 32) {
      col[d0 + i] = tcol[o0 + i];
      val[d0 + i] = tval[o0 + i];
    }
  }
}

int key_bits(int32_t n) {
  int b = 1;
  while ((int64_t(1) << b) <= (int64_t)n) ++b;
  return b;
}

struct BuildLayout {
  uint64_t *ka, *kb;
  uint32_t *pa, *pb;
  int *counts, *scan_tmp, *keep, *slot, *dev_ints;
  int *bcnt, *boff, *bcur, *bucnt;  // bucket path, per row (n + 1)
  double *fsum, *rsum, *ofs, *ors;
  uint8_t *has, *ohas;
  int32_t* orow;
  BuildFlags* flags;
};

BuildLayout carve(Arena& a, int64_t cap, int64_t nrows) {
  BuildLayout L;
  int64_t ntiles = ceil_div(cap, kSortTile);
  L.ka = a.take<uint64_t>(cap);
  L.kb = a.take<uint64_t>(cap);
  L.pa = a.take<uint32_t>(cap);
  L.pb = a.take<uint32_t>(cap);
  L.counts = a.take<int>((size_t)kRadix * ntiles + 1);
  L.scan_tmp = a.take<int>(
      scan_workspace_ints(std::max<int64_t>(std::max<int64_t>(cap, kRadix * ntiles), nrows + 1)) + 8);
  L.bcnt = a.take<int>(nrows + 1);
  L.boff = a.take<int>(nrows + 1);
  L.bcur = a.take<int>(nrows + 1);
  L.bucnt = a.take<int>(nrows + 1);
  L.keep = a.take<int>(cap + 1);
  L.slot = a.take<int>(cap + 1);
  L.fsum = a.take<double>(cap);
  L.rsum = a.take<double>(cap);
  L.ofs = a.take<double>(cap);
  L.ors = a.take<double>(cap);
  L.has = a.take<uint8_t>(cap);
  L.ohas = a.take<uint8_t>(cap);
  L.orow = a.take<int32_t>(cap);
  L.dev_ints = a.take<int>(8);
  L.flags = a.take<BuildFlags>(1);
  return L;
}

int sort_reduce_scatter(BuildLayout& L, const double* w, int64_t count, int64_t valid, int b,
                        bool symmetrized, int32_t n, int32_t* row_ptr, int32_t* col, double* val,
                        double* deg, int64_t* nnz_out, cudaStream_t st);
int bucket_build(BuildLayout& L, const int64_t* src, const int64_t* dst, const double* w, int64_t m,
                 int32_t nrows, const BkSpec& S, bool symmetrized, int32_t* row_ptr, int32_t* col,
                 double* val, double* deg, int64_t* nnz_out, bool* fell_back, cudaStream_t st);

int grid_for(int64_t work, int threads = 256) {
  int64_t g = ceil_div(std::max<int64_t>(work, 1), threads);
  return (int)std::min<int64_t>(g, (int64_t)num_sms() * 16);
}

}  // namespace
}  // namespace spb

using namespace spb;

extern "C" size_t spb_csr_build_workspace(int64_t m_edges, int32_t n, int mode) {
  Arena a;
  a.dry = true;
  int64_t cap = (mode == SPB_CSR_SYMMETRIZED ? 2 : 1) * std::max<int64_t>(m_edges, 1);
  carve(a, cap, std::max<int32_t>(n, 0));
  return a.used + 1024;
}

extern "C" int spb_csr_build(const int64_t* src, const int64_t* dst, const double* w,
                             int64_t m, int32_t n, int mode, void* ws, size_t ws_bytes,
                             int32_t* row_ptr, int32_t* col, double* val, double* deg,
                             int64_t* nnz_out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0 || m < 0) {
    set_error("negative sizes");
    return SPB_ERR_CONTRACT;
  }
  if (mode < 0 || mode > 2) {
    set_error("unknown csr build mode %d", mode);
    return SPB_ERR_DOMAIN;
  }
  if (mode == SPB_CSR_DIRECTED && deg) {
    set_error("degrees need the reverse arcs: build SYMMETRIZED or AS_SYMMETRIC");
    return SPB_ERR_CONTRACT;
  }
  if (m >= (int64_t(1) << 30)) {
    set_error("edge count %lld exceeds 2^30 per build", (long long)m);
    return SPB_ERR_CONTRACT;
  }
  const int two = (mode == SPB_CSR_SYMMETRIZED);
  const int64_t cap = (two ? 2 : 1) * std::max<int64_t>(m, 1);
  Arena a;
  a.base = (char*)ws;
  a.cap = ws_bytes;
  BuildLayout L = carve(a, cap, n);
  if (a.used > ws_bytes) {
    set_error("csr build workspace too small (%zu < %zu)", ws_bytes, a.used);
    return SPB_ERR_WORKSPACE;
  }
  if (n == 0) {
    if (m > 0) {
      set_error("edge endpoint out of range");
      return SPB_ERR_DOMAIN;
    }
    SPB_CUDA(cudaMemsetAsync(row_ptr, 0, sizeof(int32_t), st));
    *nnz_out = 0;
    return SPB_OK;
  }
  SPB_CUDA(cudaMemsetAsync(L.flags, 0, sizeof(BuildFlags), st));
  if (m > 0) {
    validate_edges<<<grid_for(m), 256, 0, st>>>(src, dst, w, m, n, L.flags);
    SPB_LAUNCH_CHECK();
  }
  BuildFlags hf;
  SPB_CUDA(cudaMemcpyAsync(&hf, L.flags, sizeof(hf), cudaMemcpyDeviceToHost, st));
  SPB_CUDA(cudaStreamSynchronize(st));
  if (hf.bad_endpoint) {
    set_error("edge endpoint out of range");
    return SPB_ERR_DOMAIN;
  }
  if (hf.bad_weight) {
    set_error("negative edge weight");
    return SPB_ERR_DOMAIN;
  }
  if (m == 0) {
    SPB_CUDA(cudaMemsetAsync(row_ptr, 0, sizeof(int32_t) * (n + 1), st));
    if (deg) SPB_CUDA(cudaMemsetAsync(deg, 0, sizeof(double) * n, st));
    *nnz_out = 0;
    return SPB_OK;
  }
  {
    const BkSpec S{two, 0, n, nullptr, 1, 0};
    bool fb = false;
    SPB_TRY(bucket_build(L, src, dst, w, m, n, S, mode == SPB_CSR_SYMMETRIZED, row_ptr, col, val, deg,
                         nnz_out, &fb, st));
    if (!fb) return SPB_OK;
  }
  const int b = key_bits(n);
  const int64_t count = (two ? 2 : 1) * m;
  emit_entries<<<grid_for(m), 256, 0, st>>>(src, dst, m, b, two, L.ka, L.pa);
  SPB_LAUNCH_CHECK();
  // self-loops carry the sentinel key and sort to the end
  const int64_t valid = count - (two ? 2 : 1) * (int64_t)hf.self_loops;
  return sort_reduce_scatter(L, w, count, valid, b, mode == SPB_CSR_SYMMETRIZED, n, row_ptr, col,
                             val, deg, nnz_out, st);
}

namespace spb {
namespace {
// Stable radix sort of the emitted (key, payload) pairs, per-(row, col) sums,
// compaction into the CSR arrays, row pointers and degrees (steps 3-6 above).
int sort_reduce_scatter(BuildLayout& L, const double* w, int64_t count, int64_t valid, int b,
                        bool symmetrized, int32_t n, int32_t* row_ptr, int32_t* col, double* val,
                        double* deg, int64_t* nnz_out, cudaStream_t st) {
  // stable LSD radix sort over 2b key bits
  uint64_t *kin = L.ka, *kout = L.kb;
  uint32_t *pin = L.pa, *pout = L.pb;
  SPB_TRY(radix_sort_pairs(&kin, &pin, &kout, &pout, count, 2 * b, L.counts, L.scan_tmp, st));
  int32_t* dev_total = L.dev_ints;
  int64_t nnz = 0;
  if (valid > 0) {
    group_reduce<<<grid_for(valid), 256, 0, st>>>(kin, pin, valid, w, symmetrized, L.keep, L.fsum,
                                                   L.rsum, L.has);
    SPB_LAUNCH_CHECK();
    SPB_TRY(exclusive_scan_i32(L.keep, L.slot, valid, L.scan_tmp, dev_total, st));
    int htot = 0;
    SPB_CUDA(cudaMemcpyAsync(&htot, dev_total, sizeof(int), cudaMemcpyDeviceToHost, st));
    SPB_CUDA(cudaStreamSynchronize(st));
    nnz = htot;
    scatter_entries<<<grid_for(valid), 256, 0, st>>>(kin, valid, b, L.keep, L.slot, L.fsum,
                                                     L.rsum, L.has, col, val, L.orow, L.ofs,
                                                     L.ors, L.ohas);
    SPB_LAUNCH_CHECK();
  }
  fill_row_ptr<<<grid_for(nnz + 1), 256, 0, st>>>(L.orow, nnz, n, row_ptr);
  SPB_LAUNCH_CHECK();
  if (deg) {
    row_degrees<<<grid_for(n), 256, 0, st>>>(row_ptr, L.ofs, L.ors, L.ohas, n, symmetrized, deg);
    SPB_LAUNCH_CHECK();
  }
  *nnz_out = nnz;
  return SPB_OK;
}
}  // namespace
}  // namespace spb

namespace spb {
namespace {
// The bucket build (see bk_rows); *fell_back when a row exceeds kBkMaxRow entries
// (nothing written then: the caller runs the radix path).
int bucket_build(BuildLayout& L, const int64_t* src, const int64_t* dst, const double* w, int64_t m,
                 int32_t nrows, const BkSpec& S, bool symmetrized, int32_t* row_ptr, int32_t* col,
                 double* val, double* deg, int64_t* nnz_out, bool* fell_back, cudaStream_t st) {
  *fell_back = false;
  SPB_CUDA(cudaMemsetAsync(L.bcnt, 0, sizeof(int) * (size_t)nrows, st));
  SPB_CUDA(cudaMemsetAsync(L.dev_ints, 0, sizeof(int) * 4, st));
  bk_count<<<grid_for(m), 256, 0, st>>>(src, dst, m, S, L.bcnt);
  SPB_LAUNCH_CHECK();
  SPB_TRY(exclusive_scan_i32(L.bcnt, L.boff, nrows, L.scan_tmp, L.boff + nrows, st));
  bk_max<<<grid_for(nrows), 256, 0, st>>>(L.bcnt, nrows, L.dev_ints + 1);
  SPB_LAUNCH_CHECK();
  int h[2] = {0, 0};
  SPB_CUDA(cudaMemcpyAsync(&h[0], L.boff + nrows, sizeof(int), cudaMemcpyDeviceToHost, st));
  SPB_CUDA(cudaMemcpyAsync(&h[1], L.dev_ints + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  SPB_CUDA(cudaStreamSynchronize(st));
  if (h[1] > kBkMaxRow) {
    *fell_back = true;
    return SPB_OK;
  }
  SPB_CUDA(cudaMemcpyAsync(L.bcur, L.boff, sizeof(int) * (size_t)nrows, cudaMemcpyDeviceToDevice, st));
  bk_scatter<<<grid_for(m), 256, 0, st>>>(src, dst, m, S, L.bcur, L.ka);
  SPB_LAUNCH_CHECK();
  int32_t* tcol = reinterpret_cast<int32_t*>(L.pa);
  const int rblocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nrows, kBkWarps), num_sms() * 8));
  bk_rows<<<rblocks, 32 * kBkWarps, 0, st>>>(L.boff, nrows, L.ka, w, symmetrized ? 1 : 0,
                                             symmetrized ? 1 : 0, tcol, L.fsum, L.bucnt, deg);
  if (h[1] > kBkSmall)
    bk_rows_big<<<(int)std::min<int64_t>(nrows, num_sms() * 16), 32, 0, st>>>(
        L.boff, nrows, L.ka, w, symmetrized ? 1 : 0, symmetrized ? 1 : 0, tcol, L.fsum, L.bucnt, deg);
  SPB_LAUNCH_CHECK();
  SPB_TRY(exclusive_scan_i32(L.bucnt, row_ptr, nrows, L.scan_tmp, row_ptr + nrows, st));
  int nnz = 0;
  SPB_CUDA(cudaMemcpyAsync(&nnz, row_ptr + nrows, sizeof(int), cudaMemcpyDeviceToHost, st));
  SPB_CUDA(cudaStreamSynchronize(st));
  bk_copy<<<grid_for((int64_t)nrows * 32), 256, 0, st>>>(L.boff, row_ptr, nrows, tcol, L.fsum, col, val);
  SPB_LAUNCH_CHECK();
  *nnz_out = nnz;
  return SPB_OK;
}
}  // namespace
}  // namespace spb

extern "C" int spb_csr_build_rows(const int64_t* src, const int64_t* dst, const double* w,
                                  int64_t m, int32_t n, int32_t row_begin, int32_t row_end,
                                  const int32_t* bounds, int32_t nranks, int32_t n_max, void* ws,
                                  size_t ws_bytes, int32_t* row_ptr, int32_t* col, double* val,
                                  double* deg, int64_t* nnz_out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0 || m < 0 || row_begin < 0 || row_end < row_begin || row_end > n || nranks < 1 ||
      n_max < row_end - row_begin || !deg) {
    set_error("csr row-shard build contract violated");
    return SPB_ERR_CONTRACT;
  }
  if (m >= (int64_t(1) << 30)) {
    set_error("edge count %lld exceeds 2^30 per build", (long long)m);
    return SPB_ERR_CONTRACT;
  }
  const int32_t nl = row_end - row_begin;
  const int64_t cap = 2 * std::max<int64_t>(m, 1);
  Arena a;
  a.base = (char*)ws;
  a.cap = ws_bytes;
  BuildLayout L = carve(a, cap, n);
  if (a.used > ws_bytes) {
    set_error("csr build workspace too small (%zu < %zu)", ws_bytes, a.used);
    return SPB_ERR_WORKSPACE;
  }
  SPB_CUDA(cudaMemsetAsync(L.flags, 0, sizeof(BuildFlags), st));
  if (m > 0) {
    validate_edges<<<grid_for(m), 256, 0, st>>>(src, dst, w, m, n, L.flags);
    SPB_LAUNCH_CHECK();
  }
  BuildFlags hf;
  SPB_CUDA(cudaMemcpyAsync(&hf, L.flags, sizeof(hf), cudaMemcpyDeviceToHost, st));
  SPB_CUDA(cudaStreamSynchronize(st));
  if (hf.bad_endpoint) {
    set_error("edge endpoint out of range");
    return SPB_ERR_DOMAIN;
  }
  if (hf.bad_weight) {
    set_error("negative edge weight");
    return SPB_ERR_DOMAIN;
  }
  if (m == 0 || nl == 0) {
    SPB_CUDA(cudaMemsetAsync(row_ptr, 0, sizeof(int32_t) * (nl + 1), st));
    if (nl) SPB_CUDA(cudaMemsetAsync(deg, 0, sizeof(double) * nl, st));
    *nnz_out = 0;
    return SPB_OK;
  }
  {
    const BkSpec S{1, row_begin, row_end, bounds, nranks, n_max};
    bool fb = false;
    SPB_TRY(bucket_build(L, src, dst, w, m, nl, S, true, row_ptr, col, val, deg, nnz_out, &fb, st));
    if (!fb) return SPB_OK;
  }
  // radix fallback: compaction of this rank's entries, in emission order (keep/slot reused)
  rows_flags<<<grid_for(m), 256, 0, st>>>(src, dst, m, row_begin, row_end, L.keep);
  SPB_LAUNCH_CHECK();
  SPB_TRY(exclusive_scan_i32(L.keep, L.slot, 2 * m, L.scan_tmp, L.dev_ints, st));
  int htot = 0;
  SPB_CUDA(cudaMemcpyAsync(&htot, L.dev_ints, sizeof(int), cudaMemcpyDeviceToHost, st));
  SPB_CUDA(cudaStreamSynchronize(st));
  const int b = key_bits(std::max<int32_t>(nl, (int32_t)std::min<int64_t>(
                                                   (int64_t)nranks * n_max, INT32_MAX)));
  if (2 * b > 64) {
    set_error("row-shard key does not fit 64 bits");
    return SPB_ERR_CONTRACT;
  }
  rows_emit<<<grid_for(m), 256, 0, st>>>(src, dst, m, row_begin, bounds, nranks, n_max, b, L.keep,
                                         L.slot, L.ka, L.pa);
  SPB_LAUNCH_CHECK();
  return sort_reduce_scatter(L, w, htot, htot, b, true, nl, row_ptr, col, val, deg, nnz_out, st);
}

// ---------------------------------------------------------------------------
// Row shard of a CSR for the multi-GPU solve: rows [r0, r1), columns remapped to
// the all-gathered layout (rank * n_max + local row of the owning rank).
namespace spb {
namespace {

__global__ void shard_rows(const int32_t* __restrict__ rp, int32_t r0, int32_t r1,
                           int32_t* __restrict__ orp) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= (int64_t)(r1 - r0);
       i += (int64_t)gridDim.x * blockDim.x)
    orp[i] = rp[r0 + i] - rp[r0];
}

__global__ void shard_cols(const int32_t* __restrict__ col, const double* __restrict__ val,
                           int64_t e0, int64_t count, const int32_t* __restrict__ bounds,
                           int32_t nranks, int32_t n_max, int32_t* __restrict__ ocol,
                           double* __restrict__ oval) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = col[e0 + e];
    int lo = 0, hi = nranks;  // owner: bounds[lo] <= c < bounds[lo + 1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (bounds[mid] <= c) lo = mid; else hi = mid;
    }
    ocol[e] = lo * n_max + (c - bounds[lo]);
    oval[e] = val[e0 + e];
  }
}

}  // namespace
}  // namespace spb

extern "C" int spb_csr_shard(const int32_t* row_ptr, const int32_t* col, const double* val,
                             int32_t row_begin, int32_t row_end, const int32_t* bounds,
                             int32_t nranks, int32_t n_max, int32_t* out_row_ptr, int32_t* out_col,
                             double* out_val, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (row_end < row_begin || nranks < 1 || n_max < 0) {
    set_error("csr shard contract violated");
    return SPB_ERR_CONTRACT;
  }
  int32_t e[2];
  SPB_CUDA(cudaMemcpyAsync(&e[0], row_ptr + row_begin, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  SPB_CUDA(cudaMemcpyAsync(&e[1], row_ptr + row_end, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  SPB_CUDA(cudaStreamSynchronize(st));
  shard_rows<<<grid_for(row_end - row_begin + 1), 256, 0, st>>>(row_ptr, row_begin, row_end,
                                                                 out_row_ptr);
  const int64_t count = (int64_t)e[1] - e[0];
  if (count > 0)
    shard_cols<<<grid_for(count), 256, 0, st>>>(col, val, e[0], count, bounds, nranks, n_max,
                                                 out_col, out_val);
  SPB_LAUNCH_CHECK();
  return SPB_OK;
}
