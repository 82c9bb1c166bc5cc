// Tall-skinny dense kernels of the LOBPCG body (CUDA-core path).
#pragma once
#include "common.cuh"

namespace spb {

constexpr int kMaxGramJobs = 20;

// One block of a batched Gram: out[out_r + i, out_c + j] = sum_k U[k, i] * V[k, j]
struct GramJob {
  const void* U;
  const void* V;
  int64_t ldu, ldv;
  int p, q;
  int out_r, out_c;
};

struct GramBatch {
  GramJob job[kMaxGramJobs];
  int tile_start[kMaxGramJobs + 1];
  int njobs;
};

// Segmented tall-skinny update: acc = init (or 0); for s in segments:
// acc += A_s[:, 0:w_s] * C_s[0:w_s, 0:q]; if emit_s: out_s = acc.
struct UpdSeg {
  const void* A;
  int64_t lda;
  const double* C;   // w x q coefficients (float64), scaled by ``scale`` on load
  int64_t ldc;
  void* out;
  int64_t ldo;
  double scale;
  int w;
  int emit;
};

struct UpdParams {
  UpdSeg seg[3];
  const void* init;
  int64_t ldi;
  int nseg;
  int q;
  float* cstage;        // optional fp32 coefficient staging (fast fp32 path)
  size_t cstage_cap;    // floats; see update_cstage_floats()
  // argmin epilogue (k-means assignment, tensor-core path only): instead of writing
  // the last emit's rows, labels[i] = argmin_j (bias[j] - 2 acc[i][j]) (lowest j on
  // ties) and *changed += rows whose label moved
  const float* argmin_bias;
  int* argmin_labels;
  unsigned long long* argmin_changed;
};

// Staging floats the fp32 update needs for segments of total width w_total.
size_t update_cstage_floats(int w_total, int nseg);
// Tensor-core (3xTF32) float32 update (update_tc.cu): false = not launched.
bool update_tc(const UpdParams& p, int64_t n, cudaStream_t st);
size_t update_tc_cstage_floats(int w_total, int nseg, int q);

// Column-reduction kinds.
enum ColReduce { CR_SUMSQ = 0, CR_SUM = 1, CR_RESIDUAL = 2 };

// ---- host entry points (dense.cu) -------------------------------------------
size_t gram_partial_doubles(int64_t n, int tiles, int out_rows, int out_cols, int* ksplit_out);
int gram_batched(int dtype, const GramBatch& b, int64_t n, int out_rows, int out_cols,
                 double* partial, size_t partial_cap, double* out, int ldo, cudaStream_t st);
int block_update(int dtype, const UpdParams& p, int64_t n, cudaStream_t st);
// sums[c] over rows of column c (kind SUMSQ / SUM), or the residual
// R = LX - X diag(theta) written to R with its column sums of squares.
size_t colreduce_partial_doubles(int64_t n, int cols);
int column_reduce(int dtype, int kind, const void* A, int64_t lda, int cols, int64_t n,
                  const void* X, int64_t ldx, const double* theta, void* R, int64_t ldr,
                  double* partial, double* out, cudaStream_t st);
int gather_columns(int dtype, void* A, int64_t lda, int64_t n, const int* idx, int count,
                   cudaStream_t st);
int scale_columns(int dtype, void* A, int64_t lda, int64_t n, const double* s, int count,
                  cudaStream_t st);
// A[:, :cols] -= sums / n_div (n_div = rows of the whole operator; <= 0 -> n)
int subtract_column_means(int dtype, void* A, int64_t lda, int64_t n, int cols,
                          const double* sums, cudaStream_t st, double n_div = 0.0);
int dense_apply(const double* Adense, int64_t n, const void* X, int64_t ldx, int cols, void* Y,
                int64_t ldy, int dtype, double* scratch, cudaStream_t st);
int copy_block(int sdt, const void* s, int64_t lds, int ddt, void* d, int64_t ldd, int64_t rows,
               int32_t cols, cudaStream_t st);
// scatter == 0: d[i] = s[idx[i]]; else d[idx[i]] = s[i] (rows, with dtype conversion)
int permute_rows(int sdt, const void* s, int64_t lds, int ddt, void* d, int64_t ldd, int64_t rows,
                 int32_t cols, const int32_t* idx, int scatter, cudaStream_t st);
// Rows [r0, r1) of W; the row's own X entry is x[(xoff + row) * ldx]; x_rows =
// rows of x the gathers can touch (L2 panel sizing; 0 -> r1).
int laplacian_spmm(int dtype, int32_t r0, int32_t r1, const int32_t* rp, const int32_t* ci,
                   const void* cv, const void* deg, const void* x, int64_t ldx, int ncols,
                   void* y, int64_t ldy, cudaStream_t st, int64_t xoff = 0, int64_t x_rows = 0);

// tcgen05 3xTF32 Gram (gram_tc.cu): out[p x (q0+q1)] = U' [V0 | V1], float32 operands.
bool gram_tc_supported();
size_t gram_tc_partial_doubles(int64_t n, int p, int qtot);
// Rayleigh-Ritz Grams on the int8 tensor cores with the Ozaki splitting (gram_oz.cu):
// Gb = B'B and Ga = B'LB (ld ldo), float32 operands n x cols, float64-accurate.
size_t gram_oz_ws_bytes(int64_t n, int p, int q);
// phase 0: one launch for both; 1: pack B, 2: Gb, 3: pack LB, 4: Ga (in this order).
int gram_oz_rr(const float* B, const float* LB, int64_t ld, int64_t n, int cols, double* Ga,
               double* Gb, int ldo, void* ws, size_t ws_bytes, cudaStream_t st, int phase = 0,
               int keep_cols = 0);
// out[(c1 + q) x q] = W' W[:, c1 : c1 + q], W = the first c1 + q columns (c1 % 8 == 0),
// packed once; ws as for gram_oz(n, c1 + q, c1 + q). rr_cols > 0: packed inside the
// Rayleigh-Ritz B operand of rr_cols columns on the same ws, whose leading c1 columns
// gram_oz_rr(phase 1, keep_cols = c1) then keeps.
int gram_oz_xr(const float* W, int64_t ld, int64_t n, int c1, int q, void* ws, size_t ws_bytes,
               double* out, int ldo, cudaStream_t st, int rr_cols = 0);
// out = U'V (p x q, ld ldo) through the Ozaki int8 path; U == V (p == q): packed once
int gram_oz(const float* U, int64_t ldu, int p, const float* V, int64_t ldv, int q, int64_t n,
            void* ws, size_t ws_bytes, double* out, int ldo, cudaStream_t st);
int gram_tc(const float* U, int64_t ldu, int p, const float* V0, int64_t ldv0, int q0,
            const float* V1, int64_t ldv1, int q1, int64_t n, double* partial, size_t partial_cap,
            double* out, int ldo, cudaStream_t st);

}  // namespace spb
