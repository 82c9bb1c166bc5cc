/*
 * specpart-b200 — C ABI of the B200-native spectral-partition hot path.
 *
 * The reference (``specpart``, pure Python over numpy/scipy) has no FFI of its
 * own; these entry points are the seams of its hot path, each
 * replacing the reference routine cited beside it (paths relative to
 * /root/reference/pkg/src/specpart/). A maintainer binds them with ctypes
 * (INTEGRATION.md); paper_1708_07481_b200/_native.py is that binding.
 *
 * Conventions
 *  - every pointer marked "device" is CUDA global memory owned by the caller
 *    (PyTorch allocates it); "host" pointers are ordinary host memory;
 *  - dense blocks are row-major (vertex-major): element (i, j) at p[i*ld + j];
 *  - ``stream`` is a cudaStream_t passed as void*; work is enqueued on it and
 *    functions that need a host decision synchronise that stream;
 *  - no C++ exception crosses the boundary; every function returns a status
 *    code and spb_last_error() holds the message of the calling thread;
 *  - reentrant: no global mutable state besides the per-thread error string.
 */
#ifndef SPECPART_B200_H
#define SPECPART_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SPB_API __attribute__((visibility("default")))
#else
#define SPB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; map 1:1 onto specpart's exception classes (errors.py:4-53). */
enum {
  SPB_OK = 0,
  SPB_ERR_CONTRACT = 1,       /* ContractError: inconsistent shapes/lengths      */
  SPB_ERR_DOMAIN = 2,         /* DomainError: argument value outside its domain   */
  SPB_ERR_CONDITIONING = 3,   /* ConditioningError (lobpcg.py:168-177, :215)      */
  SPB_ERR_SOLVER = 4,         /* SolverError with a state (lobpcg.py:343-347,:426)*/
  SPB_ERR_SOLVER_NOSTATE = 5, /* SolverError(state=None) (lobpcg.py:321-327)      */
  SPB_ERR_ASSIGNMENT = 6,     /* AssignmentError (spectral.py:156-161)            */
  SPB_ERR_CUDA = 7,           /* CUDA runtime failure                             */
  SPB_ERR_WORKSPACE = 8,      /* workspace smaller than the size query returned   */
  SPB_ERR_CALLBACK = 9,       /* a host callback reported failure                 */
  SPB_ERR_PARSE = 10          /* edge-list line outside the fast-path syntax      */
};

/* Storage type of the n-row dense blocks and of the operator values. */
enum { SPB_F32 = 0, SPB_F64 = 1 };

/* CSR build modes. */
enum {
  SPB_CSR_DIRECTED = 0,  /* A: from_edges (graph.py:135-145)                     */
  SPB_CSR_SYMMETRIZED = 1, /* W = A + A', degrees of A (graph.py:220-250)        */
  SPB_CSR_AS_SYMMETRIC = 2 /* from_edges(symmetric=True): W = A, row-sum degrees */
};

SPB_API const char* spb_last_error(void);
SPB_API int spb_version(void);
SPB_API int spb_device_sm_count(void);

/* ---------------- (a) edge list -> CSR + degrees ------------------------------
 * Replaces _coerce_edges/from_edges (graph.py:106-145), symmetrize
 * (graph.py:220-236) and degrees (graph.py:239-250).
 * src, dst: device int64[m]; w: device float64[m] or NULL (unit weights).
 * Outputs (device): row_ptr int32[n+1]; col int32[cap]; val float64[cap];
 * deg float64[n] (may be NULL for SPB_CSR_DIRECTED); cap = m (DIRECTED,
 * AS_SYMMETRIC) or 2m (SYMMETRIZED). *nnz_out (host) receives the entry count.
 * Errors: SPB_ERR_DOMAIN for an endpoint outside [0, n) or a negative weight.
 * Bit-exact to the reference for integer-valued weights (all sums exact);
 * duplicate weights are summed in input order. */
SPB_API size_t spb_csr_build_workspace(int64_t m_edges, int32_t n, int mode);
SPB_API int spb_csr_build(const int64_t* src, const int64_t* dst, const double* w, int64_t m_edges,
                  int32_t n, int mode, void* ws, size_t ws_bytes, int32_t* row_ptr,
                  int32_t* col, double* val, double* deg, int64_t* nnz_out, void* stream);

/* float64 -> dtype conversion of a device vector (operator values/degrees). */
SPB_API int spb_cast(const double* in, int64_t count, int dtype, void* out, void* stream);
/* Host -> device copy of a large pageable host array (the public API's numpy inputs:
 * from_edges' arc list, graph.py:106-145; lobpcg_solve's x0, lobpcg.py:263) through a
 * caller-provided pinned ring of spb_h2d_ring_bytes(threads) bytes, staged by `threads`
 * host threads; src_esz == dst_esz copies bytes, 8 -> 4 narrows float64 to float32
 * (round to nearest even) on the way. Ordered on `stream`; the ring is free again on
 * return. */
SPB_API size_t spb_h2d_ring_bytes(int32_t threads);
SPB_API int spb_h2d_staged(const void* src, int64_t count, int32_t src_esz, int32_t dst_esz,
                           void* dst_dev, void* pinned_ring, size_t ring_bytes, int32_t threads,
                           void* stream);
/* Strided 2-D copy/convert between float64 and dtype blocks (device). */
SPB_API int spb_copy_block(int src_dtype, const void* src, int64_t lds, int dst_dtype, void* dst,
                   int64_t ldd, int64_t rows, int32_t cols, void* stream);
/* max over a device float64 vector -> host (LaplacianOperator.scale_hint, graph.py:314). */
SPB_API int spb_max_f64(const double* v, int64_t count, double* out_host, void* stream);

/* ---------------- (b) Laplacian SpMM ------------------------------------------
 * Y[i, 0:ncols] = deg[i]*X[i, :] - sum_e val[e] * X[col[e], :] for rows
 * [row_begin, row_end) of the symmetrised CSR W: laplacian_apply
 * (graph.py:253-278) on the symmetrised operator. X and Y must not alias. */
SPB_API int spb_laplacian_spmm(int dtype, int32_t row_begin, int32_t row_end, const int32_t* row_ptr,
                       const int32_t* col, const void* val, const void* deg, const void* x,
                       int64_t ldx, int32_t ncols, void* y, int64_t ldy, void* stream);

/* ---------------- (b') locality ordering for the SpMM -----------------------
 * Not a reference function: an internal relabelling of the solve (the
 * reference's laplacian_apply, graph.py:253-278, keeps the input order). The
 * vertices are renumbered so that a block-model graph's blocks become
 * contiguous runs (random-walk-smoothed seeded random columns, 16-bit sign
 * keys, stable radix sort): perm[new] = old. val/deg are dtype values of W.
 * spb_csr_permute writes the CSR of P W P' (row i = old row perm[i], its
 * entries in their original order with renumbered columns, so every SpMM row
 * sum is bit-identical), the permuted degrees and inv[old] = new.
 * spb_permute_rows: scatter == 0: dst[i] = src[idx[i]]; else dst[idx[i]] = src[i]. */
SPB_API size_t spb_vertex_order_workspace(int32_t n);
SPB_API int spb_vertex_order(int dtype, int32_t n, const int32_t* row_ptr, const int32_t* col,
                             const void* val, const void* deg, int32_t steps, uint64_t seed,
                             void* ws, size_t ws_bytes, int32_t* perm, void* stream);
SPB_API size_t spb_csr_permute_workspace(int32_t n);
SPB_API int spb_csr_permute(int dtype, int32_t n, const int32_t* row_ptr, const int32_t* col,
                            const void* val, const void* deg, const int32_t* perm, void* ws,
                            size_t ws_bytes, int32_t* inv, int32_t* out_row_ptr, int32_t* out_col,
                            void* out_val, void* out_deg, void* stream);
SPB_API int spb_permute_rows(int src_dtype, const void* src, int64_t lds, int dst_dtype, void* dst,
                             int64_t ldd, int64_t rows, int32_t cols, const int32_t* idx,
                             int scatter, void* stream);

/* ---------------- (c) tall-skinny Gram ---------------------------------------
 * out[p x q] (float64, row stride ldo) = U' V for vertex-major blocks U (n x p),
 * V (n x q): the Gram products of lobpcg.py:228, :366, :418. mode 0: float64
 * products on the FP64 tensor pipe (DMMA; any dtype); mode 1: tcgen05, 3xTF32
 * split, TMA-fed (SPB_F32 only, sm_100; 16-byte aligned rows); mode 2: tcgen05
 * int8 Ozaki splitting (6 digits, exact int32 sums; SPB_F32 only, sm_100). Split-K partials are
 * reduced in float64 in a fixed order. ws: spb_gram_workspace(p, q, n) bytes. */
SPB_API size_t spb_gram_workspace(int32_t p, int32_t q, int64_t n);
SPB_API int spb_gram(int dtype, int mode, const void* u, int64_t ldu, int32_t p, const void* v,
                     int64_t ldv, int32_t q, int64_t n, double* out, int64_t ldo, void* ws,
                     size_t ws_bytes, void* stream);

/* ---------------- (c)(d) LOBPCG -----------------------------------------------
 * Operator handle for the solve (graph.py:300-317 / lobpcg.py:132-151). */
enum { SPB_OP_LAPLACIAN = 0, SPB_OP_DENSE = 1, SPB_OP_HOST = 2 };
/* SPB_OP_HOST: any object with the reference's operator protocol (.n, .scale_hint,
 * .apply(x, out); lobpcg.py:273, graph.py:300-317) -- out = A in, host float64
 * row-major rows x cols; return 0 on success. The solve stays on the device; only
 * the operator apply crosses to the host. */
typedef int (*spb_apply_cb)(void* user, int64_t rows, int32_t cols, const double* in, double* out);
typedef struct {
  int kind;              /* SPB_OP_LAPLACIAN, SPB_OP_DENSE or SPB_OP_HOST          */
  int32_t n;             /* operator dimension                                     */
  const int32_t* row_ptr;/* LAPLACIAN: CSR of W (device)                           */
  const int32_t* col;
  const void* val;       /* dtype values of W                                      */
  const void* deg;       /* dtype degrees                                          */
  const double* dense;   /* DENSE: device float64 n x n row-major                  */
  double scale_hint;     /* max degree (graph.py:314) / max row abs-sum (lobpcg.py:143) */
  spb_apply_cb apply;    /* HOST: the operator's apply                             */
  void* apply_user;      /* HOST: passed back to apply                             */
  const int32_t* perm;   /* LAPLACIAN, optional (NULL: identity): the CSR and deg are
                            in the spb_vertex_order numbering, perm[new] = old; x0,
                            refills, preconditioner blocks and vectors_out stay in
                            the caller's order (single-GPU solves only)             */
} spb_operator;

/* SolverConfig (lobpcg.py:38-81) plus the solve arguments of lobpcg_solve
 * (lobpcg.py:263-270). */
typedef struct {
  int32_t block_size;    /* l */
  int32_t max_iter;
  double tol;
  double lock_tol;       /* config.lock_tol (0.1*tol unless overridden)            */
  int32_t n_converge;    /* nc in [1, l]                                           */
  int32_t deflate_ones;  /* project out the constant vector (lobpcg.py:259-260)    */
  int32_t has_precond;   /* call the precond callback on R_act (lobpcg.py:361-362) */
  int32_t reserved;      /* bit 0: CUDA-event timing of every SpMM (bench)        */
} spb_solver_config;

/* callback(it, theta[:l], norms) of lobpcg.py:348-349 (host arrays, copies);
 * a nonzero return aborts the solve with SPB_ERR_CALLBACK. */
typedef int (*spb_iter_cb)(void* user, int32_t it, const double* theta, const double* norms,
                           int32_t l);
/* Gaussian refill of dependent columns (lobpcg.py:214): fill rows*cols float64
 * (row-major) from the solve's numpy Generator; return 0 on success. */
typedef int (*spb_refill_cb)(void* user, int64_t rows, int32_t cols, double* out);
/* Preconditioner on the active residual block (host float64 row-major, in place). */
typedef int (*spb_precond_cb)(void* user, int64_t rows, int32_t cols, double* inout);

SPB_API size_t spb_lobpcg_workspace(int dtype, int32_t n, int32_t l);
/* x0: device float64 n x l row-major (copied; lobpcg.py:281,304). On return
 * (status OK or SOLVER) the solver's X block is left in the workspace and
 * copied to vectors_out (device float64 n x l) when vectors_out != NULL;
 * theta_out/norms_out/converged_out are host arrays of length l;
 * stats_out (host int64[16], may be NULL) receives {[0] iterations, [1] operator
 * applies, [2] Rayleigh-Ritz solves, [3] drop_p rungs, [4] rebuild rungs, [5] float32
 * orth_p re-solves, [6] 0, [7] SpMM event time (us), [8] SpMM algorithmic bytes,
 * [9] SpMM columns, [10] final scale bits hi, [11] lo, [12] Rayleigh-Ritz Gram event
 * time (us), [13] Gram pairs, [14] their algorithmic MFLOP (4 n m^2 each), 0...}; the
 * timing entries are filled when cfg->reserved has bit 0 set. */
SPB_API int spb_lobpcg_solve(const spb_operator* op, int dtype, const double* x0,
                     const spb_solver_config* cfg, spb_iter_cb cb, spb_refill_cb refill,
                     spb_precond_cb precond, void* user, void* ws, size_t ws_bytes,
                     double* vectors_out, double* theta_out, double* norms_out,
                     uint8_t* converged_out, int64_t* stats_out, void* stream);
/* ---------------- (e) row-sharded solves over NCCL ----------
 * One process per GPU. spb_comm_unique_id (rank 0) -> broadcast by the caller
 * -> spb_comm_init on every rank. The local operator holds this rank's rows of
 * W (row_ptr local, col indices remapped to the gathered layout rank*n_max +
 * local row, see spb_csr_shard), local degrees and the GLOBAL max degree in
 * scale_hint. Per operator apply the input block is all-gathered; Gram
 * partials and column sums are all-reduced in float64; the small problems are
 * solved redundantly (identical on every rank). x0 / results are local rows. */
typedef struct {
  void* comm;         /* spb_comm_init handle (NULL when nranks == 1)          */
  int32_t nranks;
  int32_t rank;
  int64_t n_global;   /* rows of the whole operator                             */
  int32_t row_begin;  /* first global row owned by this rank                    */
  int32_t n_max;      /* max rows per rank (gather padding)                     */
} spb_shard;
SPB_API int spb_comm_unique_id(void* out, int32_t bytes);
SPB_API int spb_comm_init(int32_t nranks, int32_t rank, const void* unique_id, void** comm_out);
SPB_API int spb_comm_destroy(void* comm);
/* Drives the run-time NCCL binding with a one-rank communicator (unique id, init,
 * float64 all-reduce, byte all-gather, destroy) and checks the data: the part of
 * the multi-GPU plumbing a single-GPU box can execute. */
SPB_API int spb_comm_selftest(void* stream);
/* Host-transport communicator: the same sharded solver, with each collective
 * staged through host memory and performed by the caller's callbacks (e.g. a
 * torch.distributed gloo group). For testing the row-sharded code path with
 * several ranks when fewer GPUs than ranks exist (ranks never wait on each other
 * inside a kernel: every exchange happens between launches, on the host), and
 * for hosts without NCCL. allreduce: in-place float64 sum of count values;
 * allgather: recv[r * bytes ... ] = send of rank r. Return 0 on success. */
typedef int (*spb_allreduce_cb)(void* user, double* buf, int64_t count);
typedef int (*spb_allgather_cb)(void* user, const void* send, void* recv, int64_t bytes);
SPB_API int spb_comm_init_host(int32_t nranks, int32_t rank, spb_allreduce_cb allreduce,
                               spb_allgather_cb allgather, void* user, void** comm_out);
/* Local CSR of rows [row_begin, row_end) of a global CSR, columns remapped to
 * rank(col) * n_max + (col - bounds[rank(col)]); bounds: device int32[nranks+1]. */
SPB_API int spb_csr_shard(const int32_t* row_ptr, const int32_t* col, const double* val,
                          int32_t row_begin, int32_t row_end, const int32_t* bounds,
                          int32_t nranks, int32_t n_max, int32_t* out_row_ptr, int32_t* out_col,
                          double* out_val, void* stream);
/* This rank's rows [row_begin, row_end) of W = A + A' built directly from the
 * whole arc list (no whole-graph CSR on any rank): bit-identical to those rows of
 * spb_csr_build(SYMMETRIZED) (same per-entry summation order), columns remapped as
 * spb_csr_shard does, local degrees in deg (float64[row_end - row_begin]).
 * ws: spb_csr_build_workspace(m, n, SPB_CSR_SYMMETRIZED) bytes; col/val capacity
 * 2m. bounds: device int32[nranks + 1]. */
SPB_API int spb_csr_build_rows(const int64_t* src, const int64_t* dst, const double* w,
                               int64_t m_edges, int32_t n, int32_t row_begin, int32_t row_end,
                               const int32_t* bounds, int32_t nranks, int32_t n_max, void* ws,
                               size_t ws_bytes, int32_t* row_ptr, int32_t* col, double* val,
                               double* deg, int64_t* nnz_out, void* stream);
SPB_API size_t spb_lobpcg_workspace_sharded(int dtype, int32_t n_local, int32_t l, int32_t nranks,
                                            int32_t n_max);
SPB_API int spb_lobpcg_solve_sharded(const spb_operator* op, const spb_shard* shard, int dtype,
                                     const double* x0, const spb_solver_config* cfg,
                                     spb_iter_cb cb, spb_refill_cb refill, void* user, void* ws,
                                     size_t ws_bytes, double* theta_out, double* norms_out,
                                     uint8_t* converged_out, int64_t* stats_out, void* stream);

/* Device pointer/ld of the solver's final X block inside ``ws`` (dtype); rows in
 * the operator's numbering (map them back through op->perm when it was set). */
SPB_API int spb_lobpcg_result_block(int dtype, int32_t n, int32_t l, void* ws, void** x_out,
                            int64_t* ld_out);

/* orthonormalize (lobpcg.py:195-215) of a device block b (n x width, row stride
 * ldb) in place, with Gaussian refills of dependent columns via ``refill``. */
SPB_API size_t spb_orthonormalize_workspace(int dtype, int32_t n, int32_t width);
SPB_API int spb_orthonormalize(int dtype, void* b, int64_t ldb, int32_t n, int32_t width,
                               spb_refill_cb refill, void* user, void* ws, size_t ws_bytes,
                               void* stream);

/* Block update out = init + scale * A C (the basis update of lobpcg.py:436-439
 * and the right-multiplications of :228, :366, one segment): A device n x w
 * (row stride lda), c device float64 w x q (row stride ldc), init NULL or
 * n x q; out may alias init or A (in place). mode 0: float32 CUDA-core FMA,
 * 1: 3xTF32 tensor cores (float32 only), -1: the solver's default.
 * ws: spb_block_update_workspace(w, q) bytes. */
SPB_API size_t spb_block_update_workspace(int32_t w, int32_t q);
SPB_API int spb_block_update(int dtype, int mode, const void* a, int64_t lda, int32_t w,
                             const double* c, int64_t ldc, int32_t q, double scale,
                             const void* init, int64_t ldi, void* out, int64_t ldo, int64_t n,
                             void* ws, size_t ws_bytes, void* stream);

/* Small projected problem (lobpcg.py:168-177): ga, gb are device float64
 * m x m (symmetrised inside); gb may be NULL for B = I. Outputs: theta
 * (device, nev smallest, ascending) and c (device m x nev row-major,
 * B-orthonormal columns). SPB_ERR_CONDITIONING for non-finite input,
 * cond2(gb) > 1/sqrt(eps) or gb not positive definite. */
SPB_API size_t spb_sygv_workspace(int32_t m);
SPB_API int spb_sygv(const double* ga, const double* gb, int32_t m, int32_t nev, double* theta,
             double* c, void* ws, size_t ws_bytes, void* stream);

/* ---------------- (e) QRCP assignment -----------------------------------------
 * assign_clusters_qrcp (spectral.py:134-170) on a device embedding x (dtype,
 * n x k, row stride ldx): pivots = first k dgeqp3 pivots of x'; seeds sorted;
 * cond(x[seeds]) <= 1e12 else SPB_ERR_ASSIGNMENT; labels = argmax_j
 * |(x x[seeds]^-1)_ij| (lowest j on ties), zero rows -> 0, compacted to 0..k'-1.
 * labels_out: device int32[n]; info_out (host double[4]): {k_found,
 * zero_rows, cond, ortho_err}. pivots_out (device int32[k]) may be NULL. */
SPB_API size_t spb_assign_workspace(int32_t n, int32_t k);
SPB_API int spb_assign_qrcp(int dtype, const void* x, int64_t ldx, int32_t n, int32_t k, void* ws,
                    size_t ws_bytes, int32_t* labels_out, int32_t* pivots_out,
                    double* info_out, void* stream);
/* Row-sharded assign_clusters_qrcp: this rank holds rows
 * [shard->row_begin, +n_local) of the embedding. The k pivot steps are global
 * argmax steps (two all-gathers of one record per rank per step over
 * shard->comm); the pivots (global row ids, identical on every rank and equal to
 * the single-GPU ones), the seed block and S^-1 are replicated, the labels of the
 * local rows are written to labels_out (int32[n_local]); info_out as above, global. */
SPB_API size_t spb_assign_workspace_sharded(int32_t n_local, int32_t k, int32_t nranks);
SPB_API int spb_assign_qrcp_sharded(int dtype, const void* x, int64_t ldx, int32_t n_local,
                                    int32_t k, const spb_shard* shard, void* ws, size_t ws_bytes,
                                    int32_t* labels_out, int32_t* pivots_out, double* info_out,
                                    void* stream);

/* ---------------- (f.2) edge-list ingestion ---------------------------------
 * load_edge_list (graph.py:152-209): tab-separated "src dst [weight]" text in a
 * host buffer, parsed by nthreads host threads (<= 0: all cores) into arcs in
 * file order (ids minus base). On success *handle_out owns the arrays:
 * spb_edge_list_fetch copies them into caller buffers of *m_out entries (w may
 * be null) and releases the handle. SPB_ERR_PARSE with *bad_line_out = the
 * first line (1-based) outside the accepted syntax or breaking a rule (field
 * count, negative id after base, negative weight): the caller re-reads it with
 * the reference's rules to raise the exact ParseError / DomainError. */
SPB_API int spb_edge_list_parse(const char* data, size_t len, int32_t base, int32_t nthreads,
                                int64_t* m_out, int64_t* max_idx_out, int32_t* has_weights_out,
                                int64_t* bad_line_out, void** handle_out);
SPB_API int spb_edge_list_fetch(void* handle, int64_t* src, int64_t* dst, double* w);
SPB_API void spb_edge_list_free(void* handle);

/* (f.4) Contingency table of two device label arrays (int32, values in
 * [0, kt) and [0, kf)) into device int64 counts[kt * kf] (metrics.py:65-75).
 * ws: >= 4 bytes of device scratch. SPB_ERR_CONTRACT for a label outside range. */
SPB_API int spb_contingency(const int32_t* truth, const int32_t* found, int64_t n, int32_t kt,
                            int32_t kf, int64_t* counts, void* ws, size_t ws_bytes, void* stream);

/* Optional k-means mode (north star (e); the reference has none, so parity is
 * unpinned): Lloyd iterations on the rows of x (n x d, dtype, row stride ldx),
 * optionally row-normalised, from the rows ``seeds`` (device int32[k], e.g.
 * the QRCP pivots). labels_out device int32[n] (0..k-1, lowest index on ties);
 * centroids_out device float32[k*d]; *iterations_out = Lloyd steps run. */
SPB_API size_t spb_kmeans_workspace(int32_t k, int32_t d);
SPB_API int spb_kmeans(int dtype, const void* x, int64_t ldx, int32_t n, int32_t d, int32_t k,
                       const int32_t* seeds, int32_t max_iter, int32_t normalize_rows, void* ws,
                       size_t ws_bytes, int32_t* labels_out, float* centroids_out,
                       int32_t* iterations_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPECPART_B200_H */
