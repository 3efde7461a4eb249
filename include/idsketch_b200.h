/*
 * idsketch_b200.h -- C ABI of the B200 CountSketch / TensorSketch ID hot path.
 *
 * The reference (arXiv 1901.10559's `idsketch` package, /root/reference/pkg)
 * is pure Python and has no FFI of its own; each entry point below replaces
 * the in-process native call the reference makes at the cited line (paths
 * relative to /root/reference/pkg/src/idsketch).  INTEGRATION.md shows the
 * ctypes binding that sits behind the reference's Python surface.
 *
 * Conventions
 *   - All pointers except the explicitly host-side ones are DEVICE pointers.
 *   - Every function takes the CUDA stream as `void* stream` (cudaStream_t),
 *     enqueues asynchronously and never synchronizes, unless it says so.
 *   - Temporary memory comes from a caller-owned workspace whose size the
 *     matching *_workspace_bytes() query returns.  No hidden global state.
 *   - Return value: IDS_OK or an error code; no exceptions cross the ABI.
 *     ids_last_error() returns a thread-local message for the last failure.
 *   - Matrices: "col-major" = Fortran order with leading dimension ld;
 *     sketches Y are written col-major L x R (ld = L), the layout the
 *     pivoted QR consumes (reference linalg.py:29 keeps F order).
 *   - Reentrant: distinct workspaces / outputs may be used concurrently.
 */
#ifndef IDSKETCH_B200_H
#define IDSKETCH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    IDS_OK = 0,
    IDS_EINVAL = 1,      /* -> ValueError (shapes, bounds)                     */
    IDS_ENONFINITE = 2,  /* -> ValueError ("contains non-finite entries")      */
    IDS_ESINGULAR = 3,   /* -> SingularTriangleError (linalg.py:141-144)       */
    IDS_ECUDA = 4,       /* -> RuntimeError (CUDA launch / runtime failure)    */
    IDS_EWORKSPACE = 5,  /* -> RuntimeError (workspace too small)              */
    IDS_ERETRY = 6       /* internal: draw buffer exhausted, caller grows it   */
};

enum { IDS_ROW_MAJOR = 0, IDS_COL_MAJOR = 1 };

/* flags for the CountSketch kernels */
enum {
    IDS_FLAG_ORDERED = 1,       /* force scipy's summation order (bit-exact Y) */
    IDS_FLAG_DETERMINISTIC = 2  /* sparse: fixed (segmented) summation order, run-to-run identical */
};

const char* ids_last_error(void);
int ids_version(void);
/* Diagnostic: number of kernels this library has launched so far (process-wide). */
int64_t ids_launch_count(void);
/* Diagnostic: sustained fp64 FMA throughput of the current device in TFLOP/s
 * (DFMA chains on every SM, timed with CUDA events; synchronizes `stream`).
 * The fp64 roof bench.py reports for the TensorSketch FFT work; not on the
 * sketch / ID path.  Returns a negative value on failure. */
double ids_probe_fp64_tflops(void* stream);

/* ---------------------------------------------------------------------------
 * Hash generation.  Replaces sketch.py:77-84 (CountSketchOp.__init__):
 * numpy default_rng(seed) -> [integers(0,L,I-L); permutation(arange(L)++tail)]
 * or integers(0,L,I); then integers(0,2,I)*2-1.  (state, inc) are the 128-bit
 * PCG64 state numpy's SeedSequence produced, split into 64-bit halves.
 * Outputs: bucket int32[in_dim] in [0, out_dim), sign int8[in_dim] in {-1,+1};
 * draws_out (device int64[4], may be NULL): 32-bit draws consumed by phase A,
 * phase B (permutation), signs, and a status word (0 ok).
 * Bit-exact with numpy 2.3.5 for in_dim < 2^32.
 * ------------------------------------------------------------------------- */
size_t ids_hash_workspace_bytes(int64_t in_dim, int64_t out_dim, int surjective);
int ids_countsketch_hash(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                         uint64_t inc_lo, int64_t in_dim, int64_t out_dim,
                         int surjective, int32_t* bucket, int8_t* sign,
                         int64_t* draws_out, void* workspace, size_t ws_bytes,
                         void* stream);
/* ids_countsketch_hash with (state_hi, state_lo, inc_hi, inc_lo) read from
 * DEVICE memory (uint64[4]) when the kernels run: a CUDA graph that captured
 * the draw replays it for a new seed after a 32-byte copy into seed_dev. */
int ids_countsketch_hash_dev(const uint64_t* seed_dev, int64_t in_dim, int64_t out_dim,
                             int surjective, int32_t* bucket, int8_t* sign, int64_t* draws_out,
                             void* workspace, size_t ws_bytes, void* stream);
/* Concurrency hint for ids_countsketch_hash: cap the Fisher-Yates resolution
 * grid at `ctas` CTAs (0 = whole GPU) so that several hash draws issued on
 * different streams (independent trials) run side by side.  Process-wide;
 * read when a draw is enqueued. */
void ids_set_hash_grid_cap(int ctas);
/* Staging of the surjective draw: the Fisher-Yates chain is resolved in up to
 * `stages` band groups (1..3, default 3) and the swaps of a finished group are
 * applied on an internal side stream beside the rest of the chain; the
 * caller's stream waits for the last application before the call's later
 * work.  Draws shorter than `min_in_dim` rows (0 = keep the default, 2^21),
 * draws under a grid cap (ids_set_hash_grid_cap) and draws on a capturing
 * stream are not staged.  The hash is bit-identical
 * for every setting.  Process-wide; read when a draw is enqueued. */
void ids_set_hash_stages(int stages, int64_t min_in_dim);

/* ---------------------------------------------------------------------------
 * Bucket index: the rows of each bucket in increasing row order, i.e. the CSR
 * structure of the L x I operator S that sketch.py:108-114 (`_matrix`) builds.
 * order_signed[k] = row (sign +1) or ~row (sign -1); bstart int64[L+1];
 * sorted_bucket (may be NULL): int32[I], the bucket of order_signed[k].
 * ------------------------------------------------------------------------- */
size_t ids_bucket_index_workspace_bytes(int64_t in_dim, int64_t out_dim);
int ids_bucket_index(const int32_t* bucket, const int8_t* sign, int64_t in_dim,
                     int64_t out_dim, int32_t* order_signed, int64_t* bstart,
                     int32_t* sorted_bucket, void* workspace, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Dense CountSketch Y (+)= S[:, row0:row0+rows] @ A.  Replaces sketch.py:119
 * (`self._matrix @ a` -> scipy csr_matvecs) for dense A.
 *   A: rows x cols, layout IDS_ROW_MAJOR (A[i*ld + c]) or IDS_COL_MAJOR
 *      (A[c*ld + i]); local row i is global row row0 + i.
 *   bucket/sign: the FULL hash (global rows); order_signed/bstart: the full
 *      bucket index (used by the row-major path).
 *   Y: col-major out_dim x cols.  accumulate = 0 overwrites, 1 adds.
 *   nonfinite: device int32 flag, set to 1 when a sketch entry comes out
 *      NaN/Inf (which an input NaN/Inf always causes; linalg.py:34 rejects
 *      those); the host confirms with ids_dense_has_nonfinite before raising.
 *   flags: IDS_FLAG_ORDERED forces one pass per bucket in scipy's order
 *      (increasing row), making Y bit-identical to the reference.  Without
 *      it the kernel may split long buckets into segments whose partial sums
 *      are combined in a fixed order: still deterministic run to run.
 * ------------------------------------------------------------------------- */
size_t ids_countsketch_dense_workspace_bytes(int64_t rows, int64_t cols, int64_t out_dim,
                                             int layout);
int ids_countsketch_dense_f64(const double* A, int64_t rows, int64_t cols, int64_t ld,
                              int layout, int64_t row0, int64_t in_dim,
                              const int32_t* bucket, const int8_t* sign,
                              const int32_t* order_signed, const int64_t* bstart,
                              int64_t out_dim, double* Y, int accumulate, int flags,
                              int32_t* nonfinite, void* workspace, size_t ws_bytes,
                              void* stream);

/* Exact isfinite scan of a dense matrix (host-confirmation path). */
int ids_dense_has_nonfinite(const double* A, int64_t rows, int64_t cols, int64_t ld,
                            int layout, int32_t* flag, void* stream);

/* ---------------------------------------------------------------------------
 * CSC CountSketch Y (+)= S[:, row0:row0+rows] @ A for A in CSC form -- the
 * reference's canonical sparse container (linalg.py:39-53).  colptr int64 or
 * int32 [cols+1], rowidx int32[nnz] (local rows), data double[nnz].  With
 * sorted row indices and no duplicates (canonical), Y is bit-identical to the
 * reference's SpGEMM order.  nonfinite: as for the dense kernel (confirm with
 * ids_values_has_nonfinite).
 * ------------------------------------------------------------------------- */
size_t ids_countsketch_csc_workspace_bytes(int64_t cols, int64_t out_dim);
int ids_countsketch_csc_f64(const void* colptr, int colptr64, const int32_t* rowidx,
                            const double* data, int64_t rows, int64_t cols, int64_t nnz,
                            int64_t row0, int64_t in_dim, const int32_t* bucket,
                            const int8_t* sign, int64_t out_dim, double* Y, int accumulate,
                            int32_t* nonfinite, void* workspace, size_t ws_bytes, void* stream);

/* Exact isfinite scan of a value array (sparse host-confirmation path). */
int ids_values_has_nonfinite(const double* v, int64_t n, int32_t* flag, void* stream);

/* ---------------------------------------------------------------------------
 * CSR CountSketch Y (+)= S[:, row0:row0+rows] @ A.  Replaces sketch.py:119 with
 * CSC/CSR A (scipy csr_matmat after as_csc, linalg.py:39-53).
 *   indptr: int64[rows+1] (indptr64 = 1) or int32[rows+1] (indptr64 = 0),
 *   indices int32[nnz] (column ids < cols), data double[nnz].  Duplicate
 *   entries are summed in storage order, explicit zeros are harmless.
 *   flags: IDS_FLAG_ORDERED -> one pass per bucket in scipy's order (Y
 *   bit-identical to the reference); IDS_FLAG_DETERMINISTIC -> bucket
 *   segments combined in a fixed order (run-to-run identical); neither ->
 *   one streaming pass over A with fp64 reductions into an L2-resident Y
 *   (fastest; summation order, hence the last bits of Y, not fixed).
 *   order_signed/bstart are only read by the first two modes.
 * ------------------------------------------------------------------------- */
size_t ids_countsketch_csr_workspace_bytes(int64_t rows, int64_t cols, int64_t nnz,
                                           int64_t out_dim);
int ids_countsketch_csr_f64(const void* indptr, int indptr64, const int32_t* indices,
                            const double* data, int64_t rows, int64_t cols, int64_t nnz,
                            int64_t row0, int64_t in_dim, const int32_t* bucket,
                            const int8_t* sign, const int32_t* order_signed,
                            const int64_t* bstart, int64_t out_dim, double* Y,
                            int accumulate, int flags, int32_t* nonfinite, void* workspace,
                            size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * TensorSketch of a Khatri-Rao product, scaled columnwise.  Replaces
 * sketch.py:156-186 (per-mode csr_matvecs, rfft, spectrum product, irfft,
 * x weights).  Never forms Khatri-Rao columns.
 *   n_modes, and HOST arrays of per-mode DEVICE pointers:
 *   factors[n]: col-major dims[n] x ncols with leading dimension lds[n];
 *   order_signed[n], sorted_bucket[n]: bucket index of mode n (out_dim
 *   buckets; see ids_bucket_index).
 *   weights: device double[ncols] or NULL.  Y: col-major out_dim x ncols.
 *   colnorm2 (may be NULL): ||Y[:,r]||^2 per column (fixed-order sum of the
 *   written values: run-to-run identical), for ids_cpqr_trunc_norms_f64.
 * ------------------------------------------------------------------------- */
size_t ids_tensorsketch_workspace_bytes(int n_modes, const int64_t* dims, int64_t ncols,
                                        int64_t out_dim);
int ids_tensorsketch_f64(int n_modes, const double* const* factors, const int64_t* dims,
                         const int64_t* lds, int64_t ncols,
                         const int32_t* const* order_signed,
                         const int32_t* const* sorted_bucket, int64_t out_dim,
                         const double* weights, double* Y, double* colnorm2, void* workspace,
                         size_t ws_bytes, void* stream);
/* Scatter plan of one mode (built once per mode hash, reused for every
 * ids_tensorsketch_planned_f64 call): each row's (bucket, sign) code and its
 * rank among the rows of its bucket.  With it the fused kernel reads factor
 * columns contiguously instead of gathering rows in bucket order; the
 * per-bucket sums keep scipy's row order (bit-identical CountSketch).
 * plan: 16-byte aligned device buffer of ids_ts_mode_plan_bytes(dim) bytes;
 * bstart: the bucket index's int64[out_dim + 1] starts. */
size_t ids_ts_mode_plan_bytes(int64_t dim);
int ids_ts_mode_plan(const int32_t* order_signed, const int32_t* sorted_bucket,
                     const int64_t* bstart, int64_t dim, int64_t out_dim, void* plan,
                     size_t plan_bytes, void* stream);
/* ids_tensorsketch_f64 with per-mode scatter plans (host array of device
 * pointers; an entry may be NULL, and a plan whose collisions exceed the
 * kernel's staging falls back to the gather path for that mode). */
int ids_tensorsketch_planned_f64(int n_modes, const double* const* factors, const int64_t* dims,
                                 const int64_t* lds, int64_t ncols,
                                 const int32_t* const* order_signed,
                                 const int32_t* const* sorted_bucket, const void* const* plans,
                                 int64_t out_dim, const double* weights, double* Y,
                                 double* colnorm2, void* workspace, size_t ws_bytes,
                                 void* stream);
/* Split-spectrum TensorSketch (sm_100a clusters + tensor memory), the
 * product path for out_dim in {4096, 8192, 16384} (C4, C5).  Same operation
 * as ids_tensorsketch_f64 (reference sketch.py:156-186): a cluster of two
 * CTAs per term column computes the even / odd bins of the half-length
 * spectrum from a CountSketch folded at out_dim / 2, keeps its half of the
 * running spectrum in TMEM, and the halves meet once, in the inverse.
 * Per mode it reads a folded plan (ids_ts_split_plan, built from the hash's
 * bucket int32[dim] and sign int8[dim]; ids_ts_split_plan_bytes(dim,
 * out_dim) bytes, 16-byte aligned) instead of the bucket index.  Y must be
 * 16-byte aligned; colnorm2 as for ids_tensorsketch_f64. */
int ids_tensorsketch_split_ok(int n_modes, int64_t out_dim);
size_t ids_ts_split_plan_bytes(int64_t dim, int64_t out_dim);
int ids_ts_split_plan(const int32_t* bucket, const int8_t* sign, int64_t dim, int64_t out_dim,
                      void* plan, size_t plan_bytes, void* stream);
int ids_tensorsketch_split_f64(int n_modes, const double* const* factors, const int64_t* dims,
                               const int64_t* lds, int64_t ncols, const void* const* plans,
                               int64_t out_dim, const double* weights, double* Y,
                               double* colnorm2, void* stream);
/* 1 when ids_tensorsketch_f64 handles (n_modes, out_dim) in its fused
 * one-CTA-per-term kernel (transform half-length <= 8192: power-of-two
 * out_dim <= 16384, or n_modes * (out_dim - 1) + 1 <= 16384 otherwise).
 * Larger sketches take the per-mode CountSketch + batched FFT route of the
 * Python layer. */
int ids_tensorsketch_fused_ok(int n_modes, int64_t out_dim);

/* ---------------------------------------------------------------------------
 * Truncated column-pivoted Householder QR (k steps).  Replaces linalg.py:97-102
 * (scipy.linalg.qr(pivoting=True) -> LAPACK dgeqp3 + dorgqr, truncation,
 * numerical_rank).  Pivoting follows dgeqp3: largest partial column norm with
 * LAPACK's norm downdating / tol3z recompute rule, ties to the lowest current
 * position.
 *   Y: col-major rows x cols (ld = ldy), not modified.
 *   perm int32[cols]: the k pivots first, then the remaining columns.
 *   Rtop: row-major k x cols (R[:k, :] in pivoted order).
 *   Q: col-major rows x k or NULL.   numerical_rank: device int32[1].
 * ------------------------------------------------------------------------- */
size_t ids_cpqr_workspace_bytes(int64_t rows, int64_t cols, int64_t k);
int ids_cpqr_trunc_f64(const double* Y, int64_t rows, int64_t cols, int64_t ldy,
                       int64_t k, double rank_tol, int32_t* perm, double* Rtop,
                       double* Q, int32_t* numerical_rank, void* workspace,
                       size_t ws_bytes, void* stream);
/* ids_cpqr_trunc_f64 with the initial column norms supplied: colnorm2
 * (device double[cols], may be NULL) holds ||Y[:,j]||^2, e.g. from the
 * TensorSketch kernel's epilogue, so the factorization skips its own norm
 * pass over Y (dgeqp3's initial dnrm2 loop, linalg.py:97). */
int ids_cpqr_trunc_norms_f64(const double* Y, int64_t rows, int64_t cols, int64_t ldy, int64_t k,
                             double rank_tol, const double* colnorm2, int32_t* perm,
                             double* Rtop, double* Q, int32_t* numerical_rank, void* workspace,
                             size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * ID coefficients from the truncated factorization.  Replaces
 * matrix_id.py:56-84 (_coeffs_from_pivoted) + linalg.py:130-147: floor
 * |R11[d,d]| < rank_tol*|R11[0,0]| to +-floor when numerical_rank < k,
 * T = R11^{-1} R12, P[:, perm[:k]] = I exactly, P[:, perm[k:]] = T; zero input
 * gives T = 0.   P: row-major k x cols.  deficient: device int32[1].
 * ------------------------------------------------------------------------- */
size_t ids_id_coeffs_workspace_bytes(int64_t k, int64_t cols);
int ids_id_coeffs_f64(const double* Rtop, const int32_t* perm, int64_t k, int64_t cols,
                      double rank_tol, const int32_t* numerical_rank, double* P,
                      int32_t* deficient, void* workspace, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Upper/lower triangular solve r @ x = b (linalg.py:130-147).  r row-major
 * n x n, b/x row-major n x m.  Synchronizes the stream to report an exactly
 * zero diagonal as IDS_ESINGULAR with *bad_index set (host int64).
 * ------------------------------------------------------------------------- */
int ids_triangular_solve_f64(const double* r, const double* b, int64_t n, int64_t m,
                             int lower, double* x, int64_t* bad_index, void* stream);

/* ---------------------------------------------------------------------------
 * Error metric: the operator passes of est_spectral_norm
 * through id_residual_operator / matrix_operator (estimators.py:91-121):
 * `a @ x` and `a.T @ y` on device-resident A.  Deterministic summation order.
 *
 * Dense: y = A x (trans = 0; x[cols], y[rows]) or y = A^T x (trans = 1;
 * x[rows], y[cols]); A rows x cols with leading dimension ld in `layout`.
 * ------------------------------------------------------------------------- */
size_t ids_dense_gemv_workspace_bytes(int64_t rows, int64_t cols, int layout, int trans);
int ids_dense_gemv_f64(const double* A, int64_t rows, int64_t cols, int64_t ld, int layout,
                       int trans, const double* x, double* y, void* workspace,
                       size_t ws_bytes, void* stream);

/* CSR y = A x (x[cols], y[rows]).  For A^T x pass the CSR of A^T, built once
 * by ids_csr_transpose_f64 (estimators.py:99-109 `a_t @ y`). */
int ids_csr_spmv_f64(const void* indptr, int indptr64, const int32_t* indices,
                     const double* data, int64_t rows, int64_t cols, int64_t nnz,
                     const double* x, double* y, void* stream);

/* CSR of A^T (= CSC of A) from the CSR of A: t_indptr int64[cols+1],
 * t_indices int32[nnz] (row ids, increasing within each column), t_data[nnz]
 * (linalg.py:39-53 as_csc without the canonicalization checks). */
size_t ids_csr_transpose_workspace_bytes(int64_t rows, int64_t cols, int64_t nnz);
int ids_csr_transpose_f64(const void* indptr, int indptr64, const int32_t* indices,
                          const double* data, int64_t rows, int64_t cols, int64_t nnz,
                          int64_t* t_indptr, int32_t* t_indices, double* t_data,
                          void* workspace, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Column-distributed truncated CPQR (replaces linalg.py:97 for
 * sketches whose COLUMNS are split across ranks, e.g. the term-sharded tensor
 * path).  This rank holds columns [col0, col0 + ncols) of the L x R sketch:
 * Y col-major rows x ncols (ld = ldy).  The caller drives k steps:
 *   init  -> cand (device double[4]: value, position, global column, global
 *            column at the step's position; position -1 if no finite value);
 *   per step kk: pick the global pivot (cs, ps, ck) from every rank's cand
 *            (largest value, ties to the lowest position);
 *            ids_dcpqr_pivot_f64 on every rank (position swap; the rank owning
 *            cs also writes the residual pivot column a[rows]); broadcast a
 *            from the owner; ids_dcpqr_step_f64 on every rank -> next cand.
 *   results: positions (int64[ncols]), R rows k x ncols (row-major, by local
 *            column), beta[k] (= R diagonal, replicated).
 * All state lives in the caller's workspace (ids_dcpqr_workspace_bytes).
 * ------------------------------------------------------------------------- */
size_t ids_dcpqr_workspace_bytes(int64_t rows, int64_t ncols, int64_t k);
int ids_dcpqr_init_f64(const double* Y, int64_t rows, int64_t ncols, int64_t ldy, int64_t k,
                       int64_t col0, double* cand, void* workspace, size_t ws_bytes,
                       void* stream);
int ids_dcpqr_pivot_f64(const double* Y, int64_t rows, int64_t ncols, int64_t ldy, int64_t k,
                        int64_t col0, int64_t kk, int64_t cs, int64_t ps, int64_t ck,
                        double* a, void* workspace, size_t ws_bytes, void* stream);
int ids_dcpqr_step_f64(const double* Y, int64_t rows, int64_t ncols, int64_t ldy, int64_t k,
                       int64_t col0, int64_t kk, int64_t cs, const double* a, double* cand,
                       void* workspace, size_t ws_bytes, void* stream);
int ids_dcpqr_results_f64(int64_t rows, int64_t ncols, int64_t k, int64_t* pos, double* R,
                          double* beta, void* workspace, size_t ws_bytes, void* stream);
/* Device-driven step (no host round trip per step): gather every rank's cand
 * into cands (device double[4 * nshards], shard order) and
 *   ids_dcpqr_select_f64  -> piv (device int64[3]: pivot column, its position,
 *                            column at position kk) -- the same rule as above;
 *   ids_dcpqr_pivot_dev_f64 -> a: the owner's residual pivot column, -0.0 on
 *                            every other rank, so an all-reduce(SUM) of a
 *                            over the ranks is the owner's column bit for bit;
 *   ids_dcpqr_step_dev_f64 -> as ids_dcpqr_step_f64 with the pivot from piv. */
int ids_dcpqr_select_f64(const double* cands, int64_t nshards, int64_t kk, int64_t* piv,
                         void* stream);
int ids_dcpqr_pivot_dev_f64(const double* Y, int64_t rows, int64_t ncols, int64_t ldy, int64_t k,
                            int64_t col0, int64_t kk, const int64_t* piv, double* a,
                            void* workspace, size_t ws_bytes, void* stream);
int ids_dcpqr_step_dev_f64(const double* Y, int64_t rows, int64_t ncols, int64_t ldy, int64_t k,
                           int64_t col0, int64_t kk, const int64_t* piv, const double* a,
                           double* cand, void* workspace, size_t ws_bytes, void* stream);
/* ids_dcpqr_select_f64 + ids_dcpqr_pivot_dev_f64 in one launch (what
 * distributed.py uses): the candidates in, piv and the pivot column out. */
int ids_dcpqr_select_pivot_f64(const double* Y, int64_t rows, int64_t ncols, int64_t ldy,
                               int64_t k, int64_t col0, int64_t kk, const double* cands,
                               int64_t nshards, int64_t* piv, double* a, void* workspace,
                               size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Matrix Market input (replaces scipy.io.mmread behind
 * mmio.py:23-28 and cp_tensor.py:346-361).  Host-side, multi-threaded parse.
 * ids_mm_info: size line and kind[3] = {format (0 coordinate, 1 array),
 *   field (0 real, 1 integer, 2 pattern, 3 complex), symmetry (0 general,
 *   1 symmetric, 2 skew-symmetric, 3 hermitian)}; entries = stored entries.
 * ids_mm_read: the stored entries in file order -- coordinate: 0-based
 *   row/col and the value (1.0 for pattern, real part for complex); array:
 *   values only (column-major, symmetric storage unexpanded).  Host pointers.
 * ------------------------------------------------------------------------- */
int ids_mm_info(const char* path, int64_t* rows, int64_t* cols, int64_t* entries, int32_t* kind);
int ids_mm_read(const char* path, int nthreads, int64_t* row, int64_t* col, double* val,
                int64_t capacity, int64_t* count);

/* ---------------------------------------------------------------------------
 * TensorSketch for transforms beyond the fused kernels (sketch.py:170-186 step
 * by step; any out_dim, any number of modes).  The caller sketches each mode's
 * factor matrix with the CountSketch kernels (y: nb x out_dim row-major, one
 * row per rank-1 term) and calls ids_ts_spectral_mode_f64 once per mode: the
 * rows are zero-padded to M = ids_ts_spectral_len(n_modes, out_dim) (out_dim
 * itself when it is a power of two, else the power of two >= n_modes *
 * (out_dim - 1) + 1), transformed by a hand-written batched Stockham FFT
 * (radix-4 passes through global memory) and multiplied into `spec` (nb x M
 * complex, interleaved re/im; first != 0 stores instead).  `work` holds
 * 2 * nb * M complex.  ids_ts_spectral_pair_f64 takes two modes at once: their
 * real rows ride one complex transform (ya + i yb) and are separated in the
 * frequency domain before their product enters spec.  ids_ts_spectral_finish_f64 inverse-transforms spec
 * (destroyed; work: nb * M complex), folds the result modulo out_dim and
 * scales row b by weights[b] (NULL: 1) into out (nb x out_dim row-major). */
int64_t ids_ts_spectral_len(int n_modes, int64_t out_dim);
int ids_ts_spectral_mode_f64(const double* y, int64_t nb, int64_t out_dim, int64_t M, double* spec,
                             double* work, int first, void* stream);
int ids_ts_spectral_pair_f64(const double* ya, const double* yb, int64_t nb, int64_t out_dim,
                             int64_t M, double* spec, double* work, int first, void* stream);
int ids_ts_spectral_finish_f64(double* spec, int64_t nb, int64_t out_dim, int64_t M,
                               const double* weights, double* work, double* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* IDSKETCH_B200_H */
