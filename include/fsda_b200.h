/*
 * fsda_b200.h — C ABI of the B200-native FSDA hot path.
 *
 * This is the drop-in boundary for the reference's FSDA solver
 * (`sdakit.sda._SOLVERS["fsda"]`, /root/reference/pkg/src/sdakit/sda.py:465-486).
 * Every entry point takes plain host pointers and sizes; no torch or numpy
 * types appear here.  The Python host layer (paper_1709_04794_b200/_capi.py)
 * binds these with ctypes; INTEGRATION.md shows the stub a maintainer of the
 * reference would add.
 *
 * Data model (mirrors sdakit, /root/reference/pkg/src/sdakit/sparse.py:41-146):
 *   X   N x D CSR, int64 row offsets + int64 column indices, implicit value 1
 *       (the reference stores float64 values; a non-binary X is rejected by the
 *       host layer with ValueError before it reaches this ABI).
 *   L   N x N graph Laplacian CSR (int64 offsets, int64 columns, float64
 *       values), exactly as sdakit builds it (graph.py:191-195): -1 off the
 *       diagonal, the degree on it.  Off-diagonals other than -1 are rejected
 *       with FSDA_EINVAL (weighted graphs are out of scope).
 *   labels  int8 in {+1, -1, 0}, labeled rows first (sda.py:97-101).
 *
 * Status codes (mapped to the reference's exceptions by the host layer):
 *   FSDA_OK         0
 *   FSDA_EINVAL     1  bad argument             -> ValueError
 *   FSDA_EBREAKDOWN 2  <p, Bp> == 0             -> SolverBreakdownError   (krylov.py:215-216)
 *   FSDA_ENONFINITE 3  non-finite <p,Bp> or r.r -> NumericalFailureError  (krylov.py:213-214, 234-235)
 *   FSDA_ECUDA      4  CUDA / NCCL failure      -> RuntimeError
 *   FSDA_ELABEL     5  no labeled sample        -> LabelError             (sparse.py:258-265)
 * fsda_last_error() returns a thread-local message for the last failure.
 *
 * Arithmetic: fp64 throughout.  The projection scores X W and the fsda_matvec
 * probe are sequential in stored column order, bit-identical to scipy's
 * csr_matvec; every other sum (X p and L y rows inside the solve, X^T z
 * columns, dots, norms, class sums) uses the fixed "R256" reduction tree
 * documented in DESIGN.md §4, so results are bitwise reproducible run to run
 * and are mirrored exactly by oracle/fsda_oracle.c.
 */
#ifndef FSDA_B200_H
#define FSDA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSDA_OK 0
#define FSDA_EINVAL 1
#define FSDA_EBREAKDOWN 2
#define FSDA_ENONFINITE 3
#define FSDA_ECUDA 4
#define FSDA_ELABEL 5

/* Largest shift grid one solve accepts (per-shift scalars live in shared memory). */
#define FSDA_MAX_SHIFTS 4096

typedef struct fsda_ctx fsda_ctx;

/* ABI version, bumped on any signature change. */
int fsda_abi_version(void);

/* Thread-local description of the last non-zero status. */
const char* fsda_last_error(void);

/* Host helper: 1 when every one of the n stored values equals 1.0 (the
 * value-free device path needs a binary X; sparse.py:43-58 stores explicit
 * float64 values), else 0.  All host threads; no device work. */
int fsda_values_all_ones(const double* values, int64_t n);

/* One context per device.  Calls on a context are serialized by a mutex and
 * are synchronous unless named *_async.  `stream` may be NULL (the context
 * creates its own) or a cudaStream_t owned by the caller (e.g. torch's
 * current stream), so callers can time launches with their own events. */
int fsda_ctx_create(fsda_ctx** out, int device, void* stream);
int fsda_ctx_destroy(fsda_ctx* ctx);
int fsda_ctx_set_stream(fsda_ctx* ctx, void* stream);

/* Upload X (replaces SparseMatrix construction + the scipy handle,
 * sparse.py:70-114).  Builds the device CSR (int32 columns) and a CSC copy by
 * a stable device sort, so rows stay ascending inside every column, plus the
 * column work plan used by the X^T kernels. */
int fsda_upload_x(fsda_ctx* ctx, int64_t n_rows, int64_t n_cols,
                  const int64_t* row_offsets, const int64_t* col_indices);

/* Upload the Laplacian L = D - S (graph.py:191-195).  N must equal X's rows. */
int fsda_upload_laplacian(fsda_ctx* ctx, int64_t n, const int64_t* row_offsets,
                          const int64_t* col_indices, const double* values);

/* Ternary labels, N entries, labeled-first (LabelVector, sparse.py:198-235). */
int fsda_set_labels(fsda_ctx* ctx, const int8_t* labels);
/* X, L and labels in one call (what fsda_solve's caller uploads every time):
 * the same checks and results as fsda_upload_x + fsda_upload_laplacian +
 * fsda_set_labels, with L's host->device copies queued on a second stream
 * behind X's so they cross the link while X's CSC and plans are built. */
int fsda_upload_problem(fsda_ctx* ctx, int64_t n_rows, int64_t n_cols, const int64_t* x_offsets,
                        const int64_t* x_cols, const int64_t* l_offsets, const int64_t* l_cols,
                        const double* l_values, const int8_t* labels);
/* Labels as an arbitrary mask (no labeled-first requirement): the batched
 * label-mask solves of nested cross-validation (evaluation.py:110-123 permutes
 * every fold to labeled-first instead; the result is the same operator). */
int fsda_set_label_mask(fsda_ctx* ctx, const int8_t* labels);

/* ---- single products, host buffers in and out (parity probes) ---------- */
/* y = X v                         SparseMatrix.matvec            sparse.py:116-121 */
int fsda_matvec(fsda_ctx* ctx, const double* v, double* y);
/* u = X^T w                       SparseMatrix.matvec_transpose  sparse.py:123-134 */
int fsda_matvec_transpose(fsda_ctx* ctx, const double* w, double* u);
/* mu = X^T 1_l / l                labeled_mean                   sparse.py:258-265 */
int fsda_labeled_mean(fsda_ctx* ctx, double* mu);
/* u = X^T w - mu * sum(w)         centered_matvec_transpose      sparse.py:274-277 */
int fsda_centered_matvec_transpose(fsda_ctx* ctx, const double* mu, const double* w, double* u);
/* z = [(1-a)(I_l + 0) + a L] y    apply_smoother                 sda.py:131-140 */
int fsda_apply_smoother(fsda_ctx* ctx, double alpha, const double* y, double* z);
/* q = (X - 1 mu^T)^T M X w        fsda_operator                  sda.py:162-174 */
int fsda_operator_apply(fsda_ctx* ctx, double alpha, const double* w, double* q);

/* ---- the hot path ------------------------------------------------------- */
/* Full FSDA regularization sweep (fsda_solve, sda.py:293-320): labeled mean,
 * rhs = X_c^T (W + 0) X probe, shifted CG over the whole beta grid
 * (krylov.py:168-281) with one operator application per iteration, then the
 * per-shift projections s = X w with sign orientation (sda.py:265-284).
 *   betas          n_shifts, strictly ascending, >= 0 (ShiftGrid, krylov.py:69-90)
 *   probe          D doubles, the reference's rng.uniform(-1, 1, D) draw (sda.py:300)
 *   directions     n_shifts x D (row s = w for betas[s]), oriented
 *   scores         n_shifts x N (row s = X w), oriented; may be NULL
 *   residuals      n_shifts   iterations  n_shifts   converged  n_shifts
 *   n_applies      operator applications (LinearOperator.n_applies, krylov.py:54-56)
 *   fail_iter      iteration index of a breakdown / non-finite failure, else -1 */
int fsda_solve(fsda_ctx* ctx, double alpha, const double* betas, int n_shifts,
               double tol, int64_t max_iter, const double* probe,
               double* directions, double* scores, double* residuals,
               int64_t* iterations, uint8_t* converged, int64_t* n_applies,
               int64_t* fail_iter);

/* Shift-update mode of the shifted-CG solves on this context (krylov.py:230,
 * 240-241).  1: every iteration streams sols_s -= gamma_s P_s and
 * P_s = zeta_next r + alpha_s P_s over all D elements of every active shift.
 * 2 (deferred): the residuals r_0 .. r_K are kept, each iteration updates
 * only the coefficient rows of P_s and sols_s in that basis, and the
 * directions sols_s = sum_j c_s[j] r_j are formed once after the loop
 * (ascending j).  0 (default): 2 when the basis fits a quarter of the free
 * device memory, else 1.  Both are mirrored by oracle/fsda_oracle.c. */
int fsda_set_shift_update_mode(fsda_ctx* ctx, int mode);
/* The mode (1 or 2) the last solve on this context used. */
int fsda_last_shift_update_mode(fsda_ctx* ctx);

/* Storage precision of the FSDA solve's vectors (BASELINE cfg5: "fp32 storage
 * with fp64 reductions").  64 (default): fp64 throughout.  32: the gathered
 * and iterated vectors y = X p, z = M y, p and the residuals r_j are stored as
 * float; every sum and dot runs in double over the stored values; q, mu, the
 * rhs, the directions, the scores and every scalar stay double.  Parity gate
 * (stated): directions within 1e-3 per shift of the fp64 solve and identical
 * labeled AUC at the stable Krylov dimension.  Implies the deferred
 * shift-update mode.  Applies to fsda_solve / fsda_solve_async and to
 * fsda_solve_batch (P, Y, Z and the residual basis of every task as floats;
 * each task equals its single fp32-storage solve bit for bit). */
int fsda_set_storage(fsda_ctx* ctx, int bits);

/* 1: launch each solve's kernels one by one from the host (the same kernels,
 * the same results) instead of the cached CUDA graph with its conditional
 * WHILE node — for profilers that cannot see into conditional graphs.  The
 * default comes from FSDA_B200_EAGER at context creation. */
int fsda_set_eager(fsda_ctx* ctx, int eager);

/* Device-resident variant for throughput measurement: launches one complete
 * solve on the context stream and returns without copying results to the
 * host (inputs already resident in HBM).  Results stay in the context and can
 * be fetched with fsda_fetch_results.  The probe is uploaded once by
 * fsda_prepare_resident.  `launches` receives the number of kernels the solve
 * launched (summed over loop iterations) after fsda_fetch_results. */
int fsda_prepare_resident(fsda_ctx* ctx, double alpha, const double* betas, int n_shifts,
                          double tol, int64_t max_iter, const double* probe);
int fsda_solve_async(fsda_ctx* ctx);
int fsda_fetch_results(fsda_ctx* ctx, double* directions, double* scores, double* residuals,
                       int64_t* iterations, uint8_t* converged, int64_t* n_applies,
                       int64_t* fail_iter, int64_t* launches);

/* Per-kernel device time of one solve, measured with CUDA events around each
 * kernel launched eagerly (not from the graph) on the context stream.
 * names/ms/bytes receive up to max_kernels entries: kernel name, mean ms per
 * launch, algorithmic bytes per launch, launches per solve.  Returns the count
 * in *n_kernels. */
int fsda_profile_kernels(fsda_ctx* ctx, int max_kernels, int* n_kernels,
                         const char** names, double* ms_per_launch,
                         double* bytes_per_launch, int64_t* launches_per_solve);

/* Shifted CG on a dense symmetric operator held on the device
 * (shifted_cg with LinearOperator.from_dense, krylov.py:61-66, 168-281).
 * Same device recurrence kernels as fsda_solve; used to run the reference's
 * own shifted-CG tests against the device path.  solutions is n_shifts x dim. */
int fsda_shifted_cg_dense(fsda_ctx* ctx, int64_t dim, const double* a, const double* b,
                          const double* betas, int n_shifts, double tol, int64_t max_iter,
                          int absolute_tol, double* solutions, double* residuals,
                          int64_t* iterations, uint8_t* converged, int64_t* n_applies,
                          int64_t* fail_iter);

/* Regression-phase shifted solve: (X^T X + beta I) w = rhs for
 * every beta at once (shifted_cg(regression_operator(p), rhs, ...),
 * sda.py:177-179, 339, 439-442; bench_shifted, evaluation.py:288-291), with
 * the same device recurrence and graph loop as fsda_solve.  solutions is
 * n_shifts x D; rhs is D doubles (host). */
int fsda_regression_shifted_cg(fsda_ctx* ctx, const double* rhs, const double* betas,
                               int n_shifts, double tol, int64_t max_iter, int absolute_tol,
                               double* solutions, double* residuals, int64_t* iterations,
                               uint8_t* converged, int64_t* n_applies, int64_t* fail_iter);

/* SA-SDA (sda.py:360-396): shifted CG in sample space on the
 * centred spectral operator z -> M z - 1_l sum(M z) / l (sda.py:148-159),
 * rhs = apply_w(probe) with probe the orthogonalized draw (sda.py:287-290,
 * computed by the caller on the host: N doubles).  solutions (n_shifts x N)
 * come back oriented (sda.py:256-262, 375-380); alpha == 0 is rejected with
 * FSDA_EINVAL as the reference does. */
int fsda_sa_solve(fsda_ctx* ctx, double alpha, const double* betas, int n_shifts, double tol,
                  int64_t max_iter, const double* probe, double* solutions, double* residuals,
                  int64_t* iterations, uint8_t* converged, int64_t* n_applies, int64_t* fail_iter);

/* Multi-task batch: n_tasks FSDA sweeps on the
 * uploaded X and L, task t with its own label mask labels[t * N .. t * N + N)
 * (any row order, as fsda_set_label_mask) and probe probes[t * D ..].  One
 * operator pass serves every task (task-minor vectors, coalesced row
 * gathers); each task's results equal, bit for bit, fsda_set_label_mask +
 * fsda_solve of that task.  Outputs: directions [T][n_shifts][D], scores
 * [T][n_shifts][N] (may be NULL), residuals / iterations / converged
 * [T][n_shifts], n_applies / fail_iter / status [T] (status: FSDA_OK,
 * FSDA_EBREAKDOWN or FSDA_ENONFINITE per task; a failed task does not stop
 * the others).  Honours fsda_set_storage (32: fp32 storage, each task equal
 * to its single fp32-storage solve).  Limit: a task-minor vector, (max(N, D)
 * + 1) x tasks padded to 32 x 8 bytes, must stay below 4 GiB (32-bit gather
 * offsets); larger batches are split by the caller.  Replaces the per-fold
 * fsda_solve calls of nested_cv (evaluation.py:110-123, 173-237). */
int fsda_solve_batch(fsda_ctx* ctx, int n_tasks, const int8_t* labels, double alpha,
                     const double* betas, int n_shifts, double tol, int64_t max_iter,
                     const double* probes, double* directions, double* scores,
                     double* residuals, int64_t* iterations, uint8_t* converged,
                     int64_t* n_applies, int64_t* fail_iter, int* status);

/* ---- row-sharded building blocks ---------------------------
 * One context per GPU holds a contiguous row block [row_base, row_base+N_g)
 * of X (uploaded with fsda_upload_x as an N_g x D matrix) and of L
 * (fsda_upload_laplacian_rows: N_g rows, global column indices), plus the
 * block's labels.  The host orchestrator (paper_1709_04794_b200/sharded.py)
 * strings these together with NCCL all-gathers of y and all-reduces of the
 * D-length X^T partials; D-vectors and the shift state are replicated, so
 * every rank runs the identical recurrence.  All pointers named d_* are
 * device pointers on the context's device; calls are asynchronous on the
 * context stream unless they return host data. */
int fsda_upload_laplacian_rows(fsda_ctx* ctx, int64_t n_local, int64_t n_global, int64_t row_base,
                               const int64_t* row_offsets, const int64_t* col_indices,
                               const double* values);
/* d_y (N_g) = X_g d_v (D), rows summed by the canonical tree */
int fsda_dev_xrows(fsda_ctx* ctx, const double* d_v, double* d_y);
/* d_z (N_g) = [(1-a)(I_l + 0) + a L_g] d_y_full (N_global) */
int fsda_dev_smoother(fsda_ctx* ctx, double alpha, const double* d_y_full, double* d_z);
/* d_out[0..D) = X_g^T d_z (raw column sums), d_out[D] = sum(d_z) (canonical) */
int fsda_dev_xt_partial(fsda_ctx* ctx, const double* d_z, double* d_out);
/* d_out[0] = sum of d_t over class +1 rows, d_out[1] = over class -1 rows */
int fsda_dev_class_sums(fsda_ctx* ctx, const double* d_t, double* d_out);
/* d_w = class-mean broadcast (c1 on +1 rows, c2 on -1 rows, else 0) */
int fsda_dev_apply_w(fsda_ctx* ctx, double c1, double c2, double* d_w);
/* d_out[i] = d_q[i] - d_mu[i] * d_q[D]   (centring of an all-reduced partial) */
int fsda_dev_center(fsda_ctx* ctx, const double* d_mu, double* d_q, double scale);
/* shifted CG state on the context: reset + init from the device rhs d_b */
int fsda_dev_cg_begin(fsda_ctx* ctx, const double* betas, int n_shifts, double tol,
                      int64_t max_iter, const double* d_b);
/* one iteration given the (centred, all-reduced) d_q = B p */
int fsda_dev_cg_step(fsda_ctx* ctx, const double* d_q);
/* device pointer of the current search direction p (D doubles) */
int fsda_dev_cg_direction(fsda_ctx* ctx, const double** d_p);
int fsda_dev_cg_status(fsda_ctx* ctx, int* finished, int64_t* iterations, int* status);
/* projections of the local rows: d_scores (n_shifts x N_g), d_orient[s] = y_g . s_g */
int fsda_dev_project(fsda_ctx* ctx, double* d_scores, double* d_orient);
/* finish: flip the shifts whose all-reduced orientation is negative (host
 * array flip[n_shifts]) in d_scores and the directions, copy results out */
int fsda_dev_finish(fsda_ctx* ctx, const uint8_t* flip, double* d_scores, double* directions,
                    double* residuals, int64_t* iterations, uint8_t* converged,
                    int64_t* n_applies, int64_t* fail_iter);

/* ---- Tanimoto k-NN graph
 * Replaces sdakit.graph.knn_graph (graph.py:152-166: _knn_rows_block
 * graph.py:79-111, union symmetrization _adjacency_from_pairs
 * graph.py:141-149) for the X uploaded by fsda_upload_x (its support
 * pattern).  Row i keeps its k most similar rows j != i sharing a feature,
 * ranked by (Tanimoto descending, index ascending), padded with the lowest
 * unused indices; the result is the union of both directions.  1 <= k <= 64
 * and k < n_rows, else FSDA_EINVAL (the reference raises GraphError).  The
 * symmetric adjacency stays on the context; *nnz_out = its stored entries. */
int fsda_graph_knn(fsda_ctx* ctx, int32_t k, int64_t* nnz_out);
/* Replaces sdakit.graph.threshold_graph (graph.py:169-188,
 * _threshold_rows_block graph.py:114-133): every pair of distinct rows with
 * Tanimoto >= theta, 0 < theta <= 1 (else FSDA_EINVAL; the reference raises
 * GraphError).  Result kept on the context like fsda_graph_knn's. */
int fsda_graph_threshold(fsda_ctx* ctx, double theta, int64_t* nnz_out);
/* Copy the last graph out: row_offsets (n_rows + 1) and col_indices (nnz),
 * int64 CSR with ascending columns (graph.py:146-148's from_scipy layout). */
int fsda_graph_fetch(fsda_ctx* ctx, int64_t* row_offsets, int64_t* col_indices);
/* The graph builds' head-count contraction on its own, for tests: for an
 * n_rows x h 0/1 int8 matrix a (row-major), counts[b * n_rows + j] =
 * sum_k a[r0 + b][k] * a[j][k] for b < nb, j < n_rows (h <= 65535) — the block
 * of exact counts (16-bit on the device) the builds take from the hand-written tcgen05 GEMM
 * (csrc/graph_gemm.cuh; the reference's per-block X_blk X^T, graph.py:79-111).
 * Uses the context's device and stream. */
int fsda_head_counts(fsda_ctx* ctx, int64_t n_rows, int32_t h, const int8_t* a, int64_t r0, int64_t nb,
                     int32_t* counts);

/* ---- row-sharded solve (csrc/fsda_shard.cuh) -------------------
 * One FSDA sweep with the rows of X and L split into contiguous blocks over
 * `world` ranks.  Per iteration: an all-gather of y, a deterministic
 * reduce-scatter (send/recv, rank-ordered owner sum) + all-gather of the
 * D + 1 partials [X_g^T z_g | sum z_g]; D-vectors and scalars replicated.
 * Replaces the single-process fsda_solve of sda.py:293-320 when the problem
 * is spread over GPUs (the reference has no multi-node path).
 *
 * Set-up per rank: fsda_upload_x(local rows), fsda_upload_laplacian_rows(
 * n_local, world * slot, rank * slot, offsets, REMAPPED columns, values) with
 * slot = max rows per rank rounded up to even and global column j of rank h
 * remapped to h * slot + (j - bounds[h]); fsda_set_label_mask(local labels);
 * then fsda_shard_init. */

/* A fresh ncclUniqueId (128 bytes) for fsda_shard_init (rank 0 draws it and
 * broadcasts it).  NCCL is loaded at run time (libnccl.so.2). */
int fsda_nccl_unique_id(uint8_t* out);

/* Make ctx rank `rank` of `world` with rows [row_bounds[rank],
 * row_bounds[rank+1]).  nccl_id: 128 bytes (one process per GPU, NCCL over
 * NVLink), or NULL for a local group (all ranks driven by one process — the
 * multi-rank tests on one GPU). */
int fsda_shard_init(fsda_ctx* ctx, int world, int rank, const int64_t* row_bounds,
                    const uint8_t* nccl_id);

/* One row-sharded sweep.  ctxs: this process's NCCL rank (n_ctx 1), or all
 * `world` contexts of a local group in rank order.  probe (D) and betas are
 * replicated; n1 / n2 are the global class counts.  directions: n_shifts x D
 * (replicated); scores: n_shifts x rows_total of the driven ranks' rows (rank
 * blocks side by side per shift).  At world 1 the results equal fsda_solve's
 * bit for bit. */
int fsda_solve_sharded(fsda_ctx** ctxs, int n_ctx, double alpha, const double* betas,
                       int n_shifts, double tol, int64_t max_iter, const double* probe, int64_t n1,
                       int64_t n2, double* directions, double* scores, double* residuals,
                       int64_t* iterations, uint8_t* converged, int64_t* n_applies,
                       int64_t* fail_iter);

#ifdef __cplusplus
}
#endif

#endif /* FSDA_B200_H */
