/*
 * gpspca_b200.h -- C ABI of the B200-native GP-SPCA engine (libgpspca_b200.so).
 *
 * The reference (`gpspca` 0.1.0, /root/reference/pkg/src/gpspca) is a pure
 * Python/NumPy package with no FFI; its GPU "extension seam" is the kernel
 * set named in SPEC.md:424 (par_matvec_t, par_gram_apply,
 * par_threshold_accumulate, dense SVD) plus the solver loops that call it.
 * Each entry point below cites the reference interface it replaces
 * (path:line relative to /root/reference/pkg/src/gpspca/).  Plain C types
 * only: host buffers are caller-owned, device memory is owned by the
 * library objects, calls are stream-ordered on the context's stream and
 * BLOCKING at return unless the name says `enqueue`.
 *
 * Layout: A is p x n, column-major, column i contiguous (core.py:36,52-54),
 * stored on the device with a padded leading dimension ld = roundup(p, 32)
 * and zero padding rows.  Iterates x (length p) and all reductions are fp64.
 *
 * Error model (mapped by the Python host to the reference's exceptions):
 *   GPS_E_ARG      -> ValueError           (shape / argument / finiteness)
 *   GPS_E_RANK     -> RankDeficiencyError  (block.py:33-49)
 *   GPS_E_OOM      -> MemoryError          (parallel.py:145-156 analogue)
 *   GPS_E_CUDA     -> RuntimeError
 *   GPS_E_UNSUPPORTED -> NotImplementedError (shape outside the built kernels)
 * gps_last_error() returns a thread-local message for the last failure.
 */
#ifndef GPSPCA_B200_H
#define GPSPCA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum gps_status {
  GPS_OK = 0,
  GPS_E_ARG = 1,
  GPS_E_RANK = 2,
  GPS_E_OOM = 3,
  GPS_E_CUDA = 4,
  GPS_E_UNSUPPORTED = 5
};
enum gps_dtype { GPS_F32 = 0, GPS_F64 = 1 };
enum gps_penalty { GPS_L1 = 0, GPS_L0 = 1 }; /* core.py:13 PENALTIES */

typedef struct gps_ctx gps_ctx;       /* one device + one stream            */
typedef struct gps_matrix gps_matrix; /* device-resident DataMatrix         */
typedef struct gps_su gps_su;         /* single-unit solver state           */
typedef struct gps_bk gps_bk;         /* block solver state                 */

/* ---- library / context ------------------------------------------------ */
int gps_version(void);
const char* gps_last_error(void);
int gps_device_count(int* count);
/* Free device memory of the context's GPU (parallel.py:145-157
 * check_allocation, on HBM instead of host RAM). */
int gps_device_free_bytes(gps_ctx* ctx, size_t* free_out);
int gps_ctx_create(int device, gps_ctx** out);
int gps_ctx_destroy(gps_ctx* ctx);
/* Use a caller stream (e.g. a torch.cuda.Stream's cuda_stream; not the legacy
 * default stream, which cannot be graph-captured).  NULL restores a
 * library-owned stream. */
int gps_ctx_set_stream(gps_ctx* ctx, void* cuda_stream);
int gps_ctx_sync(gps_ctx* ctx);
/* Number of kernels this context launched so far (instrumentation). */
int64_t gps_ctx_launch_count(gps_ctx* ctx);

/* ---- data matrix: core.py:25-68 DataMatrix / as_data_matrix ------------ */
/* Copies a host column-major p x n matrix (leading dimension ld_src >= p)
 * into device memory.  dtype selects the device storage (GPS_F32 keeps an
 * fp32 input in fp32; reductions are always fp64). */
int gps_matrix_create(gps_ctx* ctx, const void* host, int64_t p, int64_t n, int64_t ld_src, int dtype,
                      gps_matrix** out);
/* Same, from a DEVICE column-major buffer (copied into padded storage). */
int gps_matrix_create_device(gps_ctx* ctx, const void* dev_src, int64_t p, int64_t n, int64_t ld_src, int dtype,
                             gps_matrix** out);
/* Adopt caller device memory without a copy: column-major, ld ==
 * roundup(p, 32) with ZERO padding rows, 128-byte aligned; the caller keeps
 * it alive and unmodified until gps_matrix_destroy. */
int gps_matrix_wrap_device(gps_ctx* ctx, void* dev_ptr, int64_t p, int64_t n, int64_t ld, int dtype,
                           gps_matrix** out);
/* Same, from a host ROW-major p x n buffer (C order), transposed on device. */
int gps_matrix_create_rowmajor(gps_ctx* ctx, const void* host, int64_t p, int64_t n, int dtype,
                               gps_matrix** out);
int gps_matrix_destroy(gps_matrix* A);
int gps_matrix_info(const gps_matrix* A, int64_t* p, int64_t* n, int64_t* ld, int* dtype);
/* Device copy back to a host column-major buffer with leading dimension p. */
int gps_matrix_download(gps_matrix* A, void* host);
/* Column i as fp64 (length p) -- core.py:52-54 DataMatrix.column. */
int gps_matrix_column(gps_matrix* A, int64_t i, double* out);
/* Device pointer of the padded storage (for callers that own a stream). */
void* gps_matrix_device_ptr(gps_matrix* A);

/* core.py:243-246 column_norms + core.py:42 isfinite check, one pass (K0).
 * Results are cached on the matrix; norms_out may be NULL. */
int gps_column_norms(gps_matrix* A, double* norms_out, int* nonfinite_out);

/* single_unit.py:287-296 deflate: new fp64 matrix (I - xx')A (x unit). */
int gps_matrix_deflate(gps_matrix* A, const double* x, gps_matrix** out);
/* core.py:234-240 center_columns: a new fp64 matrix A - 1 mean' (column
 * means in means_out, optional, length n). */
int gps_matrix_center(gps_matrix* A, double* means_out, gps_matrix** out);

/* Columns idx[0..k) as a new matrix (support-restricted power iteration,
 * single_unit.py:219-230 `A.values[:, support]`). */
int gps_matrix_gather(gps_matrix* A, const int64_t* idx, int64_t k, gps_matrix** out);

/* Instrumentation: mean ms of the K0 read-only streaming pass over A. */
int gps_bench_read_stream(gps_matrix* A, int iters, double* ms_out);

/* ---- kernel seam: parallel.py:85-142 ----------------------------------- */
int gps_matvec_t(gps_matrix* A, const double* x, double* c_out);               /* parallel.py:85  */
int gps_gram_apply(gps_matrix* A, const double* coef, double* out);            /* parallel.py:108 */
int gps_threshold_accumulate(gps_matrix* A, const double* c, double gamma,     /* parallel.py:131 */
                             int penalty, double* out);
/* One fused sweep at x: f = objective (single_unit.py:44-48), g_half =
 * sum_i w(a_i'x) a_i (the ascent direction / 2, single_unit.py:67-81),
 * optional c = A'x and w = threshold(c) (single_unit.py:100-121 before
 * normalisation).  Any output may be NULL. */
int gps_su_sweep(gps_matrix* A, const double* x, double gamma, int penalty, double* f_out,
                 double* g_half_out, double* c_out, double* w_out, int64_t* nnz_out);

/* ---- single-unit power iteration: single_unit.py:160-181 --------------- */
/* tol = 0 disables the relative-change test (benchmarking fixed-length loops). */
int gps_su_create(gps_matrix* A, int penalty, double gamma, double tol, int max_iter, gps_su** out);
int gps_su_destroy(gps_su* s);
/* Reset the loop at x0 (length p, unit norm). */
int gps_su_start(gps_su* s, const double* x0);
/* Implicit deflation (single_unit.py:287-296 without rewriting A): the
 * step projects the gradient off the k orthonormal columns of X (p x k,
 * column-major), applied in column order. k = 0 disables. */
int gps_su_set_deflation(gps_su* s, const double* X, int k);
/* Native single-device loop: device-resident iterate, history and stopping
 * rule; the host polls the control block every poll_every iterations. */
int gps_su_run(gps_su* s, int poll_every);
/* Building blocks for a multi-rank loop (column shards): sweep + local
 * reduce into the exchange vector [g (ld) | f | nnz | sum w^2 | 0]; the
 * caller all-reduces it (sum) across ranks; then the step. */
int gps_su_enqueue_sweep(gps_su* s);
int gps_su_exchange(gps_su* s, void** dev_ptr, int64_t* count);
/* Use a caller-owned device buffer (ld + 4 doubles) as the exchange vector,
 * e.g. a torch tensor handed to an NCCL all-reduce. */
int gps_su_set_exchange(gps_su* s, void* dev_ptr);
int gps_su_enqueue_step(gps_su* s);
/* Fine-grained enqueue for instrumentation: bit 1 sweep kernel, bit 2 the
 * cross-CTA reduction, bit 4 the step (gps_su_enqueue_sweep == mask 3). */
int gps_su_enqueue(gps_su* s, int mask);
/* Copies the control block to the host (synchronises the stream). */
int gps_su_poll(gps_su* s, int* done, int* iter, int* converged);
/* Results of the finished loop: x (p), history (n_hist <= max_iter+1),
 * the weights w of the final sweep (n; z = w / ||w||), sum w^2. */
int gps_su_result(gps_su* s, double* x_out, double* hist_out, int* n_hist, int* converged, double* w_out,
                  double* w_sumsq_out);
/* Kernel launches per power iteration of gps_su_run (instrumentation). */
int gps_su_launches_per_iter(gps_su* s);
/* Near-threshold log of the final sweep (north_star: support entries within
 * 1e-6 gamma of the threshold are logged; thresholds of parallel.py:117-128):
 * entries col * 64 + component with ||c| - gamma| <= 1e-6 gamma (l1) or
 * |c^2 - gamma| <= 1e-6 gamma (l0); *count_out = entries found (the first
 * min(count, cap, 8192) are copied). */
int gps_su_band(gps_su* s, int64_t* entries_out, int cap, int* count_out);

/* ---- block power iteration: block.py:190-235 ---------------------------- */
/* m <= 64 components; gamma, mu: length m (mu_j > 0, gamma_j >= 0).  Each
 * iteration runs ceil(m/MG) fused sweeps (MG = 4 for fp32 storage with
 * p <= 4096, else 2) and the device polar step. */
int gps_bk_create(gps_matrix* A, int penalty, int m, const double* gamma, const double* mu, double tol,
                  int max_iter, gps_bk** out);
int gps_bk_destroy(gps_bk* s);
/* Starts: X0 used as is (p x m column-major, user_supplied, block.py:160-161);
 * M orthonormalised by device CholeskyQR2 (random_orthonormal, block.py:155,
 * 162-170); columns idx[0..m) of A, then CholeskyQR2 (max_norm_column,
 * block.py:157-158).  A rank-deficient start returns GPS_E_ARG. */
int gps_bk_start(gps_bk* s, const double* X0);
int gps_bk_start_qr(gps_bk* s, const double* M);
int gps_bk_start_columns(gps_bk* s, const int64_t* idx);
int gps_bk_run(gps_bk* s, int poll_every);
int gps_bk_enqueue_sweep(gps_bk* s);
int gps_bk_exchange(gps_bk* s, void** dev_ptr, int64_t* count);
int gps_bk_set_exchange(gps_bk* s, void* dev_ptr);
int gps_bk_enqueue_step(gps_bk* s);
int gps_bk_poll(gps_bk* s, int* done, int* iter, int* converged);
/* X (p x m), history, W of the final sweep (m columns of length n, for
 * Z_j = W_j / ||W_j||, block.py:174-187), rank_fail = 1 when the polar step
 * found rank(G) < m at iteration n_hist - 1 (block.py:215-218). */
int gps_bk_result(gps_bk* s, double* X_out, double* hist_out, int* n_hist, int* converged, double* W_out,
                  int* rank_fail, int* rank_out);
/* Per-iterate ||X_k'X_k - I||_F for k = 0 .. n_hist - 1 (the StiefelPoint
 * every polar output becomes, block.py:149 / core.py:113-129; a value above
 * 1e-10 stops the loop with status 3, the reference's ValueError), the
 * loop status (0 running / converged / max_iter, 2 rank loss, 3 Stiefel
 * violation) and the number of steps the exact Householder + Jacobi polar
 * path took. */
int gps_bk_diagnostics(gps_bk* s, double* stiefel_out, int* status_out, int* exact_steps_out);
/* Objective and active (column, component) count of the most recent sweep
 * (instrumentation; the loop may still be running). */
int gps_bk_last_sweep(gps_bk* s, double* f_out, double* nnz_out);
/* Near-threshold log of the final block sweep: entries col * 64 + j with
 * the mu-scaled correlation s = mu_j c_ij within 1e-6 gamma_j of the
 * threshold (block.py:80-89 rules); as gps_su_band. */
int gps_bk_band(gps_bk* s, int64_t* entries_out, int cap, int* count_out);
/* One-shot block sweep at X (p x m): objective (block.py:80-111), ascent
 * direction G = 2 mu_j sum_i w a_i (block.py:114-132), optional W (n x m). */
int gps_bk_sweep(gps_matrix* A, const double* X, int m, const double* gamma, const double* mu, int penalty,
                 double* f_out, double* G_out, double* W_out);
/* block.py:135-149 polar_projection on the device: X = G (G'G)^{-1/2};
 * GPS_E_RANK (rank in *rank_out) when rank(G) < m by the reference rule. */
int gps_polar(gps_ctx* ctx, const double* G, int64_t p, int m, double* X_out, int* rank_out);
/* The same polar factor through the block loop's multi-CTA step (CholeskyQR2
 * + Newton-Schulz, Stiefel check, exact Householder + Jacobi fallback; used
 * in the loop for p m >= 4096): ||X'X - I||_F in *stiefel_out, 1 in
 * *exact_out when the exact path took the step. */
int gps_polar_cholqr2(gps_ctx* ctx, const double* G, int64_t p, int m, double* X_out, int* rank_out,
                      double* stiefel_out, int* exact_out);

/* ---- peer-memory all-reduce of the sharded loops ------------------------
 * the one exchange per power iteration of the column-sharded
 * solves (the sum over ranks of the exchange vector, gps_su_exchange /
 * gps_bk_exchange), done by ONE kernel per rank over NVLink peer memory (the
 * reference has no multi-GPU path; this replaces an NCCL all-reduce).  One
 * process per GPU: each rank creates a gps_px with the same world / count,
 * exports its buffer with gps_px_ipc_handle (gps_px_handle_size() bytes),
 * the caller exchanges the handles (e.g. torch.distributed.all_gather_object)
 * and opens every peer's.  gps_px_allreduce enqueues buf (count doubles,
 * device) <- sum over ranks in rank order (identical on every rank) on the
 * context's stream; every rank must issue the same sequence of calls. */
typedef struct gps_px gps_px;
int gps_px_create(gps_ctx* ctx, int world, int rank, int64_t count, gps_px** out);
int gps_px_handle_size(void);
int gps_px_ipc_handle(gps_px* px, void* handle);
int gps_px_open(gps_px* px, int peer, const void* handle);
int gps_px_allreduce(gps_px* px, double* buf);
/* The two halves of one exchange as separate launches (phase 1: push this
 * rank's vector into every rank's slots and release the epoch flags; phase 2:
 * wait for every rank's flags, rank-order sum, publish the epoch; 3: both =
 * gps_px_allreduce).  gps_px_reduce_phase does the same for the fused
 * reduction kernel (su_reduce_px_kernel) on given CTA partials part_g
 * [nparts][rows], part_s [nparts_s][4] into exch [rows + 4].  Used by the
 * cross-process test that runs several ranks on ONE GPU: with a host barrier
 * between the phases no rank's kernel waits on another process's kernel. */
int gps_px_allreduce_phase(gps_px* px, double* buf, int phase);
int gps_px_reduce_phase(gps_px* px, const double* part_g, const double* part_s, int nparts, int rows, int nparts_s,
                        double* exch, int phase);
/* Bound (seconds) on every peer-flag wait of this exchange; default
 * GPSPCA_PX_TIMEOUT_S or 60 s.  A wait that expires raises the exchange's
 * error flag (gps_px_error) and stops the attached loop, whose run / poll
 * then return GPS_E_CUDA instead of every GPU spinning forever. */
int gps_px_set_timeout(gps_px* px, double seconds);
int gps_px_error(gps_px* px, int* error_out);
/* Test: rank 0 of a world-`world` exchange whose peers never arrive must
 * time out after timeout_s with the error flag set (*error_out = 1). */
int gps_px_emulate_timeout(gps_ctx* ctx, int world, int64_t count, double timeout_s, int* error_out);
int gps_px_destroy(gps_px* px);
/* Fuse the exchange into the loop's cross-CTA reduction (K2): with a peer
 * exchange attached (count = gps_su_exchange's count, or ONE group's
 * exchange vector for gps_bk: gps_bk_exchange's count / groups), the K2 kernel
 * itself reduces this rank's partials, stores them into every rank's slots,
 * and sums the ranks' vectors in rank order into the exchange vector -- no
 * separate all-reduce call.  NULL detaches. */
int gps_su_attach_px(gps_su* s, gps_px* px);
int gps_bk_attach_px(gps_bk* s, gps_px* px);
int gps_bk_exchange_stride(gps_bk* s, int64_t* stride); /* one group's exchange length */
/* Test harness: `world` ranks emulated on the context's device as one
 * cooperative kernel; per round k the rank vectors are in (world x count,
 * rank-major) times (k + 1); out receives every round's results
 * (rounds x world x count). */
int gps_px_emulate(gps_ctx* ctx, int world, int64_t count, int rounds, const double* in, double* out);
/* Same for the fused K2: per rank, partials part_g (nparts x rows) and
 * part_s (nparts_s x 4), rank-major; exch_out: rounds x world x (rows + 4). */
int gps_px_emulate_reduce(gps_ctx* ctx, int world, int rows, int nparts, int nparts_s, int rounds,
                          const double* part_g, const double* part_s, double* exch_out);
/* Device CholeskyQR2 of M (p x m): Q with positive-diagonal R (= the
 * reference's sign-fixed QR, block.py:162-170). */
int gps_orthonormalize(gps_ctx* ctx, const double* M, int64_t p, int m, double* Q_out);

/* ---- Recognition path ---------------------------------
 * Y = A C for m coefficient vectors (C: n x m column-major, Y: p x m
 * column-major, host buffers): the building block of project (pca.py:57-71,
 * (S - mean) L with S = A) and explained_variance (pca.py:74-103).  One pass
 * over the columns with a nonzero coefficient row, fp64 accumulation, fixed
 * reduction order. */
int gps_gram_apply_block(gps_matrix* A, const double* C, int m, double* Y_out);
/* Squared row norms of a row-major rows x dim fp64 device matrix. */
int gps_row_sqnorms(gps_ctx* ctx, const double* X_dev, int64_t rows, int dim, double* out_dev);
/* k-NN distances (datasets.py:213-220): dist[t][r] = max((|t|^2 - 2 t.s_r) +
 * |s_r|^2, 0) for the row-major test rows (n_test x dim) against the train
 * rows given column-major (trainT: dim x n_train) with their squared norms;
 * all device pointers on the context's device.  argmin_dev (optional,
 * n_test) receives the first minimal train index per test row (np.argmin,
 * datasets.py:255).  Blocking at return. */
int gps_knn_distances(gps_ctx* ctx, const double* test_dev, int64_t n_test, const double* trainT_dev,
                      int64_t n_train, int dim, const double* train_sqnorm_dev, double* dist_dev,
                      int64_t* argmin_dev);

/* k-NN neighbour selection (datasets.py:258): the k nearest train rows of
 * every test row of the device distance matrix (n_test x n_train), in
 * (distance, index) order like np.argsort(kind="stable")[:, :k]; idx_dev is
 * n_test x k int64 on the device. */
int gps_knn_topk(gps_ctx* ctx, const double* dist_dev, int64_t n_test, int64_t n_train, int k, int64_t* idx_dev);
/* Thin SVD of the device matrix A (p x n) by one-sided Jacobi (pca.py:37-54
 * pca_fit's np.linalg.svd): sigma_out min(p, n) non-increasing singular
 * values, V_out n x min(p, n) column-major right singular vectors, sweeps
 * used in *sweeps_out. */
int gps_matrix_svd(gps_matrix* A, double* sigma_out, double* V_out, int* sweeps_out);

#ifdef __cplusplus
}
#endif
#endif /* GPSPCA_B200_H */
