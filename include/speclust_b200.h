/*
 * speclust_b200 — C ABI of the B200-native spectral-clustering engine.
 *
 * Every entry point takes plain pointers and sizes.  Pointers marked (dev) are
 * CUDA device pointers (any allocator; the Python host uses torch tensors);
 * pointers marked (host) are host memory.  All device work is enqueued on the
 * caller's stream `stream` (a cudaStream_t passed as void*; NULL = legacy
 * default stream).  Functions return an int status (SC_OK or one negative code
 * per error class of the reference's errors.py); sc_last_error() returns the
 * thread-local message of the last failure.
 *
 * The entry points replace the reference's Python operators on the hot path
 * (reference = /root/reference/pkg/src/speclust; see INTEGRATION.md for the
 * ctypes binding the host package uses):
 *
 *   sc_spmv_f64            sparse.py:195-207        spmv(a, x)
 *   sc_degrees_f64         laplacian.py:27-31       degrees(w)
 *   sc_find_nonpositive    laplacian.py:44-52,67-72 handle_isolated / _check_positive
 *   sc_sym_scale_f64       laplacian.py:84-91       sym_scale(w, d)
 *   sc_csr_is_symmetric    sparse.py:210-222        is_symmetric(a)
 *   sc_knn_graph_f64       graph.py:185-237 +       build_edges_knn + build_similarity
 *                          sparse.py:182-187        + coo_to_csr   (exp_decay measure)
 *   sc_lanczos_*           eigen.py:86-266          RciSession / rci_new / rci_advance / rci_extract
 *   sc_eigensolve_csr      eigen.py:269-302         eigensolve(a, cfg) (device-resident loop)
 *   sc_symmetry_probe      eigen.py:279-288         _check_symmetric
 *   sc_recover_embedding   laplacian.py:94-106 +    recover_row_eigvecs (+ normalize_rows,
 *                          pipeline.py:242-245      pipeline stage "kmeans" prologue)
 *   sc_pairwise_sq_dist    kmeans.py:84-98          pairwise_sq_dist(v, c)
 *   sc_kmeanspp_*          kmeans.py:107-136        kmeanspp_init (host supplies the PCG64 draws)
 *   sc_lloyd               kmeans.py:159-196        lloyd(v, init_c, cfg)
 *   sc_ncut                metrics.py:34-67         ncut(w, labels)
 *   sc_partition_cuts      metrics.py:42-56         cut(w, labels), ratio_cut(w, labels)
 *   sc_csr_remove_isolated laplacian.py:34-64       handle_isolated(w, d, "remove")
 *   sc_row_scale_f64       laplacian.py:75-81       row_scale(w, d)
 *   sc_edge_similarity_f64 graph.py:136-147,214-237 build_similarity (cosine, cross_correlation)
 *   sc_pattern_edges_f64   graph.py:160-176,206-211 build_edges_eps, build_edges_threshold
 *   sc_sbm_csr             sbm.py:68-108            sbm_generate (device, distributional parity)
 */
#ifndef SPECLUST_B200_H
#define SPECLUST_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: one per errors.py class on the hot path --------------- */
enum {
    SC_OK = 0,
    SC_ERR_VALUE = -1,           /* ValueError / BadConfig (usage errors)        */
    SC_ERR_DIMENSION = -2,       /* errors.DimensionMismatch                     */
    SC_ERR_FORMAT = -3,          /* errors.InvalidFormat                         */
    SC_ERR_NOT_SQUARE = -4,      /* errors.NotSquare                             */
    SC_ERR_NOT_SYMMETRIC = -5,   /* errors.NotSymmetric                          */
    SC_ERR_ISOLATED = -6,        /* errors.IsolatedNode                          */
    SC_ERR_ZERO_DEGREE = -7,     /* errors.ZeroDegree                            */
    SC_ERR_BREAKDOWN = -8,       /* errors.Breakdown                             */
    SC_ERR_MAX_RESTARTS = -9,    /* errors.MaxRestartsExceeded (payload: stats)  */
    SC_ERR_NOT_CONVERGED = -10,  /* errors.NotConverged                          */
    SC_ERR_STATE = -11,          /* errors.SpeclustError (wrong session state)   */
    SC_ERR_CUDA = -20,           /* CUDA runtime failure                         */
    SC_ERR_NO_MEMORY = -21,      /* device allocation failed                     */
    SC_ERR_INTERNAL = -22        /* numerical kernel failed (e.g. QL no convergence) */
};

typedef void* sc_stream_t;                 /* cudaStream_t */
typedef struct sc_lanczos sc_lanczos_t;    /* opaque RCI session (library-owned) */

const char* sc_last_error(void);
int sc_version(void);
/* number of kernel launches issued by this library since the last reset */
/* return the library's cached device memory (stream-ordered pool) to the
 * driver; the pipeline calls it between stages */
void sc_trim_pool(void);
int64_t sc_launch_count(void);
void sc_launch_count_reset(void);

/* ---- kernel timing (CUDA events on the launching stream) ------------------ */
/* When enabled, launches of the named kernel classes ("spmv", "knn_tile",
 * "reorth", "ritz", "symeig", "kmeans_assign", "kmeans_update", ...) are
 * bracketed by events; sc_profile_query syncs and reports the accumulated
 * device milliseconds, launch count and algorithmic bytes/flops recorded. */
void sc_profile_enable(int on);
void sc_profile_reset(void);
int sc_profile_query(const char* name, double* ms, int64_t* launches, double* work);

/* ---- sparse (CSR: row_ptr int64[n+1], col int32[nnz], vals f64[nnz]) ----- */
/* y = A x.  deterministic=1: each row summed sequentially in column order
 * (bit-identical to sparse.py:205-207); 0: vectorised sub-warp reduction. */
int sc_spmv_f64(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, const int32_t* col,
                const double* vals, const double* x, double* y, int deterministic,
                sc_stream_t stream);
/* d = W 1, rows summed sequentially (laplacian.py:27-31). */
int sc_degrees_f64(int64_t n, const int64_t* row_ptr, const double* vals, double* d,
                   sc_stream_t stream);
/* mode 0: entries == 0.0 (isolated nodes); mode 1: entries <= 0.0.
 * count_out/first_out are HOST pointers; idx_out (dev, optional, capacity
 * max_idx) receives the first max_idx matching indices in ascending order. */
int sc_find_nonpositive(int64_t n, const double* d, int mode, int64_t* count_out,
                        int64_t* idx_out, int64_t max_idx, sc_stream_t stream);
/* out = vals / sqrt(d[row] * d[col]) (laplacian.py:84-91). */
int sc_sym_scale_f64(int64_t n, const int64_t* row_ptr, const int32_t* col,
                     const double* vals, const double* d, double* out, sc_stream_t stream);
/* B = P A P^T: row p of B is row perm[p] of A, columns relabelled pos[c]
 * (pos = perm^-1, see sc_invert_perm) and re-sorted; out_* have A's sizes.
 * Used to run the eigensolver on the locality-ordered operator. */
int sc_csr_permute_f64(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* vals,
                       const int32_t* perm, const int32_t* pos, int64_t* out_row_ptr, int32_t* out_col,
                       double* out_vals, sc_stream_t stream);
/* SELL-32-sigma operator for repeated y = A x (the eigensolver's matvec
 * format): rows sorted by length inside 256-row windows, 32-row slices stored
 * column-major, rows longer than 2x the mean kept in CSR and summed by a
 * warp-per-row kernel.  A's CSR arrays must outlive the handle.  The operator
 * may have fewer rows than columns (a row shard with global columns). */
typedef struct sc_sell sc_sell_t;
int sc_sell_create(int64_t n_rows, const int64_t* row_ptr, const int32_t* col, const double* vals,
                   sc_stream_t stream, sc_sell_t** out);
int sc_sell_spmv(const sc_sell_t* op, const double* x, double* y, sc_stream_t stream);
int sc_sell_info(const sc_sell_t* op, int64_t* stored, int64_t* n_long_rows);
void sc_sell_destroy(sc_sell_t* op);
/* SpMV plan for repeated y = A x (the eigensolver's matvec; replaces
 * eigen.py:269-276 `_fast_apply` / sparse.py:195-207 `spmv` inside the
 * solve): built once (nnz read once, chunk table), applied without host
 * syncs.  Default kernel: one contiguous row range per SM, 16 lanes per row
 * (best measured on the C2 operator); SPECLUST_SPMV_KERNEL=bulk selects the
 * cp.async.bulk-staged chunk pipeline (one persistent CTA per SM streams
 * ~2048-nonzero chunks of whole rows through a shared-memory ring).  A's CSR
 * arrays must outlive the handle; n_rows may be a row shard (columns global). */
typedef struct sc_spmv_plan sc_spmv_plan_t;
int sc_spmv_plan_create(int64_t n_rows, const int64_t* row_ptr, const int32_t* col, const double* vals,
                        sc_stream_t stream, sc_spmv_plan_t** out);
int sc_spmv_plan_apply(const sc_spmv_plan_t* plan, const double* x, double* y, sc_stream_t stream);
void sc_spmv_plan_destroy(sc_spmv_plan_t* plan);
/* pos[perm[p]] = p */
int sc_invert_perm(int64_t n, const int32_t* perm, int32_t* pos, sc_stream_t stream);
/* dst row r = src row idx[r] (row-major n x k f64) */
int sc_gather_rows_f64(int64_t n, int64_t k, const double* src, const int32_t* idx, double* dst,
                       sc_stream_t stream);
/* *result (host) = 1 iff A == A^T bit-for-bit (sparse.py:210-222). */
int sc_csr_is_symmetric(int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col,
                        const double* vals, int* result, sc_stream_t stream);
/* CSR invariants of a device container (sparse.py:83-142, CsrMatrix checks):
 * row_ptr from 0 to nnz and non-decreasing, columns in range and strictly
 * increasing per row, finite values.  SC_ERR_FORMAT names the violation. */
int sc_csr_validate(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* row_ptr, const int32_t* col,
                    const double* vals, sc_stream_t stream);

/* ---- stage 1: kNN + exp_decay similarity graph straight into CSR ---------- */
/* x: (dev) n x d row-major f64.  Outputs (dev): row_ptr[n+1], col/vals with
 * capacity 2*n*knn; *nnz_out (host) receives the true nnz.  Semantics:
 * graph.py:149-157 ranking (similarity desc, index asc), union symmetrisation
 * (graph.py:203-204), one exp(-d2/(2 sigma^2)) per unordered pair
 * (graph.py:136-141).  stats_out (host, optional, 8 int64): candidates per row
 * budget, rows that needed the exact fallback, max row degree, ...         */
int sc_knn_graph_f64(int64_t n, int64_t d, const double* x, int64_t knn, double two_sigma_sq,
                     int64_t* row_ptr, int32_t* col, double* vals, int64_t* nnz_out,
                     int64_t* stats_out, sc_stream_t stream);
/* The same graph in two stages, for a build sharded over query rows
 * (SURVEY.md §8(e)); sc_knn_graph_f64 == select(0, n) + union(0, n).
 * select: the top-knn of the points at scan positions [p0, p1) (p0 a multiple
 *   of 128) into sel ((p1-p0) x knn int32, each row ascending) and the scan
 *   order perm (n int32: position -> point; identical for the same x on
 *   every caller).  Concatenating every shard's sel gives the n x knn
 *   selection in scan order.
 * union: CSR rows [r0, r1) (row_ptr local, r1-r0+1 entries; global columns)
 *   from the full selection; SC_ERR_VALUE with *nnz_out = the required size
 *   when it exceeds cap. */
int sc_knn_select_f64(int64_t n, int64_t d, const double* x, int64_t knn, double two_sigma_sq,
                      int64_t p0, int64_t p1, int32_t* sel, int32_t* perm, int64_t* stats_out,
                      sc_stream_t stream);
int sc_knn_union_f64(int64_t n, int64_t d, const double* x, int64_t knn, double two_sigma_sq,
                     const int32_t* sel, const int32_t* perm, int64_t r0, int64_t r1,
                     int64_t* row_ptr, int32_t* col, double* vals, int64_t cap, int64_t* nnz_out,
                     sc_stream_t stream);
/* The same two stages carrying the exact value of every selection slot
 * (sel_vals, (p1-p0) x knn fp64, in sel's order: the einsum-order d2 of the
 * pair): the union then fills the CSR values without recomputing a distance
 * (a reverse entry takes the value of the other endpoint's slot, the same
 * number).  Results are bit-identical to the plain forms. */
int sc_knn_select_vals_f64(int64_t n, int64_t d, const double* x, int64_t knn, double two_sigma_sq,
                           int64_t p0, int64_t p1, int32_t* sel, double* sel_vals, int32_t* perm,
                           int64_t* stats_out, sc_stream_t stream);
int sc_knn_union_vals_f64(int64_t n, int64_t d, const double* x, int64_t knn, double two_sigma_sq,
                          const int32_t* sel, const double* sel_vals, const int32_t* perm, int64_t r0,
                          int64_t r1, int64_t* row_ptr, int32_t* col, double* vals, int64_t cap,
                          int64_t* nnz_out, sc_stream_t stream);
/* out[p] = exp(-|x_a - x_b|^2 / two_sigma_sq) for pairs (a, b) = pairs[2p..2p+1]
 * (graph.py:136-141, used by build_similarity on a given edge list). */
int sc_pair_weights(int64_t n, int64_t d, const double* x, int64_t m, const int64_t* pairs,
                    double two_sigma_sq, double* out, sc_stream_t stream);

/* ---- stage 2: thick-restart Lanczos ----------------------------------------- */
typedef struct {
    int64_t restarts;        /* RciSession.restart_count  */
    int64_t breakdowns;      /* RciSession.breakdown_count */
    int64_t matvecs;         /* operator applications       */
    int64_t n_history;       /* valid entries in history    */
    double history[512];     /* residual_history (first 512 sweeps) */
    int64_t second_passes;   /* steps that needed a second CGS pass */
    int64_t flushes;         /* block reorthogonalisations of the window */
    double max_loss;         /* largest |B_old^T V| found by a flush */
    double mean_window;      /* average window length between flushes */
} sc_lanczos_stats;

/* RCI session (eigen.py:86-266).  m <= 0 selects default_subspace_dim. */
int sc_lanczos_create(int64_t n, int64_t k, int64_t m, double tol, int64_t max_restarts,
                      uint64_t seed, sc_stream_t stream, sc_lanczos_t** out);
void sc_lanczos_destroy(sc_lanczos_t* s);
/* state: 0 need_matvec, 1 converged, 2 failed */
int sc_lanczos_state(const sc_lanczos_t* s);
/* (dev) pointer to the current in_slot vector (length n, read-only for callers) */
const double* sc_lanczos_in_slot(const sc_lanczos_t* s);
/* (dev) pointer to the out_slot buffer the caller fills with A * in_slot */
double* sc_lanczos_out_slot(sc_lanczos_t* s);
/* one Lanczos step consuming out_slot; returns SC_ERR_MAX_RESTARTS /
 * SC_ERR_BREAKDOWN on failure (session then in state 2). */
int sc_lanczos_advance(sc_lanczos_t* s);
int sc_lanczos_get_stats(const sc_lanczos_t* s, sc_lanczos_stats* st);
/* values (host, k) and residual estimates (host, k) of the last sweep; valid
 * after convergence or after SC_ERR_MAX_RESTARTS. */
int sc_lanczos_ritz(const sc_lanczos_t* s, double* values, double* estimates);
/* converged pairs: values (host, k) descending, vectors (dev) n x k row-major */
int sc_lanczos_extract(sc_lanczos_t* s, double* values, double* vectors);

/* Device-resident eigensolve of a symmetric CSR: symmetry probe excluded;
 * vectors (dev) n x k row-major; values/residuals host arrays of length k. */
int sc_eigensolve_csr(int64_t n, const int64_t* row_ptr, const int32_t* col,
                      const double* vals, int64_t k, int64_t m, double tol,
                      int64_t max_restarts, uint64_t seed, double* values, double* vectors,
                      double* residuals, sc_lanczos_stats* stats, sc_stream_t stream);
/* sc_eigensolve_csr with a caller-owned Krylov basis: `basis` holds
 * (m + 1) * sc_lanczos_basis_ld(n) doubles (column-major, leading dimension
 * ld = n rounded up to 32) and on return its columns 0..k-1 are the unit
 * eigenvectors (eigen.py:291-302).  For operators whose basis and a separate
 * n x k result do not fit the device together (C4: 16M x 1001 basis); the
 * embedding is then built from the basis columns (sc_recover_embedding_cm)
 * into its unused columns. */
int sc_eigensolve_csr_basis(int64_t n, const int64_t* row_ptr, const int32_t* col,
                            const double* vals, int64_t k, int64_t m, double tol,
                            int64_t max_restarts, uint64_t seed, double* values, double* basis,
                            double* residuals, sc_lanczos_stats* stats, sc_stream_t stream);
int64_t sc_lanczos_basis_ld(int64_t n);
/* sc_eigensolve_csr for A = D^-1/2 W D^-1/2 with the degrees d (device, n)
 * it was scaled with (laplacian.py:84-91).  Eigenvalue 1 of A has one
 * eigenvector per connected component, u_C = D^1/2 1_C / |D^1/2 1_C|; when
 * there are 2 <= c < k components (and n >= 32768) those c pairs are locked
 * up front and the Lanczos recurrence runs on their orthogonal complement for
 * the other k - c (the reference finds the copies one verification sweep at
 * a time, eigen.py:195-206).  *locked_out = c (0: the plain solve ran).
 * Output as sc_eigensolve_csr: values descending, vectors row-major n x k. */
int sc_eigensolve_csr_deflate(int64_t n, const int64_t* row_ptr, const int32_t* col,
                              const double* vals, const double* d, int64_t k, int64_t m, double tol,
                              int64_t max_restarts, uint64_t seed, double* values, double* vectors,
                              double* residuals, sc_lanczos_stats* stats, int64_t* locked_out,
                              sc_stream_t stream);
/* max over the three probes of eigen.py:279-288 of |x'Ay - y'Ax| / (|x| |y|)
 * divided by max(1, max|a|) (host *ratio_out); probes are device Philox normals.
 * The caller raises NotSymmetric when ratio > 1e-10. */
int sc_symmetry_probe(int64_t n, const int64_t* row_ptr, const int32_t* col,
                      const double* vals, uint64_t seed, double* ratio_out,
                      sc_stream_t stream);

/* ---- embedding ------------------------------------------------------------- */
/* v = u / sqrt(d) rowwise, columns to unit norm, optionally rows to unit norm.
 * u, out: (dev) n x k row-major (may alias). */
int sc_recover_embedding(int64_t n, int64_t k, const double* u, const double* d,
                         int normalize_rows, double* out, sc_stream_t stream);
/* sc_recover_embedding from column-major eigenvectors (element (r, c) at
 * u[c * ld + r]); out row-major n x k, not overlapping u; same values. */
int sc_recover_embedding_cm(int64_t n, int64_t k, const double* u, int64_t ld, const double* d,
                            int normalize_rows, double* out, sc_stream_t stream);
int sc_normalize_rows(int64_t n, int64_t k, const double* v, double* out, sc_stream_t stream);

/* ---- stage 3: k-means --------------------------------------------------------- */
int sc_pairwise_sq_dist(int64_t n, int64_t k, int64_t d, const double* v, const double* c,
                        double* out, sc_stream_t stream);

typedef struct sc_kmeanspp sc_kmeanspp_t;
/* k-means++ (kmeans.py:107-136).  The host owns the numpy PCG64 stream:
 * begin(first) picks chosen[0] = first; then per step the host calls
 * sc_kmeanspp_candidates (host count of untaken rows with d2 > 0), draws
 * u = rng.random() (or rng.integers(free) when the count is 0) and calls
 * sc_kmeanspp_pick. */
int sc_kmeanspp_create(int64_t n, int64_t d, const double* v, sc_stream_t stream,
                       sc_kmeanspp_t** out);
void sc_kmeanspp_destroy(sc_kmeanspp_t* s);
int sc_kmeanspp_take(sc_kmeanspp_t* s, int64_t index);
int sc_kmeanspp_candidates(sc_kmeanspp_t* s, int64_t* count, int64_t* n_free);
/* mode 0: weighted draw with uniform u in [0,1); mode 1: the r-th untaken row */
int sc_kmeanspp_pick(sc_kmeanspp_t* s, int mode, double u, int64_t r, int64_t* index);

/* Lloyd iterations (kmeans.py:159-196).  v (dev) n x d row-major, c_init (dev)
 * k x d; outputs labels (dev int64 n), centroids (dev k x d), sse_history
 * (host, capacity max_iters+1), *iters_out (host). */
int sc_lloyd(int64_t n, int64_t d, int64_t k, const double* v, const double* c_init,
             int64_t max_iters, int64_t tol_changes, int64_t* labels, double* centroids,
             double* sse_history, int64_t* iters_out, sc_stream_t stream);

/* ---- per-shard building blocks (row-sharded Lanczos, point-sharded k-means;
 *      driven by paper_1802_04450_b200/distributed.py over NCCL) -------------- */
/* h = B^T w for the first ncols columns of a column-major shard (ld rows) */
int sc_gemv_t_f64(int64_t n, int64_t ld, int64_t ncols, const double* B, const double* w, double* h,
                  sc_stream_t stream);
/* w -= B h; *sq_out (dev, optional) = |w|^2 of the updated shard */
int sc_gemv_n_f64(int64_t n, int64_t ld, int64_t ncols, const double* B, const double* h, double* w,
                  double* sq_out, sc_stream_t stream);
/* dst = src / div */
int sc_div_copy_f64(int64_t n, const double* src, double div, double* dst, sc_stream_t stream);
/* out[i] = normal draw of global element offset + i (shard-independent) */
int sc_fill_normal(int64_t n, int64_t offset, uint64_t seed, uint64_t stream_id, double* out,
                   sc_stream_t stream);
/* eigen-decomposition of the m x m projected matrix (eigen.py:189-192):
 * theta (dev, m) stable descending, S (dev, m x kout column-major) */
int sc_symeig_f64(int64_t m, int64_t kout, const double* T, double* theta, double* S, sc_stream_t stream);
/* the same for the structured projected matrix of the thick restart
 * (eigen.py:189-192, 226-235): rows 0..p-1 diag(theta) coupled only to row p,
 * rows p..m-1 tridiagonal (p = 0 before the first restart).  Arrowhead
 * divide and conquer; theta (dev, m) descending, S (dev, m x kout). */
int sc_symeig_arrow_f64(int64_t m, int64_t p, int64_t kout, const double* T, double* theta, double* S,
                        sc_stream_t stream);
/* block Gram-Schmidt against basis columns as DMMA GEMMs (B, V column-major,
 * leading dimension ld, 1 <= c <= 40):  H (nb x c row-major) = B[:, :nb]^T V */
int sc_block_tn_f64(int64_t n, int64_t ld, int64_t nb, const double* B, const double* V, int64_t c,
                    double* H, sc_stream_t stream);
/* V -= B[:, :nb] H */
int sc_block_nn_f64(int64_t n, int64_t ld, int64_t nb, const double* B, const double* H, int64_t c,
                    double* V, sc_stream_t stream);
/* C = A (n x kk, col-major lda) * S (kk x kc, col-major lds); C col-major ldc or row-major */
int sc_dgemm_tall(int64_t n, int64_t kk, int64_t kc, const double* A, int64_t lda, const double* S,
                  int64_t lds, double* C, int64_t ldc, int rowmajor, sc_stream_t stream);
/* local assignment: labels/cost, *changes vs old_labels (null -> 0), *sse (host) */
int sc_kmeans_assign(int64_t n, int64_t d, int64_t k, const double* v, const double* c,
                     const int64_t* old_labels, int64_t* labels, double* cost, int64_t* changes,
                     double* sse, sc_stream_t stream);
/* unnormalised per-cluster sums (point order) and counts of the local points */
int sc_kmeans_local_sums(int64_t n, int64_t d, int64_t k, const double* v, const int64_t* labels,
                         double* sums, int64_t* counts, sc_stream_t stream);
int sc_centroid_divide(int64_t k, int64_t d, const double* sums, const int64_t* counts, double* cent,
                       sc_stream_t stream);
/* first e indices (host) of the stable descending order of cost (kmeans.py:151) */
int sc_farthest(int64_t n, const double* cost, int64_t e, int64_t* idx_out, sc_stream_t stream);
/* shard-aware k-means++: draw given by coordinates (row dev, d) and the local
 * index (-1 when the row is on another shard) */
int sc_kmeanspp_take_row(sc_kmeanspp_t* s, const double* row, int64_t local_index);
int sc_kmeanspp_weight(sc_kmeanspp_t* s, double* wsum, int64_t* count, int64_t* n_free);
int sc_kmeanspp_psum(sc_kmeanspp_t* s, double total_global, double* psum);
int sc_kmeanspp_search(sc_kmeanspp_t* s, double target, int64_t* index);
int sc_kmeanspp_nth_free(sc_kmeanspp_t* s, int64_t r, int64_t* index);
/* sym_scale on rows row_offset .. row_offset+n_local-1 (global degree vector) */
int sc_sym_scale_shard_f64(int64_t n_local, int64_t row_offset, const int64_t* row_ptr, const int32_t* col,
                           const double* vals, const double* d_global, double* out, sc_stream_t stream);
/* two-phase embedding of a row shard: scale + column sums of squares (dev k),
 * then finish with the all-reduced column sums */
int sc_embed_scale(int64_t n, int64_t k, const double* u, const double* d, double* out, double* colsq,
                   sc_stream_t stream);
int sc_embed_finish(int64_t n, int64_t k, const double* colsq, int normalize_rows, double* out,
                    sc_stream_t stream);
/* per-part boundary weight, volume and member count of a row shard (dev k each) */
int sc_ncut_partials(int64_t n_local, int64_t row_offset, const int64_t* row_ptr, const int32_t* col,
                     const double* vals, const int64_t* labels_global, int64_t k, double* bnd, double* vol,
                     int64_t* counts, sc_stream_t stream);

/* ---- metrics ---------------------------------------------------------------- */
/* ncut over labels (dev int64) in [0, k) (metrics.py:59-67); *out host.
 * skip_empty=1 drops parts without members first (the pipeline's np.unique
 * compaction, pipeline.py:256-257) and *occupied (host, optional) receives
 * the number of occupied parts.  Returns SC_ERR_VALUE with *out = -1 when a
 * remaining part has zero volume. */
int sc_ncut(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* vals,
            const int64_t* labels, int64_t k, int skip_empty, double* out, int64_t* occupied,
            sc_stream_t stream);
/* cut and ratio_cut (metrics.py:42-56: cut(w, labels), ratio_cut(w, labels)):
 * *cut_out = 1/2 of the crossing weight, *ratio_out = 1/2 sum_c bnd_c/|c|;
 * *empty_part (host) = first empty part (ratio_cut raises EmptyPart) or -1. */
int sc_partition_cuts(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* vals,
                      const int64_t* labels, int64_t k, double* cut_out, double* ratio_out, int64_t* empty_part,
                      sc_stream_t stream);
/* handle_isolated(w, d, "remove") (laplacian.py:34-64): induced submatrix on
 * the nodes with d != 0.  remap (dev, n): new index or -1; outputs are
 * caller-allocated with the input sizes (row_ptr n+1, col/vals nnz, d n);
 * *n_new / *nnz_new (host) receive the reduced sizes. */
int sc_csr_remove_isolated(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* vals,
                           const double* d, int64_t* remap, int64_t* out_row_ptr, int32_t* out_col,
                           double* out_vals, double* out_d, int64_t* n_new, int64_t* nnz_new, sc_stream_t stream);
/* cosine / cross-correlation similarity of each (i, j) pair of `pairs`
 * (m x 2 int64, dev) (graph.py:136-147 + the negative policy, graph.py:229-
 * 236): kind 1 cosine, 2 cross_correlation; negative_policy 0 clamp_zero,
 * 1 abs, 2 keep.  A zero-norm (cosine) / constant (cross_correlation)
 * endpoint returns SC_ERR_VALUE with *degenerate (host) = its index
 * (DegenerateVector). */
int sc_edge_similarity_f64(int64_t n, int64_t d, const double* x, int64_t m, const int64_t* pairs, int kind,
                           int negative_policy, double* out, int64_t* degenerate, sc_stream_t stream);
/* union-kNN similarity graph for any measure (graph.py:149-163, 185-237):
 * kind 0 exp_decay (sigma), 1 cosine, 2 cross_correlation; negative_policy
 * 0 clamp_zero, 1 abs, 2 keep.  Outputs as sc_knn_graph_f64 (capacity
 * 2 n knn).  A degenerate point returns SC_ERR_VALUE with *degenerate (host)
 * = its index (DegenerateVector). */
int sc_knn_graph_measure_f64(int64_t n, int64_t d, const double* x, int64_t knn, int kind, double sigma,
                             int negative_policy, int64_t* row_ptr, int32_t* col, double* vals, int64_t* nnz_out,
                             int64_t* stats_out, int64_t* degenerate, sc_stream_t stream);
/* Planted-partition SBM straight into CSR (sbm.py:68-108):
 * offsets (dev int64, nblocks+1) = block boundaries; p_in / p_out edge
 * probabilities; deterministic per seed (Philox, geometric skipping per row).
 * Call with col == NULL for *nnz_out (host), then with caller-allocated
 * row_ptr (n+1) / col / vals (nnz) (dev): symmetric, unit weights, no
 * self-loops, columns ascending. */
int sc_sbm_csr(int64_t n, const int64_t* offsets, int64_t nblocks, double p_in, double p_out, uint64_t seed,
               int64_t* row_ptr, int32_t* col, double* vals, int64_t* nnz_out, sc_stream_t stream);
/* eps / threshold patterns (graph.py:160-176, 206-211): (i < j) pairs in
 * row-major order.  mode 0 eps (a = eps), 1 threshold exp_decay (a = lambda,
 * b = sigma), 2 threshold cosine, 3 threshold cross_correlation (a = lambda).
 * Call with pairs == NULL for the count (*m_out, host), then with a
 * caller-allocated m x 2 int64 (dev) buffer. */
int sc_pattern_edges_f64(int64_t n, int64_t d, const double* x, int mode, double a, double b, int64_t* pairs,
                         int64_t* m_out, int64_t* degenerate, sc_stream_t stream);
/* row_scale(w, d) (laplacian.py:75-81): out = vals / d[row], IEEE division. */
int sc_row_scale_f64(int64_t n, const int64_t* row_ptr, const double* vals, const double* d, double* out,
                     sc_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SPECLUST_B200_H */
