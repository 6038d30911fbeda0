/* as.h — C ABI of libalphasparse: the data-parallel hot path of AlphaSparse
 * (arXiv 2212.10432) re-designed for NVIDIA B200 (sm_100a).
 *
 * The paper's statement of the problem: a sparse matrix comes in as Matrix Market / COO
 * ("takes a sparse matrix stored in the Matrix Market file format as input", PAPER.md
 * P:2; "AlphaSparse chooses the COO format as the universal source format"); an
 * Operator Graph ("connecting operators in order", §IV-B) is executed on the
 * Matrix Metadata Set (§V-A) into a format plus the SpMV kernel that reads it
 * (§V-B, §V-C); the Search Engine runs candidate graphs on the device and
 * keeps the fastest (§VI-A).  The operation is y = alpha*A*x + beta*y ("y=Ax";
 * alpha/beta per BASELINE.json north_star, reading A1 in DESIGN.md).
 *
 * Conventions for every entry point
 *   - returns as_status_t, never throws across the ABI; as_last_error() gives a message
 *     (thread-local) for the last non-OK status;
 *   - on a precondition failure nothing is launched and no output is written;
 *   - device pointers are CUDA device memory of the plan's device; "stream" is a
 *     cudaStream_t passed as void* (NULL = legacy default stream);
 *   - index arrays in the API are int64, values are the plan dtype (AS_R32F = float,
 *     AS_R64F = double); the device format uses int32 indices (all counts < 2^31,
 *     checked: AS_ERR_PLAN_INFEASIBLE otherwise).
 */
#ifndef ALPHASPARSE_AS_H
#define ALPHASPARSE_AS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  AS_OK = 0,
  AS_ERR_INVALID_ARG = 1,      /* NULL / size / alignment / aliasing / dtype precondition */
  AS_ERR_MALFORMED = 2,        /* Matrix Market header or entry line malformed */
  AS_ERR_INDEX_OUT_OF_RANGE = 3,
  AS_ERR_DUPLICATE = 4,        /* duplicate (row, col) triplet: reading A4, not summed */
  AS_ERR_GRAPH_PARSE = 5,      /* graph text does not follow the DSL grammar */
  AS_ERR_GRAPH_ILLEGAL = 6,    /* operator dependency rule R1..R11 violated (reading A16) */
  AS_ERR_PLAN_INFEASIBLE = 7,  /* matrix-dependent check failed (P1..P4, cut ranges, no kernel) */
  AS_ERR_OOM = 8,
  AS_ERR_CUDA = 9,
  AS_ERR_NO_FEASIBLE = 10,     /* as_search: no candidate could be planned */
  AS_ERR_DTYPE = 11,
  AS_ERR_NOT_FOUND = 12,       /* as_plan_export: key not present in this plan */
  AS_ERR_NCCL = 13             /* NCCL missing or an NCCL call failed (as_dist_*) */
} as_status_t;

typedef enum { AS_R32F = 0, AS_R64F = 1 } as_dtype_t;

typedef struct as_matrix_s* as_matrix_t;
typedef struct as_graph_s* as_graph_t;
typedef struct as_plan_s* as_plan_t;

/* Row statistics (§VII-C average row length nnz/n and row variance
 * sum((len - nnz/n)^2)/n, population; "irregular" <=> variance > 100). */
typedef struct {
  int64_t m, n, nnz, max_row_len, min_row_len, empty_rows;
  double avg_row_len, row_len_variance;
  int irregular;
} as_stats_t;

/* Plan summary.  bytes_model = algorithmic HBM bytes of one as_spmv call under the plan's
 * own traffic model (arrays read + x + y + extra passes) for beta == 0; bytes_model_beta
 * for beta != 0; bytes_floor = nnz*(sv+4) + n*sv + m*sv (DESIGN.md §Bytes model). */
typedef struct {
  int64_t nnz_real, stored_slots, pads, n_parts, n_launches, prepass_rows;
  double bytes_model, bytes_model_beta, bytes_floor;
  char kernels[512]; /* ';'-separated kernel names in launch order */
  int single_writer;  /* every row's final value comes from exactly one STORE: as_spmv_dist
                         with AS_EXCH_PEER fuses the peer stores into the SpMV epilogue */
  int modeled_arrays; /* index arrays replaced by fitted models (Model-Driven Format
                         Compression): computed in the kernel instead of loaded */
  int device_built;   /* 1: the format was built by the on-device Designer (see as_plan) */
} as_plan_info_t;

const char* as_last_error(void);
const char* as_version(void);

/* ---------------------------------------------------------------- a1: matrix (host)
 * as_matrix_create: copies the triplets (caller may free on return).  row/col are
 * index_base-based (0 or 1), any order; duplicates -> AS_ERR_DUPLICATE; out-of-range ->
 * AS_ERR_INDEX_OUT_OF_RANGE.  Empty rows are accepted (reading A6).  val has dtype dt.
 * m, n < 2^31. */
as_status_t as_matrix_create(int64_t m, int64_t n, int64_t nnz, const int64_t* row,
                             const int64_t* col, const void* val, as_dtype_t dt,
                             int index_base, as_matrix_t* out);
/* CSR ingest for very large inputs (0-based row_ptr[m+1] int64, col[nnz] int32, val[nnz]);
 * columns must be strictly ascending within each row (checked). */
as_status_t as_matrix_create_csr(int64_t m, int64_t n, const int64_t* row_ptr,
                                 const int32_t* col, const void* val, as_dtype_t dt,
                                 as_matrix_t* out);
/* Matrix Market 'matrix coordinate' real|integer|pattern, general|symmetric (reading A3). */
as_status_t as_matrix_create_mtx(const char* path, as_dtype_t dt, as_matrix_t* out);
as_status_t as_matrix_stats(as_matrix_t, as_stats_t* out);
/* ROW_DIV band [r0, r1) as a new matrix with r1-r0 rows and the same n (global columns). */
as_status_t as_matrix_row_slice(as_matrix_t, int64_t r0, int64_t r1, as_matrix_t* out);
/* Host CSR view of the canonical matrix: row_ptr[m+1] int64, col[nnz] int64, val dtype. */
as_status_t as_matrix_export_csr(as_matrix_t, int64_t* row_ptr, int64_t* col, void* val);
void as_matrix_destroy(as_matrix_t);

/* ---------------------------------------------------------------- graph
 * Grammar (DESIGN.md §Graph DSL):
 *   seq := op (';' op)* ;  op := NAME ['(' [arg (',' arg)*] ')'] ['{' seq ('|' seq)* '}']
 * Validates the operator dependencies (no BMTB after BMW/BMT; full list
 * R1..R11 = reading A16).  AS_ERR_GRAPH_PARSE | AS_ERR_GRAPH_ILLEGAL (message names the
 * pre-order node id and the rule). */
as_status_t as_graph_parse(const char* text, as_graph_t* out);
/* Canonical one-line form; buf == NULL or *len too small -> *len = required bytes
 * (incl. NUL) and AS_ERR_INVALID_ARG when buf != NULL. */
as_status_t as_graph_print(as_graph_t, char* buf, size_t* len);
void as_graph_destroy(as_graph_t);

/* ---------------------------------------------------------------- a2-a4: plan
 * Executes the graph on the Matrix Metadata Set (converting -> COMPRESS -> mapping ->
 * implementing) and uploads the resulting device format to `device`
 * (device = -1: host-only plan, usable for as_plan_export but not for as_spmv).
 * Blocking.  The plan owns its device arrays and keeps no reference to the matrix.
 * flags: AS_PLAN_KEEP_HOST keeps the logical metadata on the host for as_plan_export.
 * On-device Designer: graphs of the NNZ-blocked family
 *   [SORT|SORT_SUB]; COMPRESS; [BMW_NNZ_BLOCK]; BMT_NNZ_BLOCK; [BMT_PAD(GLOBAL|BMW)];
 *   THREAD_BITMAP_RED_G; [WARP_SEG_ADD_RED|WARP_BITMAP_RED]; [SET_RESOURCE]; GMEM_ATOM_RED
 * are built on the GPU (CUB sorts/scans + kernels) unless AS_PLAN_KEEP_HOST, AS_PLAN_SPMM or
 * AS_PLAN_HOST_BUILD is given; the first such plan uploads the matrix's canonical CSR to the
 * device once and the matrix keeps that copy (freed by as_matrix_destroy) for later plans. */
#define AS_PLAN_KEEP_HOST 1
#define AS_PLAN_SPMM 2      /* also upload the plain CSR arrays of CSR-family parts (as_spmm) */
#define AS_PLAN_GRAPH 4     /* as_spmv captures its launch sequence into a CUDA graph once per
                               (x, y, alpha, beta) and replays it: one launch per call.  The
                               plan then caches one graph: calls on the same plan must not run
                               concurrently from several host threads */
#define AS_PLAN_HOST_BUILD 8 /* always run the host Designer (A/B of the on-device one) */
as_status_t as_plan(as_matrix_t, as_graph_t, int device, void* stream, as_plan_t* out);
as_status_t as_plan_ex(as_matrix_t, as_graph_t, int device, void* stream, int flags,
                       as_plan_t* out);
as_status_t as_plan_info(as_plan_t, as_plan_info_t* out);
/* *out = 1 if as_plan_ex(M, G, device >= 0, flags) would build the format with the
 * on-device Designer (the NNZ-blocked family above), else 0.  Host-only query. */
as_status_t as_graph_device_buildable(as_matrix_t, as_graph_t, int flags, int* out);
/* Logical metadata array `key` (DESIGN.md §Export keys, e.g. "p0.bmt.bitmap"), copied to
 * host_dst.  host_dst == NULL -> *bytes = size.  Needs a host-only plan or
 * AS_PLAN_KEEP_HOST.  Index arrays are int64, bitmaps uint32, values the plan dtype. */
as_status_t as_plan_export(as_plan_t, const char* key, void* host_dst, size_t* bytes);
/* ';'-separated list of export keys present in this plan. */
as_status_t as_plan_keys(as_plan_t, char* buf, size_t* len);
void as_plan_destroy(as_plan_t);

/* ---------------------------------------------------------------- a5-a6: SpMV
 * y = alpha*A*x + beta*y.  x[n], y[m] device pointers of the plan's dtype and device,
 * aligned to the value size, non-aliasing (a ROW_DIV band may write into a slice of a
 * larger y); alpha/beta point to HOST scalars of the plan's dtype.
 * beta == 0: y is write-only (NaN in y not propagated).  Asynchronous on `stream`;
 * device faults surface as AS_ERR_CUDA at a later call.  Parts whose SET_RESOURCE names
 * another stream than the first part's (DESIGN.md R-conc) run on plan-owned side streams
 * forked from `stream` after the beta pre-pass and joined back into it before the call's
 * last launch, so the call stays ordered on `stream` (also under CUDA-graph capture). */
as_status_t as_spmv(as_plan_t, const void* alpha, const void* x, const void* beta, void* y,
                    void* stream);
/* Same with HOST x[n] / y[m] (pinned for overlap; pageable works): copies x (and y when
 * beta != 0) to the plan's device scratch, runs as_spmv, copies y back; synchronous.
 * Plans with several launches (e.g. ROW_DIV bands) are pipelined: x goes up in
 * column chunks on a plan-owned copy stream, launch i waits only for the chunk holding the
 * last column it reads, and each y row range no later launch writes goes down on a second
 * copy stream once its last writer is done (PCIe is full duplex).  Not pipelined: a single
 * launch, fp32 plans with heavy rows, plans with concurrent branches (R-conc), or
 * AS_HOST_NOPIPE set in the environment.  The
 * result is identical either way (same kernels, same order on the device). */
as_status_t as_spmv_host(as_plan_t, const void* alpha, const void* x_host, const void* beta,
                         void* y_host, void* stream);
/* (as_spmv_host and as_spmv_host_batch use the plan's device scratch buffers and copy
 * streams: calls on the same plan must not run concurrently from several host threads.)
 * k independent SpMVs y_i = alpha*A*x_i + beta*y_i on host buffers (pinned for overlap),
 * pipelined across i: x_{i+1} is copied up while SpMV i runs and y_{i-1} is copied down
 * (two device buffer pairs, two copy streams; x buffer j is reused once SpMV i-2 read it,
 * y buffer j once y_{i-2} came down, so both directions run at once); every x_i goes up and
 * every y_i comes back.  Blocking; the steady state per SpMV is max(H2D x, kernels,
 * D2H y) with both copy directions sharing the link.  Same errors as
 * as_spmv_host. */
as_status_t as_spmv_host_batch(as_plan_t, int64_t k, const void* alpha, const void* const* x_host,
                               const void* beta, void* const* y_host, void* stream);

/* SpMM (NEXT-4): Y = alpha*A*X + beta*Y with k right-hand sides.  X[n x k] and Y[m x k]
 * are row-major device arrays of the plan's dtype with leading dimensions ldx, ldy >= k;
 * they must not overlap.  The plan must be built with AS_PLAN_SPMM.  Parts run in the SpMV's
 * writer-rule order (beta pre-pass, STORE / ADD per row): DENSE tiles as tensor-core
 * contractions (fp64 DMMA m8n8k4; fp32 tiles widened exactly), DIA parts per (row, column),
 * CSR-family parts by a row-parallel CSR SpMM over their COMPRESS arrays (rows summed in
 * fp64 by one thread group).  Asynchronous on `stream`.  Tolerance per element as the SpMV
 * (O2). */
as_status_t as_spmm(as_plan_t, int64_t k, const void* alpha, const void* X, int64_t ldx,
                    const void* beta, void* Y, int64_t ldy, void* stream);

/* Per-launch profile (measurement): runs as_spmv (alpha 1, beta 0) `reps`
 * times on `stream` with CUDA events between the launches and returns, per entry of
 * as_plan_info_t.kernels ([pre-pass], parts in launch order, [heavy-row epilogue]), the mean
 * device time in ms and the entry's algorithmic bytes under the plan's model (arrays read
 * + x of the part's distinct columns + its y traffic; beta == 0).  ms == NULL or bytes ==
 * NULL -> *n = number of entries.  Overwrites y.  Concurrent branches (R-conc) are
 * profiled serialised on `stream` (same result; per-launch times of each kernel alone). */
as_status_t as_plan_profile(as_plan_t, const void* x, void* y, int reps, void* stream,
                            double* ms, double* bytes, size_t* n);

/* ---------------------------------------------------------------- a7: search
 * Random dependency-respecting graphs ("operators ... randomly chosen and connected
 * behind"; P:369 step 1) over a coarse parameter grid (P:369 step 2), each planned and
 * timed on the device (median of `reps` CUDA-event-timed calls after `warmup`, L2 flushed
 * before each when flush_l2), keeping the fastest.  The seed graphs run first.  Stops at
 * max_candidates or budget_seconds.  Returns the best plan and its canonical graph
 * (size-query convention on best_graph/len).  log_path (optional): one JSON line per
 * candidate. */
typedef struct {
  uint64_t seed;
  int max_candidates;
  double budget_seconds;
  int warmup, reps, flush_l2;
  const char* const* seed_graphs;
  int n_seed_graphs;
  const char* log_path;
  /* Optional cost-model history from earlier searches (NEXT-3; the paper's model is trained
   * on other matrices): n_history timed candidates, each a graph text, the
   * AS_MATRIX_FEATURES features of its matrix (history_matrix[i*AS_MATRIX_FEATURES ...]) and
   * log(median ms / nnz).  The model stage then fits graph + matrix features on the history
   * and the candidates of this search together (target log time per nonzero). */
  const char* const* history_graphs;
  const double* history_matrix;
  const double* history_log_t_per_nnz;
  int n_history;
} as_search_cfg_t;
#define AS_MATRIX_FEATURES 8
/* The matrix features of the search's cost model: log2(1+m), log2(1+n), log2(1+nnz), average
 * row length, log2(1+row-length variance), log2(1+max row length), empty-row fraction, value
 * size in bytes.  out holds AS_MATRIX_FEATURES doubles. */
as_status_t as_matrix_features(as_matrix_t, double* out);
as_status_t as_search(as_matrix_t, const as_search_cfg_t*, int device, void* stream,
                      as_plan_t* best, char* best_graph, size_t* len);
/* Model-Driven Format Compression (§V-D): fit an index array a[n] (n >= 2) to
 * model(i) = b + k1*(i / w) + k2*(i % w) -- linear (w = 1), periodic linear (w = 2..256,
 * powers of two), step (k2 = 0, w = first run length) -- with at most `budget` (<= 8)
 * patches; fewest patches wins, linear before periodic before step on ties.
 * out[6 + 2*budget] = {kind (1 linear, 2 periodic, 3 step), b, k1, k2, w, n_patches,
 * (index, value) x n_patches}.  No model within the budget -> AS_ERR_NOT_FOUND.  as_plan
 * applies it to origin_rows and the NNZ-BMT first rows (as_plan_info_t.modeled_arrays;
 * AS_NO_MDC in the environment disables it). */
as_status_t as_fit_array_model(const int64_t* a, size_t n, int budget, int64_t* out);

/* The search's cost model (NEXT-3; the paper's learned performance model of P:369 step 3,
 * P:371-377).  as_graph_features: fixed-length feature vector of a graph -- per operator
 * the occurrence count over all branches (24: ROW_DIV ... SHMEM_OFFSET_RED, SET_RESOURCE),
 * per numeric parameter class the mean log2(1 + value) (17: BMT/BMW/BMTB block sizes,
 * tpb, grid, stages, xcache, stream, vec, DIA theta/max, DENSE b/theta, SORT_SUB g), then the number of
 * leaves.  out == NULL -> *n = length.  as_surrogate_fit_predict: fits the gradient-boosted
 * regression-tree ensemble the search uses (60 rounds, depth 3, shrinkage 0.2, squared
 * loss) on X[n x d] (row-major) -> y[n] and writes its predictions for Xq[nq x d] to
 * out[nq].  Deterministic; host only. */
as_status_t as_graph_features(as_graph_t, double* out, size_t* n);
as_status_t as_surrogate_fit_predict(const double* X, const double* y, size_t n, size_t d,
                                     const double* Xq, size_t nq, double* out);
/* One random legal graph text for this matrix (the search's generator), for tests. */
as_status_t as_random_graph(as_matrix_t, uint64_t seed, char* buf, size_t* len);

/* ---------------------------------------------------------------- device memory
 * Route every device allocation of the library (plan arrays, as_spmv_host / as_search
 * scratch, dist flags) through caller hooks, e.g. torch's caching allocator:
 * alloc(bytes, stream, ctx) returns device memory of the current device or NULL (->
 * AS_ERR_OOM); release(ptr, stream, ctx) frees it.  Both NULL restores cudaMalloc/cudaFree.
 * Process-wide; set it before creating plans (a plan frees through the hooks that were
 * active when it was created only if they are still installed: do not swap hooks while
 * plans are alive). */
as_status_t as_set_allocator(void* (*alloc)(size_t bytes, void* stream, void* ctx),
                             void (*release)(void* ptr, void* stream, void* ctx), void* ctx);

/* ---------------------------------------------------------------- e: multi-GPU helpers
 * nnz-balanced ROW_DIV cuts over `world` ranks (reading A35): cuts[world+1]. */
as_status_t as_dist_row_cuts(as_matrix_t, int world, int64_t* cuts);
/* The same cuts from a host row_ptr[m+1] alone (int64, non-decreasing, row_ptr[0] = 0):
 * ranks that generate or load only their own band (C5 at 10^9 nonzeros) agree on the cuts
 * without building the whole matrix.  AS_ERR_INVALID_ARG on NULL, m < 0, world < 1. */
as_status_t as_dist_row_cuts_ptr(const int64_t* row_ptr, int64_t m, int world, int64_t* cuts);
/* Column span [*lo, *hi] referenced by the matrix (a ROW_DIV band): the x rows a rank needs
 * from its peers when y becomes the next x (halo exchange).  An empty
 * matrix gives lo = 0, hi = -1. */
as_status_t as_matrix_col_span(as_matrix_t, int64_t* lo, int64_t* hi);

/* ---------------------------------------------------------------- e: multi-GPU SpMV
 * ROW_DIV across ranks ("divide the matrix in the row direction", P:46
 * ROW_DIV example): one process per GPU; rank r owns rows [cuts[r], cuts[r+1]) of y (the
 * nnz-balanced cuts of as_dist_row_cuts), holds a plan of its band
 * (as_matrix_row_slice(A, cuts[r], cuts[r+1]), global column indices) and the full x.
 * The SpMV itself needs no communication; the exchange makes the new y whole on every rank
 * (it is the next x of an iterative solver, north_star):
 *   AS_EXCH_NONE  only the band y_full[cuts[r]:cuts[r+1]] is written;
 *   AS_EXCH_NCCL  AllGatherV of the bands: one ncclBroadcast per rank inside an NCCL group
 *                 (needs a communicator: as_dist_init with an id);
 *   AS_EXCH_PEER  the band is pushed by one kernel straight into every peer's y_full over
 *                 peer memory (NVLink P2P stores through CUDA IPC mappings, no NCCL), then
 *                 each rank's stream waits for its peers' release flags (one epoch per
 *                 call).  y_full must be registered on every rank first
 *                 (as_dist_ipc_handle + as_dist_open_peers).  The wait times out after
 *                 AS_DIST_WAIT_TIMEOUT_NS and reports AS_ERR_CUDA at as_dist_check.
 *                 Fused form: when the band plan is single-writer (as_plan_info_t.
 *                 single_writer) and world <= 8, the SpMV kernels themselves store every
 *                 final y value into the peers' y_full (the exchange overlaps the SpMV tile
 *                 by tile) and the push kernel only publishes the flags; AS_DIST_NO_FUSE in
 *                 the environment forces the separate push.
 * Every rank must make the same sequence of as_spmv_dist calls.  x_full and y_full must
 * not alias (iterate with two buffers).  NCCL is loaded at run time (dlopen
 * libnccl.so.2), so the library itself has no link-time NCCL dependency. */
typedef struct as_dist_s* as_dist_t;
#define AS_DIST_ID_BYTES 128      /* ncclUniqueId */
#define AS_DIST_HANDLE_BYTES 256  /* one rank's IPC registration blob */
#define AS_DIST_MAX_WORLD 64
#define AS_DIST_WAIT_TIMEOUT_NS 20000000000ull
enum { AS_EXCH_NONE = 0, AS_EXCH_NCCL = 1, AS_EXCH_PEER = 2 };
/* ncclGetUniqueId into id[AS_DIST_ID_BYTES] (rank 0; the caller broadcasts the bytes). */
as_status_t as_dist_unique_id(void* id);
/* Communicator of `world` ranks on `device`.  id NULL: peer-memory mode only (no NCCL). */
as_status_t as_dist_init(int rank, int world, const void* id, int device, as_dist_t* out);
/* The world+1 row cuts of y (as_dist_row_cuts); required before as_spmv_dist. */
as_status_t as_dist_set_cuts(as_dist_t, const int64_t* cuts);
/* IPC registration of this rank's y buffer `y_full` (device memory from cudaMalloc or a
 * caching allocator built on it): writes handle[AS_DIST_HANDLE_BYTES] to be all-gathered
 * by the caller (any transport), in rank order, then passed to as_dist_open_peers. */
as_status_t as_dist_ipc_handle(as_dist_t, void* y_full, void* handle);
as_status_t as_dist_open_peers(as_dist_t, void* y_full, const void* handles /* world x HANDLE_BYTES */);
/* Halo windows (NEXT-1(ii), banded matrices): lo_hi[2q], lo_hi[2q+1] = first and last row of
 * y_full rank q reads (its band's column span, as_matrix_col_span; last < first = none).
 * Afterwards AS_EXCH_PEER sends each peer only the rows of this band inside its window
 * (fused or pushed), instead of the whole band; the flags are still released to every peer.
 * Every rank must install the same table.  lo_hi == NULL restores full bands. */
as_status_t as_dist_set_windows(as_dist_t, const int64_t* lo_hi /* world x 2 */);
as_status_t as_spmv_dist(as_dist_t, as_plan_t local, const void* alpha, const void* x_full,
                         const void* beta, void* y_full, int exchange, void* stream);
/* Device-side status of the peer exchange (AS_ERR_CUDA after a wait timeout); synchronizes
 * the dist's device. */
as_status_t as_dist_check(as_dist_t);
void as_dist_destroy(as_dist_t);

#ifdef __cplusplus
}
#endif
#endif /* ALPHASPARSE_AS_H */
