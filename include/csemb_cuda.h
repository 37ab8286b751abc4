/*
 * csemb_cuda.h -- C ABI of the B200-native fused SpMM-Legendre recurrence
 * (compressive spectral embedding, arXiv 1509.08360).
 *
 * Reference = the `csemb` Python package (/root/reference/pkg/src/csemb).
 * It has no formal plugin API; its single seam for this path is
 *   engine._apply_expansion(S, expansion, block, *, stage, n_workers, counter)
 *   (engine.py:231-258), plus sample_projection (engine.py:79-99),
 *   estimate_spectral_norm (engine.py:165-192) and scale_values (sparse.py:295-301).
 * Each entry point below names the reference function it replaces.
 *
 * Conventions
 *   - Every function returns an int status (CSEMB_OK = 0) and never throws;
 *     csemb_last_error() returns a thread-local message for the last failure.
 *   - Host pointers are borrowed for the duration of the call.
 *   - Device buffers are owned by the opaque handles.
 *   - Matrices are CSR with int64 row offsets / int64 column indices / f64
 *     values on the host side, exactly the reference's SparseMatrix arrays
 *     (sparse.py:55-99, design decision D6 64-bit indices).
 *   - Dense blocks are n_rows x d, row-major, float64 on the host side.
 *   - One context per device; calls on one context are serialised by a
 *     mutex; all work of a context runs on that context's CUDA stream.
 */
#ifndef CSEMB_CUDA_H
#define CSEMB_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CSEMB_ABI_VERSION 1

/* status codes */
#define CSEMB_OK 0
#define CSEMB_ERR_INVALID 1     /* bad argument: Python shim raises ValueError   */
#define CSEMB_ERR_CUDA 2        /* CUDA runtime failure                          */
#define CSEMB_ERR_NOMEM 3       /* device allocation failed                      */
#define CSEMB_ERR_DIVERGED 4    /* non-finite iterate: DivergenceError            */
#define CSEMB_ERR_UNSUPPORTED 5 /* valid request this build does not handle      */

/* arithmetic types */
#define CSEMB_F64 0
#define CSEMB_F32 1

/* projection-block sources */
#define CSEMB_OMEGA_GIVEN 0    /* caller supplies the block                      */
#define CSEMB_OMEGA_SPLITMIX 1 /* the reference's hash, bit-exact (engine.py:79) */
#define CSEMB_OMEGA_PHILOX 2   /* Philox4x32-10 signs (benchmark generator)      */

typedef struct csemb_ctx csemb_ctx;
typedef struct csemb_mat csemb_mat;
typedef struct csemb_plan csemb_plan;
typedef struct csemb_kmeans csemb_kmeans;

const char *csemb_last_error(void);
int csemb_abi_version(void);
int csemb_device_count(int *out);

/* ---- context ------------------------------------------------------------ */
int csemb_ctx_create(int device, csemb_ctx **out);
int csemb_ctx_destroy(csemb_ctx *ctx);
/* the context's cudaStream_t, for callers that time or order work on it */
void *csemb_ctx_stream(csemb_ctx *ctx);
int csemb_ctx_sync(csemb_ctx *ctx);
int csemb_ctx_sm_count(csemb_ctx *ctx, int *out);

/* ---- matrices -------------------------------------------------------------
 * csemb_matrix_upload replaces SparseMatrix._csr (sparse.py:160-165): the CSR
 * is validated for shape, copied once and kept device-resident (int64 row
 * offsets, int32 column indices, values in `dtype`).  */
int csemb_matrix_upload(csemb_ctx *ctx, int64_t n_rows, int64_t n_cols, int64_t nnz,
                        const int64_t *row_offsets, const int64_t *col_indices,
                        const double *values, int dtype, csemb_mat **out);
/* same, from device pointers (int64 offsets, int64 or int32 indices
 * per idx_bytes = 8|4, f64 values); used by device-side input builders */
int csemb_matrix_upload_device(csemb_ctx *ctx, int64_t n_rows, int64_t n_cols, int64_t nnz,
                               const void *row_offsets_dev, const void *col_indices_dev,
                               int idx_bytes, const double *values_dev, int dtype,
                               csemb_mat **out);
int csemb_matrix_destroy(csemb_mat *m);
int csemb_matrix_info(csemb_mat *m, int64_t *n_rows, int64_t *n_cols, int64_t *nnz, int *dtype);
/* scale_values (sparse.py:295-301): values *= factor on the device (same
 * IEEE product as numpy's S.values * factor). */
int csemb_matrix_scale(csemb_mat *m, double factor);
/* 1 if every stored value of m is bit-identical to normalized_adjacency's
 * 1/sqrt(deg(u) deg(v)) with deg = the stored row lengths (sparse.py:224):
 * K1 then recomputes values instead of streaming them (CSEMB_OPT_VALUE_FREE).
 * Runs the device check on first use; csemb_matrix_scale clears it. */
int csemb_matrix_value_free(csemb_mat *m, int *out);
/* copy the device values back (f64) -- for tests of csemb_matrix_scale */
int csemb_matrix_download_values(csemb_mat *m, double *values_out);
/* a copy of m in another arithmetic type (values converted; CSR shared shape) */
int csemb_matrix_convert(csemb_mat *m, int dtype, csemb_mat **out);
/* borrowed device pointers of m's arrays (int64 offsets, int32 column ids,
 * values in m's dtype); valid until csemb_matrix_destroy(m).  Read-only:
 * the library caches properties of the arrays (schedules, the value-free
 * check); change values only through csemb_matrix_scale */
int csemb_matrix_device_arrays(csemb_mat *m, void **row_offsets, void **col_indices, void **values);

/* ---- measurement probes (bench.py roofline objects; not the embedding path) ----
 * GB/s of one probe on the context's device, best of 3 timed launches:
 *   CSEMB_DIAG_L2_STREAM  coalesced 16-byte .cg re-reads of an L2-resident
 *                         `bytes` buffer, `reps` passes (L2 -> SM fabric)
 *   CSEMB_DIAG_L2_GATHER  K1's load shape: random rows of `row_bytes` inside
 *                         a `bytes` window, K1's lanes per row (16 for 640 B,
 *                         8 for 320 B), 4 rows in flight per lane group
 *   CSEMB_DIAG_HBM_COPY   read + write of a `bytes` buffer (DRAM copy)   */
#define CSEMB_DIAG_L2_STREAM 0
#define CSEMB_DIAG_L2_GATHER 1
#define CSEMB_DIAG_HBM_COPY 2
int csemb_diag_bandwidth(csemb_ctx *ctx, int kind, int64_t bytes, int64_t row_bytes, int reps, double *gbs);
/* Gather-only pass over m: every stored entry fetches one `row_bytes` row of
 * an n_cols-row block (K1's gathered bytes, in stored order, K1's lanes per
 * row), no arithmetic or streamed blocks, `in_flight` (4 | 8) entries in
 * flight per lane group.  Best of 3 timed launches: ms per pass and the
 * gathered GB/s (nnz * row_bytes / time).  The floor for K1 on m. */
int csemb_diag_gather_csr(csemb_mat *m, int64_t row_bytes, int in_flight, double *ms, double *gbs);

/* ---- device-side input construction --------------------
 * normalized_adjacency (sparse.py:202-226): edges is an n_edges x 2 int64
 * (u, v) array, host or device memory per edges_on_device.  Self-loops are
 * dropped, duplicate undirected edges merged, degrees counted, and every
 * stored value is 1/sqrt(deg u * deg v) computed with the reference's IEEE
 * operations; rows ascending, columns strictly increasing, isolated vertices
 * empty rows -- bit-identical to the host builder.  Values stored in dtype.
 * An endpoint outside [0, n) is CSEMB_ERR_INVALID (ValueError). */
int csemb_build_normalized_adjacency(csemb_ctx *ctx, int64_t n, int64_t n_edges, const int64_t *edges,
                                     int edges_on_device, int dtype, csemb_mat **out);
/* dilate (sparse.py:191-199): [0 A^T; A 0] of an m x n device matrix, square
 * (m+n); indices 0..n-1 are A's columns, n..n+m-1 its rows; same dtype. */
int csemb_build_dilation(csemb_mat *a, csemb_mat **out);

/* ---- plans: device workspace for one (matrix, d) ----------------------------
 * Holds Y (two n x ld buffers, Q(r-1) and Q(r-2)/Q(r) in place), E (n x ld)
 * and the per-step diagnostics.  ld = d rounded up to 16 bytes.  */
int csemb_plan_create(csemb_mat *m, int64_t d, csemb_plan **out);
int csemb_plan_destroy(csemb_plan *p);

/* Plan options.
 *  CSEMB_OPT_EXACT_PEAKS (default 0): 1 = record the exact per-chunk max|Q(r)|
 *    of every step (the reference's debug log, engine.py:217-220); 0 = record
 *    only non-finite flags (+inf key where a chunk diverged), which is all the
 *    DivergenceError check needs and keeps K1's register footprint small.
 *  CSEMB_OPT_REVERSE_SWEEP (default 1): alternate the row sweep direction each
 *    step so the rows written last (still in L2) are gathered first.
 *  CSEMB_OPT_SPLIT_THRESHOLD / CSEMB_OPT_ROW_ORDER: load balancing for skewed
 *    (power-law, dilation) row lengths; rows at or below the threshold keep the
 *    reference's stored-order accumulation (bit-exact).  */
#define CSEMB_OPT_EXACT_PEAKS 1
#define CSEMB_OPT_REVERSE_SWEEP 2
#define CSEMB_OPT_SPLIT_THRESHOLD 3 /* rows longer than this (default 2048) are split
                                       into chunks of <= 1024 entries summed in chunk
                                       order; on matrices with >= 8 column windows of
                                       3*2^16 (f32) / 2^16 (f64) columns the limit is
                                       min(this, max(64, 20 * windows)) and rows up to
                                       65536 entries are cut at the window boundaries
                                       (the cuts depend on the matrix and dtype only,
                                       never on the block width);
                                       0 = never split (bit-exact for every input) */
#define CSEMB_OPT_ROW_ORDER 4       /* -1 auto (default: 1 for skewed row lengths,
                                       else 2), 0 natural, 1 bucketed by batch count,
                                       2 bucketed within windows of consecutive rows
                                       (window chosen against the grid's wave), >= 64:
                                       that window.  Row order never changes results. */
#define CSEMB_OPT_GRAPH 6           /* -1 auto (default: blocks of <= 2^22 elements, where
                                       launches dominate), 0 off, 1 on: the second
                                       csemb_plan_run with an identical signature
                                       (coefficients, options, block pointer, seed, slice)
                                       is captured as a CUDA graph, later ones replay it */
#define CSEMB_OPT_VALUE_FREE 7      /* -1 default (off unless CSEMB_VALUE_FREE=1), 0 off, 1 on:
                                       when every stored value of the matrix is bit-identical to
                                       normalized_adjacency's 1/sqrt(deg(u) deg(v)) with deg = the
                                       stored row lengths (sparse.py:224; checked once on the
                                       device), K1 recomputes it from the row offsets instead of
                                       streaming the values (bit-identical results; whole rows
                                       only -- split heavy-row chunks and row partitions read
                                       the values).  Measured slower than streaming the values
                                       (a dependent gather + IEEE sqrt/div per entry), so off, and
                                       compiled out of the default build (K1_VF=0: setting 1 is
                                       CSEMB_ERR_UNSUPPORTED); the device check itself
                                       (csemb_matrix_value_free) is always available */
#define CSEMB_OPT_E_FOLD 5           /* 1..3 (default 3): E is read and written every
                                       e_fold steps; a flush adds the pending terms in
                                       the reference's order, so results are unchanged */
int csemb_plan_set_option(csemb_plan *p, int option, int64_t value);

/* Device-resident run: _apply_expansion (engine.py:231-258) chained over
 * n_stages cascade stages (engine.py:332-336).  coeffs[0..order] are the
 * stage's Legendre coefficients (LegendreExpansion.coeffs).  The projection
 * block is `block_dev` (device, n x d f64 row-major) when omega_kind ==
 * CSEMB_OMEGA_GIVEN, else generated on the device for global columns
 * [col0, col0+d) of an n x d_global block with `seed`.  normalize_rows != 0
 * appends the row normalisation (zero rows stay 0).  Asynchronous on the
 * context stream; results stay in the plan.  */
int csemb_plan_run(csemb_plan *p, const double *coeffs, int order, int n_stages,
                   const double *block_dev, int omega_kind, uint64_t seed, int64_t col0,
                   int64_t d_global, int normalize_rows);
/* Output access.  download converts to f64 (out_dtype CSEMB_F64) or f32. */
int csemb_plan_download(csemb_plan *p, void *out_host, int out_dtype);
int csemb_plan_output(csemb_plan *p, void **dev_ptr, int64_t *ld, int *dtype);
/* Device-to-device copy of E (n x d, plan dtype) into dst with row stride
 * dst_ld elements, on the context stream (for NCCL assembly of column shards). */
int csemb_plan_copy_output(csemb_plan *p, void *dst_dev, int64_t dst_ld);
/* Synchronises; max_abs (optional) receives n_stages*order*n_chunks values,
 * n_chunks = ceil(d_global/32): the reference's per-32-column-chunk max|Q(r)|
 * (engine.py:217-220).  first_bad_r / bad_stage follow the reference's
 * DivergenceError (engine.py:221-225): 0 when every iterate is finite.  */
int csemb_plan_diagnostics(csemb_plan *p, double *max_abs, int *first_bad_r, int *bad_stage);
/* CUDA-event timings of the last run: whole run and the recurrence steps */
int csemb_plan_timing(csemb_plan *p, float *ms_total, float *ms_steps, int *step_launches);

/* Host-to-host drop-in for _apply_expansion (engine.py:231-258): uploads
 * `block_host` (n x d f64; NULL when omega_kind generates it), runs, and
 * writes `out_host` (n x d f64).  Returns CSEMB_ERR_DIVERGED with
 * *first_bad_r / *bad_stage set if an iterate was non-finite.  */
int csemb_apply_expansion(csemb_plan *p, const double *coeffs, int order, int n_stages,
                          const double *block_host, int omega_kind, uint64_t seed,
                          int64_t col0, int64_t d_global, int normalize_rows,
                          double *out_host, double *max_abs, int *first_bad_r, int *bad_stage);

/* ---- row-partitioned runs (graphs larger than one GPU) ---------
 * The plan's matrix holds rows [row0, row0 + n_rows) of an n_global x n_global
 * operator (local CSR with GLOBAL column ids).  Each step gathers from the
 * caller-owned full buffer full_dev (n_global x ld, plan dtype) holding Q(r-1)
 * and writes the local Q(r) into q[r & 1] (q0_dev/q1_dev: caller-owned
 * n_rows x ld buffers, or NULL for the plan's own).  Between steps the caller
 * all-gathers the local Q(r) of every rank into full_dev (e.g. NCCL
 * all_gather_into_tensor).  Stored-order accumulation per row is unchanged,
 * so the assembled E is bit-identical to the single-GPU run.  */
int csemb_plan_partition(csemb_plan *p, int64_t row0, int64_t n_global, void *full_dev, void *q0_dev,
                         void *q1_dev);
/* Fused exchange over peer memory (instead of an all-gather between steps).
 * full0_dev / full1_dev: this rank's two replicated n_global x ld buffers;
 * Q(r) lives in parity r & 1.  peer_full0[i] / peer_full1[i]: the same two
 * buffers of peer i, mapped into this process (CUDA IPC / torch symmetric
 * memory over NVLink); n_peer <= 15.  Step r gathers from full[(r-1) & 1]
 * and its epilogue stores each Q(r) row in place into this rank's rows of
 * full[r & 1] AND into the same rows of every peer's full[r & 1], so the
 * exchange overlaps the step.  The caller places one barrier across ranks
 * after each step (all of Q(r) delivered, all reads of Q(r-1) done) and before
 * the next.  Generated projections only (SPLITMIX / PHILOX); results are
 * bit-identical to the all-gather variant and to one GPU.  */
int csemb_plan_partition_peers(csemb_plan *p, int64_t row0, int64_t n_global, void *full0_dev,
                               void *full1_dev, int n_peer, void *const *peer_full0,
                               void *const *peer_full1);
/* Same exchange through NVLS multicast: mc0 / mc1 are the multicast addresses
 * of full0 / full1 (a multicast object bound to every rank's replica, e.g.
 * torch symmetric memory's multicast_ptr).  K1 stores each Q(r) row once
 * (multimem.st) and the NVSwitch writes it into every replica, so each GPU
 * sends its rows once instead of once per peer.  */
int csemb_plan_partition_multicast(csemb_plan *p, int64_t row0, int64_t n_global, void *full0_dev,
                                   void *full1_dev, void *mc0, void *mc1);
/* Split exchange (SURVEY 8(e) "Overlap"): like csemb_plan_partition, and the
 * row block is split by column into the entries inside its own row range
 * [row0, row0 + n_rows) and the rest.  Step r is then
 *   csemb_plan_step_local(p, r)  -- the local-column partial sums from this
 *                                   rank's own Q(r-1) rows (q[(r-1) & 1]),
 *                                   launchable while the caller's all-gather
 *                                   of Q(r-1) into full is still in flight;
 *   csemb_plan_step(p, r)         -- after the all-gather: the remote-column
 *                                   partial sums, Q(r) = alpha * ((+0 + local)
 *                                   + remote) - beta * Q(r-2), the E fold and
 *                                   the diagnostics, into q[r & 1].
 * Per row, local columns are summed before remote ones: the result agrees
 * with the single-GPU stored order within rounding, not bit for bit. */
int csemb_plan_partition_split(csemb_plan *p, int64_t row0, int64_t n_global, void *full_dev,
                               void *q0_dev, void *q1_dev);
int csemb_plan_step_local(csemb_plan *p, int r);
/* Stage init for the local rows (hash of the GLOBAL row index); for generated
 * kinds also writes the full Q(0) into full_dev (no exchange before step 1). */
int csemb_plan_begin(csemb_plan *p, const double *coeffs, int order, const double *block_dev,
                     int omega_kind, uint64_t seed, int64_t col0, int64_t d_global);
int csemb_plan_step(csemb_plan *p, int r); /* r = 1..order, asynchronous */
int csemb_plan_end(csemb_plan *p, int normalize_rows);

/* ---- projection block: sample_projection (engine.py:79-99) -----------------
 * Columns [col0, col0+w) of the n x d_global block, hashed with the global d.
 * kind CSEMB_OMEGA_SPLITMIX is bit-identical to the reference.  */
int csemb_sample_projection(csemb_ctx *ctx, int64_t n, int64_t d_global, uint64_t seed,
                            int64_t col0, int64_t w, int kind, double *out_host);

/* ---- row normalisation (K4) of an external device block -------------------
 * E_i <- E_i / ||E_i||, zero rows stay 0 (the semantics of the reference's
 * cosine harness, oracle.py:88-96); used after assembling column shards.  */
int csemb_rownorm(csemb_ctx *ctx, void *E_dev, int64_t n, int64_t d, int64_t ld, int dtype);

/* ---- spectral norm: estimate_spectral_norm (engine.py:165-192) -------------
 * k start vectors: v0_host (n x k f64, unnormalised -- pass the reference's
 * PCG64 block for parity) or NULL for Philox normals from `seed`.  Returns
 * max over iterations of max|Rayleigh quotient| times `safety`.  */
int csemb_spectral_norm(csemb_mat *m, int iters, int64_t k, const double *v0_host,
                        uint64_t seed, double safety, double *out);

/* ---- downstream consumers of an embedding -------------
 * Reference: cluster.py (k-means, modularity) and oracle.py:88-119 (sampled
 * pair correlations).  Row squared norms follow numpy's pairwise order and
 * centroid sums follow np.add.at's row order (bit-identical); dot products are
 * fused in a fixed order where the reference uses BLAS (agreement to ulps).  */

/* _pair_correlations (oracle.py:88-96): cos_out[p] = <E_a, E_b> / (|E_a| |E_b|)
 * for pairs_host[2p], pairs_host[2p+1]; zero-norm pairs give 0 and
 * zero_out[p] = 1 (zero_out may be NULL).  E: n x ld block, in device memory
 * (on_device != 0, e.g. csemb_plan_output) or on the host (uploaded).  */
int csemb_pair_cosines(csemb_ctx *ctx, const void *E, int dtype, int on_device, int64_t n, int64_t d,
                       int64_t ld, const int64_t *pairs_host, int64_t n_pairs, double *cos_out,
                       uint8_t *zero_out);

/* k-means (cluster.py:59-107).  The caller runs the reference's loop and owns
 * the random stream (numpy Generator); the handle holds an f64 copy of X and
 * the device state.  Steps:
 *   seed(k, row, &total)   centroid k = X[row]; closest = d2 (k == 0) or
 *                          min(closest, d2); total = sum(closest)   (:46-55)
 *   pick(u, &row)          rng.choice(n, p=closest/total) given u = rng.random()
 *                          (first i with cumsum(p)[i] / cumsum(p)[-1] > u)
 *   assign(&inertia, &changed, counts)  labels/mindist of the current
 *                          centroids, sum(mindist), #labels changed, counts (:74-82)
 *   reseed(c, &row)        empty cluster c: row = argmax(avail); centroid c =
 *                          X[row]; new_labels[row] = c; avail[row] = -1 (:84-90)
 *   commit(update)         labels = new_labels; update != 0 also recomputes the
 *                          centroids as per-cluster means (:95-100)  */
int csemb_kmeans_create(csemb_ctx *ctx, const void *X, int dtype, int on_device, int64_t n, int64_t d,
                        int64_t ld, int K, csemb_kmeans **out);
int csemb_kmeans_destroy(csemb_kmeans *km);
int csemb_kmeans_seed(csemb_kmeans *km, int k, int64_t row, double *total);
int csemb_kmeans_pick(csemb_kmeans *km, double u, int64_t *row);
int csemb_kmeans_assign(csemb_kmeans *km, double *inertia, int64_t *changed, int64_t *counts);
int csemb_kmeans_reseed(csemb_kmeans *km, int c, int64_t *row);
int csemb_kmeans_commit(csemb_kmeans *km, int update_centroids);
int csemb_kmeans_download(csemb_kmeans *km, int64_t *labels_host, double *centroids_host);
int csemb_kmeans_set_centroids(csemb_kmeans *km, const double *centroids_host);
int csemb_kmeans_reset(csemb_kmeans *km); /* labels back to -1 for a new restart (same rows) */
const int32_t *csemb_kmeans_labels(csemb_kmeans *km); /* device, n int32 (current labels) */

/* modularity (cluster.py:110-128) counts over the matrix's CSR pattern, which
 * must be the simple undirected graph (each edge stored both ways, no
 * diagonal -- e.g. a normalized_adjacency).  intra[c] = edges inside cluster c,
 * degsum[c] = sum of degrees in c, for labels in [0, k).  The caller forms
 * Q = sum(intra/m - (degsum/2m)^2) with m = nnz/2 exactly as the reference.  */
int csemb_modularity_counts(csemb_mat *m, const int32_t *labels, int on_device, int64_t k, int64_t *intra,
                            int64_t *degsum);

#ifdef __cplusplus
}
#endif
#endif /* CSEMB_CUDA_H */
