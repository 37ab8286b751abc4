// runtime.h -- handle structs and error plumbing shared by the C-ABI translation
// units (csemb_cuda.cu: recurrence, projection, norm; downstream.cu: pair cosines,
// k-means, modularity).  Internal: not part of include/csemb_cuda.h.
#pragma once
#include <cuda_runtime.h>

#include <mutex>
#include <vector>

#include "../../include/csemb_cuda.h"

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
#define CSEMB_INTERNAL __attribute__((visibility("hidden")))

// sets the thread-local csemb_last_error() text and returns `code`
CSEMB_INTERNAL int fail(int code, const char *fmt, ...);

#define CK(...)                                                                            \
    do {                                                                                   \
        cudaError_t e_ = (__VA_ARGS__);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            cudaGetLastError();                                                            \
            return fail(e_ == cudaErrorMemoryAllocation ? CSEMB_ERR_NOMEM : CSEMB_ERR_CUDA, \
                        "%s failed: %s (%s:%d)", #__VA_ARGS__, cudaGetErrorString(e_), __FILE__,     \
                        __LINE__);                                                         \
        }                                                                                  \
    } while (0)

// ---------------------------------------------------------------------------
// handles
// ---------------------------------------------------------------------------
struct csemb_ctx {
    int device = 0;
    int sm_count = 0;
    cudaStream_t stream = nullptr;
    std::mutex mu;
    void *scratch = nullptr;  // grow-only device scratch for per-call temporaries
    size_t scratch_bytes = 0;
    cudaMemPool_t pool = nullptr;  // stream-ordered allocations of this context (dmalloc/dfree)
};

// Device memory of a context: stream-ordered allocations from the context's pool
// on its stream.  Freed blocks stay in the pool (up to its release threshold)
// and are reused without cudaMalloc/cudaFree round trips; an allocation that
// fails trims the pool and retries once.
CSEMB_INTERNAL cudaError_t dmalloc(csemb_ctx *c, void **p, size_t bytes);
CSEMB_INTERNAL void dfree(csemb_ctx *c, void *p);
template <typename T>
static inline cudaError_t dmalloc(csemb_ctx *c, T **p, size_t bytes) {
    return dmalloc(c, reinterpret_cast<void **>(p), bytes);
}

// the context's scratch buffer with at least `bytes` (call with c->mu held;
// valid until the next call that grows it)
CSEMB_INTERNAL cudaError_t ctx_scratch(csemb_ctx *c, size_t bytes, void **out);

// Load-balance schedule of a matrix for one group width G (see K1c in kernels.cuh):
// rows longer than `threshold` are cut into chunks of `chunk` entries (heavy);
// the other rows are swept in natural order or, when their lengths are skewed,
// stably bucketed by batch count ceil(len/G) so a warp's rows need the same
// number of batches.
struct Schedule {
    int G = 0;
    int64_t threshold = 0;
    int order = 0;
    int64_t wcols = 0;  // heavy-row chunks never straddle a multiple of wcols columns (0: fixed chunks)
    int *perm = nullptr;  // light rows (null: natural order, no heavy rows)
    int64_t n_light = 0;
    int64_t *cbeg = nullptr, *cend = nullptr;  // heavy-row chunk entry ranges
    int64_t n_chunks = 0;
    int *hrows = nullptr, *hoff = nullptr;     // heavy rows and their chunk offsets
    int n_heavy = 0;
    int *corder = nullptr;  // chunk execution order: by first column, so concurrently
                            // running chunks gather neighbouring rows (L2 reuse)
};

struct csemb_mat {
    csemb_ctx *ctx = nullptr;
    int64_t n_rows = 0, n_cols = 0, nnz = 0;
    int dtype = CSEMB_F64;
    int64_t *rowptr = nullptr;
    int *cols = nullptr;
    void *vals = nullptr;
    std::vector<int64_t> rowptr_host;
    std::vector<Schedule *> schedules;
    // value-free normalized adjacency (kernels.cuh k_vf_check / vf_value): a
    // device int, 1 while every stored value is 1/sqrt(len(row) len(col));
    // checked once, lazily, on the context stream (-1 = not checked yet)
    int *vf_flag = nullptr;
    int vf_state = -1;
    // row-length statistics (max, sum, sum of squares in row order), computed on
    // the host while csemb_matrix_upload's copies are in flight; the schedule
    // builder reuses them
    bool len_stats = false;
    int64_t len_max = 0;
    double len_s1 = 0.0, len_s2 = 0.0;
};

CSEMB_INTERNAL size_t dsize(int dtype);
// a matrix handle with device arrays for n_rows+1 offsets / nnz ids / nnz values
// (rowptr_host left empty); mat_free releases everything incl. schedules
CSEMB_INTERNAL int mat_alloc(csemb_ctx *c, int64_t n_rows, int64_t n_cols, int64_t nnz, int dtype,
                             csemb_mat **out);
CSEMB_INTERNAL void mat_free(csemb_mat *m);
// a row block's columns split at its own row range [lo, hi): *loc holds the
// entries with lo <= col < hi (ids col - lo, n_rows x (hi - lo)), *rem the
// rest (global ids); both keep each row's stored order (build.cu; call with
// the context lock held)
CSEMB_INTERNAL int mat_split_columns(csemb_mat *m, int64_t lo, int64_t hi, csemb_mat **loc, csemb_mat **rem);
// the light-row order of a schedule with no split rows: rows 0..n-1 stably
// sorted by (r / window, key), key = min(exact ? len : ceil(len / G), 2^16)
// (window 0: one window); *perm is a new device array (dmalloc) of n ids
// (build.cu; call with the context lock held)
CSEMB_INTERNAL int sched_order_device(csemb_mat *m, int G, bool exact, int64_t window, int **perm);
CSEMB_INTERNAL int grid_for(int64_t work_items, int threads, int sm_count, int per_sm = 8);
