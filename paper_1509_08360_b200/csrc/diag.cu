// diag.cu -- live memory-system ceilings for the roofline objects of bench.py.
//
// K1 (kernels.cuh) moves two kinds of bytes: HBM traffic (the north_star's
// algorithmic model) and the gathered rows of Q(r-1) that cross the L2 -> SM
// fabric, T*ld*dtype per step (3.7x the algorithmic HBM bytes on config 2).
// The measured peaks in MEASURED_PEAKS.json cover only the first.  These
// probes measure, on the same device and right next to the timed K1 region
// (same clocks / power state), the ceilings of the second:
//   CSEMB_DIAG_L2_STREAM : coalesced 16-byte .cg loads re-reading an
//                          L2-resident buffer (the fabric's streaming rate)
//   CSEMB_DIAG_L2_GATHER : K1's load shape -- G lanes x up to 3 x 16 B per
//                          row of row_bytes (G as K1 picks it: 16 for
//                          640-byte rows, 8 for 320-byte rows), rows at random
//                          inside the window, 4 rows in flight per lane group
//   CSEMB_DIAG_HBM_COPY  : read + write of a DRAM-sized buffer (the
//                          MEASURED_PEAKS definition, at these clocks)
// They are measurement tools, not part of the embedding path.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <mutex>

#include "runtime.h"

namespace {

__device__ __forceinline__ float4 ld_cg4(const float4 *p) {
    float4 v;
    asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}

__global__ void k_diag_stream(const float4 *__restrict__ a, int64_t n, int reps, float *sink) {
    float acc = 0.f;
    for (int r = 0; r < reps; ++r)
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
            const float4 v = ld_cg4(a + i);
            acc += v.x + v.y + v.z + v.w;
        }
    if (acc == 1234.5f) *sink = acc;
}

// G-lane groups (K1's group for this row width: the smallest power of two
// with ceil(vpr / G) <= 3); each lane reads vectors gl, gl+G, gl+2G (< vpr) of
// a row; 4 rows in flight per group (K1's shape: 16 lanes for 640-byte fp64
// rows, 8 lanes for 320-byte fp32 rows)
template <int G>
__global__ void k_diag_gather(const float4 *__restrict__ a, uint32_t nrows, int vpr, uint32_t rows_per_group,
                              float *sink) {
    const int gl = threadIdx.x & (G - 1);
    const uint32_t g = (blockIdx.x * blockDim.x + threadIdx.x) / G;
    uint32_t h = g * 2654435761u + 12345u;
    float acc = 0.f;
    for (uint32_t it = 0; it < rows_per_group; it += 4) {
        float4 v[4][3];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            h = h * 1664525u + 1013904223u;
            const uint32_t row = (uint32_t)(((uint64_t)(h >> 3) * nrows) >> 29);
            const float4 *p = a + (size_t)row * vpr + gl;
#pragma unroll
            for (int k = 0; k < 3; ++k)
                v[u][k] = (gl + G * k < vpr) ? __ldg(p + G * k) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int k = 0; k < 3; ++k) acc += v[u][k].x + v[u][k].y + v[u][k].z + v[u][k].w;
    }
    if (acc == 1234.5f) *sink = acc;
}

__global__ void k_diag_copy(const float4 *__restrict__ a, float4 *b, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        b[i] = __ldcs(a + i);
}

// Gather-only pass over a real matrix: every stored entry fetches the whole
// row of Q(r-1) its column id names -- exactly K1's gathered bytes, in the
// matrix's stored order, with K1's lanes per row -- but with no recurrence,
// no epilogue and no streamed blocks, and U entries in flight per lane group
// (K1 keeps 4 in fp64 / 2 in fp32).  The warps sweep consecutive entry blocks
// in grid-stride order, so the set of rows gathered at any moment is the
// same moving front as K1's row sweep.  Its time is the floor for any K1
// that reads the gathered rows through the L1/L2 load path.
template <int G, int U>
__global__ void __launch_bounds__(256, 2) k_diag_csr_gather(const int *__restrict__ cols, int64_t nnz,
                                                           const float4 *__restrict__ q, int ldv, int nv,
                                                           float *sink) {
    constexpr int RPW = 32 / G;  // lane groups per warp
    constexpr int VPL = 3;
    const int lane = threadIdx.x & 31, gl = lane & (G - 1), grp = lane / G;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    constexpr int EPW = RPW * U;  // entries per warp block
    bool valid[VPL];
#pragma unroll
    for (int k = 0; k < VPL; ++k) valid[k] = gl + k * G < nv;
    float acc = 0.f;
    auto ids = [&](int64_t blk, int (&j)[U], bool (&ok)[U]) {
        const int64_t e0 = blk * EPW + (int64_t)grp * U;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            ok[u] = e0 + u < nnz;
            j[u] = ok[u] ? __ldg(cols + e0 + u) : 0;
        }
    };
    int j[U];
    bool ok[U];
    ids(warp, j, ok);
    for (int64_t blk = warp; blk * EPW < nnz; blk += nwarps) {
        float4 v[U][VPL];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const float4 *p = q + (int64_t)j[u] * ldv + gl;
#pragma unroll
            for (int k = 0; k < VPL; ++k)
                v[u][k] = (ok[u] && valid[k]) ? __ldg(p + k * G) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        ids(blk + nwarps, j, ok);  // next block's ids while this block's gathers are in flight
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < VPL; ++k) acc += v[u][k].x + v[u][k].y + v[u][k].z + v[u][k].w;
    }
    if (acc == 1234.5f) *sink = acc;
}

template <int U>
static void launch_csr_gather(int G, int grid, cudaStream_t s, const int *cols, int64_t nnz, const float4 *q,
                              int nv, float *sink) {
    switch (G) {
        case 1: k_diag_csr_gather<1, U><<<grid, 256, 0, s>>>(cols, nnz, q, nv, nv, sink); break;
        case 2: k_diag_csr_gather<2, U><<<grid, 256, 0, s>>>(cols, nnz, q, nv, nv, sink); break;
        case 4: k_diag_csr_gather<4, U><<<grid, 256, 0, s>>>(cols, nnz, q, nv, nv, sink); break;
        case 8: k_diag_csr_gather<8, U><<<grid, 256, 0, s>>>(cols, nnz, q, nv, nv, sink); break;
        case 16: k_diag_csr_gather<16, U><<<grid, 256, 0, s>>>(cols, nnz, q, nv, nv, sink); break;
        default: k_diag_csr_gather<32, U><<<grid, 256, 0, s>>>(cols, nnz, q, nv, nv, sink); break;
    }
}

}  // namespace

extern "C" int csemb_diag_gather_csr(csemb_mat *m, int64_t row_bytes, int in_flight, double *ms_out,
                                     double *gbs_out) {
    if (!m || !m->ctx || !ms_out || !gbs_out) return fail(CSEMB_ERR_INVALID, "null argument");
    if (row_bytes < 16 || row_bytes % 16 || row_bytes > 96 * 16)
        return fail(CSEMB_ERR_INVALID, "row_bytes must be a multiple of 16 in [16, 1536]");
    if (in_flight != 4 && in_flight != 8) return fail(CSEMB_ERR_INVALID, "in_flight must be 4 or 8");
    csemb_ctx *c = m->ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    const int nv = (int)(row_bytes / 16);
    int G = 1;
    while (G < 32 && (nv + G - 1) / G > 3) G *= 2;  // K1's lanes per row
    const int64_t qbytes = (m->n_cols > 0 ? m->n_cols : 1) * row_bytes;
    void *q = nullptr, *sink = nullptr;
    cudaError_t e = dmalloc(c, &q, (size_t)qbytes);
    if (e == cudaSuccess) e = dmalloc(c, &sink, 16);
    if (e == cudaSuccess) e = cudaMemsetAsync(q, 0, (size_t)qbytes, s);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (e == cudaSuccess) e = cudaEventCreate(&e0);
    if (e == cudaSuccess) e = cudaEventCreate(&e1);
    float best = 1e30f;
    const int grid = c->sm_count * 2;  // 2 CTAs x 256 threads per SM, as K1
    for (int rep = 0; rep < 4 && e == cudaSuccess; ++rep) {
        e = cudaEventRecord(e0, s);
        if (e == cudaSuccess) {
            if (in_flight == 8)
                launch_csr_gather<8>(G, grid, s, m->cols, m->nnz, (const float4 *)q, nv, (float *)sink);
            else
                launch_csr_gather<4>(G, grid, s, m->cols, m->nnz, (const float4 *)q, nv, (float *)sink);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaEventRecord(e1, s);
        if (e == cudaSuccess) e = cudaEventSynchronize(e1);
        float ms = 0.f;
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
        if (e == cudaSuccess && rep > 0) best = std::min(best, ms);  // first launch warms up
    }
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    dfree(c, q);
    dfree(c, sink);
    CK(e);
    CK(cudaStreamSynchronize(s));
    *ms_out = best;
    *gbs_out = (double)m->nnz * (double)row_bytes / (best * 1e-3) / 1e9;
    return CSEMB_OK;
}

extern "C" int csemb_diag_bandwidth(csemb_ctx *c, int kind, int64_t bytes, int64_t row_bytes, int reps,
                                    double *gbs_out) {
    if (!c || !gbs_out) return fail(CSEMB_ERR_INVALID, "null argument");
    if (bytes < (1 << 20) || reps < 1) return fail(CSEMB_ERR_INVALID, "need bytes >= 1 MiB and reps >= 1");
    if (kind == CSEMB_DIAG_L2_GATHER && (row_bytes < 16 || row_bytes % 16 || row_bytes > 768))
        return fail(CSEMB_ERR_INVALID, "row_bytes must be a multiple of 16 in [16, 768]");
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    const int64_t nvec = bytes / 16;
    void *a = nullptr, *b = nullptr, *sink = nullptr;
    cudaError_t e = dmalloc(c, &a, (size_t)nvec * 16);
    if (e == cudaSuccess && kind == CSEMB_DIAG_HBM_COPY) e = dmalloc(c, &b, (size_t)nvec * 16);
    if (e == cudaSuccess) e = dmalloc(c, &sink, 16);
    if (e == cudaSuccess) e = cudaMemsetAsync(a, 0, (size_t)nvec * 16, s);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (e == cudaSuccess) e = cudaEventCreate(&e0);
    if (e == cudaSuccess) e = cudaEventCreate(&e1);
    double moved = 0.0;
    float best = 1e30f;
    const int sms = c->sm_count;
    auto launch = [&]() {
        if (kind == CSEMB_DIAG_L2_STREAM) {
            k_diag_stream<<<sms * 4, 512, 0, s>>>((const float4 *)a, nvec, reps, (float *)sink);
            moved = (double)nvec * 16.0 * reps;
        } else if (kind == CSEMB_DIAG_L2_GATHER) {
            const int vpr = (int)(row_bytes / 16);
            const uint32_t nrows = (uint32_t)(bytes / row_bytes);
            int G = 1;
            while (G < 16 && (vpr + G - 1) / G > 3) G *= 2;
            const uint32_t groups = (uint32_t)sms * 2 * 256 / G;  // 2 CTAs x 256 threads per SM, as K1
            const uint32_t per = (uint32_t)std::max<int64_t>(4, (int64_t)reps * 4 * G / 16);
            switch (G) {
                case 1: k_diag_gather<1><<<sms * 2, 256, 0, s>>>((const float4 *)a, nrows, vpr, per, (float *)sink); break;
                case 2: k_diag_gather<2><<<sms * 2, 256, 0, s>>>((const float4 *)a, nrows, vpr, per, (float *)sink); break;
                case 4: k_diag_gather<4><<<sms * 2, 256, 0, s>>>((const float4 *)a, nrows, vpr, per, (float *)sink); break;
                case 8: k_diag_gather<8><<<sms * 2, 256, 0, s>>>((const float4 *)a, nrows, vpr, per, (float *)sink); break;
                default: k_diag_gather<16><<<sms * 2, 256, 0, s>>>((const float4 *)a, nrows, vpr, per, (float *)sink);
            }
            moved = (double)groups * per * row_bytes;
        } else {
            k_diag_copy<<<sms * 8, 512, 0, s>>>((const float4 *)a, (float4 *)b, nvec);
            moved = 2.0 * (double)nvec * 16.0;
        }
    };
    for (int rep = 0; rep < 4 && e == cudaSuccess; ++rep) {
        e = cudaEventRecord(e0, s);
        if (e == cudaSuccess) launch();
        if (e == cudaSuccess) e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaEventRecord(e1, s);
        if (e == cudaSuccess) e = cudaEventSynchronize(e1);
        float ms = 0.f;
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
        if (e == cudaSuccess && rep > 0) best = std::min(best, ms);  // first launch warms up
    }
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    dfree(c, a);
    dfree(c, b);
    dfree(c, sink);
    CK(e);
    CK(cudaStreamSynchronize(s));
    *gbs_out = moved / (best * 1e-3) / 1e9;
    return CSEMB_OK;
}
