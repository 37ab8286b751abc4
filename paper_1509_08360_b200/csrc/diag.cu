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

}  // namespace

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
