// fp64peak.cu -- FP64 CUDA-core throughput ceilings on this B200 (the roofline
// denominator of the k-means assignment kernel K8, which issues separately
// rounded DMUL + DADD pairs to keep numpy's rounding).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/fp64peak tools/fp64peak.cu && tools/fp64peak
//
// dfma    : 8 independent fused chains per thread           (2 flop / DFMA)
// dmul+dadd: 8 independent a = a + x*y chains, unfused       (2 flop / pair)
// dmma    : 8 independent mma.sync.m8n8k4.f64 accumulator chains per warp
//           (512 flop / instruction) -- the FP64 tensor-core path, for the
//           question "would DMMA lift K8's ceiling?"
// CUDA events, best of 5, grid = 8 blocks x 256 threads per SM.
#include <cuda_runtime.h>
#include <stdio.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <bool FUSED>
__global__ void k_fp64(double *out, int iters, double x, double y) {
    double a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = FUSED ? fma(a[i], x, y) : __dadd_rn(a[i], __dmul_rn(a[i], x));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 12345.678) out[0] = s;
}

__global__ void k_dmma(double *out, int iters, double x, double y) {
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(x), "d"(y));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[0] = s;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    CK(cudaMalloc(&out, 8));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int grid = sms * 8, block = 256, iters = 8192;
    for (int fused = 1; fused >= 0; --fused) {
        float best = 1e30f;
        for (int rep = 0; rep < 6; ++rep) {
            cudaEventRecord(a);
            if (fused)
                k_fp64<true><<<grid, block>>>(out, iters, 0.999999, 1e-7);
            else
                k_fp64<false><<<grid, block>>>(out, iters, 1e-9, 0.0);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep) best = ms < best ? ms : best;  // first launch is warm-up
        }
        const double flops = 2.0 * 8 * iters * (double)grid * block;
        printf("%-10s %.2f TFLOP/s\n", fused ? "dfma" : "dmul+dadd", flops / best / 1e9);
    }
    {
        float best = 1e30f;
        for (int rep = 0; rep < 6; ++rep) {
            cudaEventRecord(a);
            k_dmma<<<grid, block>>>(out, iters, 1e-9, 1e-9);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep) best = ms < best ? ms : best;
        }
        // one m8n8k4 = 8*8*4*2 = 512 flop per warp instruction
        const double flops = 512.0 * 8 * iters * (double)grid * (block / 32);
        printf("%-10s %.2f TFLOP/s\n", "dmma", flops / best / 1e9);
    }
    return 0;
}
