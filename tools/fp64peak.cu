// fp64peak.cu -- FP64 CUDA-core throughput ceilings on this B200 (the roofline
// denominator of the k-means assignment kernel K8, which issues separately
// rounded DMUL + DADD pairs to keep numpy's rounding).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/fp64peak tools/fp64peak.cu && tools/fp64peak
//
// dfma    : 8 independent fused chains per thread           (2 flop / DFMA)
// dmul+dadd: 8 independent a = a + x*y chains, unfused       (2 flop / pair)
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
    return 0;
}
