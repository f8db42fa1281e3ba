// Does the FP64 tensor path (mma.sync m8n8k4 f64, "DMMA") share the FP64
// CUDA-core pipe (DFMA)?  Three runs on all SMs: DFMA chains only, DMMA chains
// only, and both in the same CTAs (half the warps each).  Reports FP64 FMA
// throughput of each part in TFLOP/s (2 flop per FMA; DMMA m8n8k4 = 256 FMA).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
// mode 0: all warps DFMA; 1: all warps DMMA; 2: even warps DFMA, odd warps DMMA
__global__ void __launch_bounds__(256) k_mix(int iters, int mode, double *out) {
    const int w = threadIdx.x >> 5;
    const bool do_dmma = mode == 1 || (mode == 2 && (w & 1));
    double a[8], c0[8], c1[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) { a[q] = 1.0 + 1e-9 * (threadIdx.x + q); c0[q] = c1[q] = 0.0; }
    const double b = 0.999999;
    if (do_dmma) {
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int q = 0; q < 8; ++q) dmma(c0[q], c1[q], a[q], b);
        }
    } else {
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                c0[q] = fma(a[q], b, c0[q]);
                c1[q] = fma(a[q], c1[q], b);
            }
        }
    }
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += c0[q] + c1[q];
    if (s == 123.456) out[0] = s;
}
int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    cudaMalloc(&out, 8);
    const int blocks = sms * 4, threads = 256, iters = 20000;
    for (int mode = 0; mode < 3; ++mode) {
        k_mix<<<blocks, threads>>>(100, mode, out);
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        k_mix<<<blocks, threads>>>(iters, mode, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        const double warps = (double)blocks * threads / 32;
        const double dfma_warps = mode == 0 ? warps : mode == 1 ? 0 : warps / 2;
        const double dmma_warps = warps - dfma_warps;
        const double dfma_flop = dfma_warps * 32 * iters * 16 * 2.0;   // 16 DFMA per iteration per lane
        const double dmma_flop = dmma_warps * iters * 8 * 256 * 2.0;   // 8 DMMA per iteration per warp
        printf("{\"mode\": \"%s\", \"ms\": %.3f, \"dfma_tflops\": %.2f, \"dmma_tflops\": %.2f, \"total_tflops\": %.2f, \"err\": \"%s\"}\n",
               mode == 0 ? "dfma" : mode == 1 ? "dmma" : "both", ms, dfma_flop / ms / 1e9, dmma_flop / ms / 1e9,
               (dfma_flop + dmma_flop) / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
