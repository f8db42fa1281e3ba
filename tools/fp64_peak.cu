// FP64 pipe microbenchmark: independent DFMA chains on every SM, CUDA events.
// Prints achieved DFMA TFLOP/s (2 flop per DFMA) and the SM clock seen via clock64.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k_dfma(double *out, int iters, double a, double b) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;
}
__global__ void k_rcp(double *out, int iters, double a) {
    double x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = 1.0 + threadIdx.x * 1e-3 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x[c])); x[c] = r + a; }
    }
    double s = 0;
    for (int c = 0; c < 8; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;
}
__global__ void k_rcp_err(double *out, int n) {
    // max |1 - x * rcp.approx(x)| over x = 1 + j/n (all mantissas), via exact FMA residual
    double m = 0;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        double x = (1.0 + (double)j / n) * 3.7e-3;
        double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
        double e = fabs(fma(-x, r, 1.0));
        m = fmax(m, e);
    }
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax((unsigned long long *)out, __double_as_longlong(m));
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *d; cudaMalloc(&d, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int iters = 20000;
    for (int blocksPerSm : {4, 8}) {
        int grid = sms * blocksPerSm, thr = 256;
        k_dfma<8><<<grid, thr>>>(d, 1000, 0.999999, 1e-7);
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) k_dfma<8><<<grid, thr>>>(d, iters, 0.999999, 1e-7);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 5.0 * grid * thr * (double)iters * 8 * 2;
        printf("{\"test\":\"dfma\",\"blocks_per_sm\":%d,\"tflops\":%.3f,\"ms\":%.3f}\n", blocksPerSm, flops / (ms * 1e-3) / 1e12, ms);
    }
    {
        int grid = sms * 8, thr = 256;
        k_rcp<<<grid, thr>>>(d, 1000, 1e-9);
        cudaEventRecord(e0);
        k_rcp<<<grid, thr>>>(d, iters, 1e-9);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)grid * thr * iters * 8;
        printf("{\"test\":\"rcp64h+dadd\",\"gops\":%.1f,\"per_sm_per_clk_at_1965\":%.2f}\n", ops / (ms * 1e-3) / 1e9, ops / (ms * 1e-3) / sms / 1.965e9);
    }
    {
        cudaMemset(d, 0, 8);
        k_rcp_err<<<sms * 4, 256>>>(d, 1 << 26);
        double h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("{\"test\":\"rcp_approx_seed_max_rel_err\",\"value\":%.3e,\"log2\":%.2f}\n", h, log2(h));
    }
    return 0;
}
