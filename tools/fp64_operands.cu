// FP64 pipe throughput vs number of distinct register operands (RF-bank model check).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double *out, int iters, double a0) {
    double x[8], y[8], z[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) { x[c] = threadIdx.x * 1e-3 + c; y[c] = a0 + c * 1e-9; z[c] = 1e-12 * c; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (MODE == 0) x[c] = fma(x[c], 0.999999, 1e-7);          // 1 reg operand + 2 immediates/const
            if (MODE == 1) x[c] = fma(x[c], y[0], z[0]);               // 3 distinct, y/z shared across chains
            if (MODE == 2) x[c] = fma(y[c], z[c], x[c]);               // 3 distinct per chain
            if (MODE == 3) x[c] = x[c] * y[c];                         // DMUL 2 distinct
            if (MODE == 4) x[c] = fma(x[c], x[c], x[c]);               // 1 distinct
            if (MODE == 5) x[c] = x[c] + y[c];                         // DADD 2 distinct
        }
        if (MODE == 2) {
#pragma unroll
            for (int c = 0; c < 8; ++c) y[c] = y[c] * 0.0 + 1.0000001;   // keep y alive, cheap
        }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;
}
template <int MODE> void run(double *d, int sms, const char *name, int extra) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int grid = sms * 8, thr = 256, iters = 20000;
    k<MODE><<<grid, thr>>>(d, 100, 1.0);
    cudaEventRecord(e0);
    k<MODE><<<grid, thr>>>(d, iters, 1.0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)grid * thr * iters * (8 + extra);
    printf("{\"mode\":\"%s\",\"fp64_lane_ops_per_sm_per_clk_at_1965\":%.2f}\n", name, ops / (ms * 1e-3) / sms / 1.965e9);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *d; cudaMalloc(&d, 8);
    run<0>(d, sms, "dfma_1reg", 0);
    run<1>(d, sms, "dfma_3reg_shared", 0);
    run<2>(d, sms, "dfma_3reg_distinct(+8 dfma y-refresh)", 8);
    run<3>(d, sms, "dmul_2reg", 0);
    run<4>(d, sms, "dfma_same_reg", 0);
    run<5>(d, sms, "dadd_2reg", 0);
    return 0;
}
