// FP64 pipe throughput vs warps per SMSP and independent chains per warp.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double *out, int iters) {
    double x[CH], y[CH], z[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) { x[c] = threadIdx.x * 1e-3 + c; y[c] = 0.999999 + c * 1e-9; z[c] = 1e-12 * c; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = fma(x[c], y[c], z[c]);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c] + y[c] + z[c];
    if (s == 12345.678) out[0] = s;
}
template <int CH> void run(double *d, int sms, int warps_per_sm) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int thr = 32 * warps_per_sm, grid = sms, iters = 200000 / CH;
    k<CH><<<grid, thr>>>(d, 100);
    cudaEventRecord(e0);
    k<CH><<<grid, thr>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)grid * thr * iters * CH;
    printf("{\"chains\":%d,\"warps_per_smsp\":%.1f,\"pct_of_64\":%.1f}\n", CH, warps_per_sm / 4.0, 100.0 * ops / (ms * 1e-3) / sms / 1.965e9 / 64);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *d; cudaMalloc(&d, 8);
    for (int w : {4, 8, 16, 32}) { run<1>(d, sms, w); run<2>(d, sms, w); run<4>(d, sms, w); run<8>(d, sms, w); run<16>(d, sms, w); }
    return 0;
}
