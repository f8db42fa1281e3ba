// Microbenchmark of the symmetric pair mix (22 FP64 + 1 MUFU.RCP64H per pair-pair)
// in registers only, vs the same with the MUFU replaced by a DMUL.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rcp_approx(double x) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
template <int CH, bool MUFU>
__global__ void k(double *out, int iters, double sx0, double sy0) {
    double tx[CH], ty[CH], ax[CH], ay[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) { tx[c] = threadIdx.x * 1e-3 + c; ty[c] = 0.5 * c; ax[c] = 0; ay[c] = 0; }
    double sx = sx0, sy = sy0, qa = 0.3, qb = 0.2, qc = 0.1, bx = 0, by = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const double rx = tx[c] - sx, ry = ty[c] - sy;
            const double xx = rx * rx, xy = rx * ry, yy = fma(ry, ry, 1e-300);
            const double d = xx + yy;
            double inv = MUFU ? rcp_approx(d) : d * 0.999;
            const double e = fma(-d, inv, 1.0);
            inv = fma(inv, fma(e, e, e), inv);
            const double q = inv * inv;
            const double cs = fma(qa, xx, fma(qb, xy, qc * yy)) * q;
            const double ct = fma(qc, xx, fma(qa, xy, qb * yy)) * q;
            ax[c] = fma(cs, rx, ax[c]); ay[c] = fma(cs, ry, ay[c]);
            bx = fma(-ct, rx, bx); by = fma(-ct, ry, by);
        }
        sx += 1e-7; sy -= 1e-7;
    }
    double s = bx + by;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += ax[c] + ay[c];
    if (s == 12345.678) out[0] = s;
}
template <int CH, bool MUFU> void run(double *d, int sms, int warps) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int thr = 32 * warps, iters = 4000;
    k<CH, MUFU><<<sms, thr>>>(d, 10, 0.1, 0.2);
    cudaEventRecord(e0);
    k<CH, MUFU><<<sms, thr>>>(d, iters, 0.1, 0.2);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double instr = (double)sms * thr * iters * CH * 22 + (double)sms * thr * iters * 2;  // FP64 lane-instr
    printf("{\"chains\":%d,\"mufu\":%d,\"warps_per_smsp\":%.1f,\"fp64_pipe_pct\":%.1f}\n", CH, (int)MUFU, warps / 4.0,
           100.0 * instr / (ms * 1e-3) / sms / 1.965e9 / 64);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *d; cudaMalloc(&d, 8);
    for (int w : {8, 16, 32}) { run<8, true>(d, sms, w); run<8, false>(d, sms, w); run<4, true>(d, sms, w); }
    return 0;
}
