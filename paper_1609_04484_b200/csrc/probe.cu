// probe.cu -- measurement hook: the FP64 peak of THIS device, measured in-run
// (bench.py reports the all-pairs roofline against it beside the derived
// 148 SM x 64 FMA/clk x 2 x f_max figure; MEASURED_PEAKS.json has no FP64 entry).
#include <cuda_runtime.h>

#include "internal.cuh"

namespace bie {

// 8 independent DFMA chains per thread, 8 CTAs of 256 threads per SM
// (8 warps per SMSP): enough independent work to saturate the FP64 pipe.
__global__ void __launch_bounds__(256) k_fp64_peak(double *out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;  // never true; keeps the chains live
}

}  // namespace bie

using namespace bie;

extern "C" int bie_fp64_peak(int iters, double *tflops, double *ms, void *stream) {
    if (!tflops || !ms || iters < 1) {
        set_error("bie_fp64_peak: null output or iters < 1");
        return BIE_EINVAL;
    }
    int dev = 0, sms = 0;
    BIE_CUDA_TRY(cudaGetDevice(&dev));
    BIE_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    cudaStream_t st = (cudaStream_t)stream;
    double *d = nullptr;
    BIE_CUDA_TRY(cudaMalloc(&d, sizeof(double)));
    cudaEvent_t e0, e1;
    BIE_CUDA_TRY(cudaEventCreate(&e0));
    BIE_CUDA_TRY(cudaEventCreate(&e1));
    const int grid = sms * 8, thr = 256;
    k_fp64_peak<<<grid, thr, 0, st>>>(d, iters / 10 + 1, 0.999999, 1e-7);  // warm-up / clock ramp
    BIE_CUDA_TRY(cudaEventRecord(e0, st));
    k_fp64_peak<<<grid, thr, 0, st>>>(d, iters, 0.999999, 1e-7);
    BIE_CUDA_TRY(cudaEventRecord(e1, st));
    count_launch(2);
    BIE_CUDA_TRY(cudaEventSynchronize(e1));
    float t = 0.f;
    BIE_CUDA_TRY(cudaEventElapsedTime(&t, e0, e1));
    *ms = t;
    *tflops = 2.0 * 8.0 * (double)grid * thr * (double)iters / (t * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d);
    return BIE_OK;
}
