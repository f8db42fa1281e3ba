// Cost of one cooperative-groups grid barrier on the B200 (the BD factor's
// cooperative panel does one per column): G CTAs x 128 threads, `iters`
// barriers, each preceded by a global store and followed by a global load of
// a neighbour's value (the panel's candidate exchange pattern).
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__global__ void k_sync(int iters, double *buf, int mode) {
    cg::grid_group grid = cg::this_grid();
    double acc = 0.0;
    for (int it = 0; it < iters; ++it) {
        if (mode && threadIdx.x == 0) buf[blockIdx.x + (it & 1) * gridDim.x] = acc + it;
        grid.sync();
        if (mode && threadIdx.x < 32) acc += __ldcg(buf + ((blockIdx.x + threadIdx.x) % gridDim.x) + (it & 1) * gridDim.x);
    }
    if (acc == -1.0) buf[0] = acc;
}
int main() {
    double *buf;
    cudaMalloc(&buf, sizeof(double) * 4096);
    for (int G : {32, 62, 124, 148, 296}) {
        for (int mode : {0, 1}) {
            int iters = 4096;
            void *args[] = {&iters, &buf, &mode};
            cudaLaunchCooperativeKernel((void *)k_sync, G, 128, args, 0, 0);
            cudaDeviceSynchronize();
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void *)k_sync, G, 128, args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("{\"ctas\": %d, \"exchange\": %d, \"us_per_barrier\": %.3f, \"err\": \"%s\"}\n", G, mode,
                   ms * 1000.0 / iters, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
