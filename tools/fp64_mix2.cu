// FP64 pipe microbenchmark, round 2: why the symmetric pair mix (21 FP64 +
// 1 MUFU.RCP64H per unordered pair) reaches ~80% of the pipe at 2 warps/SMSP
// while pure DFMA chains reach ~92%.
//   dmul / dadd / dfma : independent chains of one instruction type
//   mix  FMAIFY=0      : the k_dlp_sym pair-pair (Q' form) in registers, SR targets x NS sources
//   mix  FMAIFY=1      : the same with every DADD/DMUL written as a DFMA
//                        (a - b = fma(a, one, -b), a b = fma(a, b, zero), one/zero at run time)
// Prints FP64 lane-instructions per SM per clock as % of 64 (clock 1965 MHz assumed;
// the run's clocks are sampled separately).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ double rcp_approx(double x) {
    double r;
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    return r;
}

template <int OPK, int CH>
__global__ void k_chain(double *out, int iters, double y0) {
    double x[CH], yv[CH], zv[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        x[c] = threadIdx.x * 1e-3 + c;
        yv[c] = y0 + c * 1e-12 * threadIdx.x;  // distinct registers per chain
        zv[c] = y0 * 1e-9 * (c + threadIdx.x);
    }
    const double y = y0, z = y0 * 1e-9;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            if (OPK == 0) x[c] = x[c] * y;
            if (OPK == 1) x[c] = x[c] + z;
            if (OPK == 2) x[c] = fma(x[c], y, z);
            if (OPK == 3) x[c] = fma(x[c], yv[c], zv[c]);  // 3 distinct operands, no reuse
            if (OPK == 4) x[c] = x[c] * yv[c];             // 2 distinct operands
            if (OPK == 5) x[c] = x[c] + zv[c];
        }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;
}

template <bool F>
__device__ __forceinline__ double sub_(double a, double b, double one) { return F ? fma(a, one, -b) : a - b; }
template <bool F>
__device__ __forceinline__ double mul_(double a, double b, double zero) { return F ? fma(a, b, zero) : a * b; }

template <int SR, int NS, bool F>
__global__ void k_mix(double *out, int iters, double one, double zero) {
    double tx[SR], ty[SR], ta[SR], tb[SR], tc[SR], ax[SR], ay[SR];
#pragma unroll
    for (int r = 0; r < SR; ++r) {
        tx[r] = threadIdx.x * 1e-3 + r;
        ty[r] = 0.5 * r;
        ta[r] = 0.3 + r;
        tb[r] = 0.2;
        tc[r] = 0.1;
        ax[r] = ay[r] = 0.0;
    }
    // the sources come from shared memory as in k_dlp_sym: lane l reads source
    // (l + i + k 32/NS) mod 32 at step i; the source accumulators rotate by __shfl
    __shared__ double2 s_xy[4][32], s_ab[4][32];
    __shared__ double s_c[4][32];
    const int lane = threadIdx.x & 31, wv = (threadIdx.x >> 5) & 3;
    s_xy[wv][lane] = make_double2(0.1 * lane + 7.0, 0.2 * lane - 3.0);
    s_ab[wv][lane] = make_double2(0.3, 0.2 * lane);
    s_c[wv][lane] = 0.1;
    __syncwarp();
    double bx[NS], by[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) bx[k] = by[k] = 0.0;
    for (int i = 0; i < iters; ++i) {
        double sx[NS], sy[NS], sa[NS], sb[NS], sc[NS];
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            const int l = (lane + i + k * (32 / NS)) & 31;
            const double2 xy = s_xy[wv][l], ab = s_ab[wv][l];
            sx[k] = xy.x; sy[k] = xy.y; sa[k] = ab.x; sb[k] = ab.y; sc[k] = s_c[wv][l];
        }
#pragma unroll
        for (int r = 0; r < SR; ++r) {
#pragma unroll
            for (int k = 0; k < NS; ++k) {
                const double rx = sub_<F>(tx[r], sx[k], one), ry = sub_<F>(ty[r], sy[k], one);
                const double yy = fma(ry, ry, 1e-150), xy = mul_<F>(rx, ry, zero);
                const double d = fma(rx, rx, yy);
                double iv = rcp_approx(d);
                const double cs = fma(sa[k], d, fma(sb[k], xy, mul_<F>(sc[k], yy, zero)));
                const double ct = fma(ta[r], d, fma(tb[r], xy, mul_<F>(tc[r], yy, zero)));
                const double e = fma(-d, iv, 1.0);
                iv = fma(iv, fma(e, e, e), iv);
                const double q = mul_<F>(iv, iv, zero);
                const double a = mul_<F>(cs, q, zero), b = mul_<F>(ct, q, zero);
                ax[r] = fma(a, rx, ax[r]);
                ay[r] = fma(a, ry, ay[r]);
                bx[k] = fma(-b, rx, bx[k]);
                by[k] = fma(-b, ry, by[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            bx[k] = __shfl_sync(0xffffffffu, bx[k], (lane + 1) & 31);
            by[k] = __shfl_sync(0xffffffffu, by[k], (lane + 1) & 31);
        }
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < NS; ++k) s += bx[k] + by[k];
#pragma unroll
    for (int r = 0; r < SR; ++r) s += ax[r] + ay[r];
    if (s == 12345.678) out[0] = s;
}

static float time_ms(void (*launch)(double *, int), double *d, int iters) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch(d, 10);
    cudaEventRecord(e0);
    launch(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}

static int g_sms, g_thr, g_grid;

template <int OPK, int CH>
static void chain(int warps_per_sm) {
    double *d;
    cudaMalloc(&d, 8);
    g_thr = 128;
    g_grid = g_sms * warps_per_sm / 4;
    const int iters = 100000 / CH;
    float ms = time_ms([](double *o, int it) { k_chain<OPK, CH><<<g_grid, g_thr>>>(o, it, 0.999999); }, d, iters);
    double ops = (double)g_grid * g_thr * iters * CH;
    const char *nm[6] = {"dmul", "dadd", "dfma", "dfma_distinct", "dmul_distinct", "dadd_distinct"};
    printf("{\"kind\":\"%s\",\"chains\":%d,\"warps_per_smsp\":%.2f,\"pct_of_64\":%.1f}\n", nm[OPK], CH,
           warps_per_sm / 4.0, 100.0 * ops / (ms * 1e-3) / g_sms / 1.965e9 / 64);
    cudaFree(d);
}

template <int SR, int NS, bool F>
static void mix(int warps_per_sm) {
    double *d;
    cudaMalloc(&d, 8);
    g_thr = 128;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_mix<SR, NS, F>, 128, 0);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_mix<SR, NS, F>);
    if (occ * 4 < warps_per_sm) {  // that many warps do not fit at this register count
        printf("{\"kind\":\"mix\",\"SR\":%d,\"NS\":%d,\"fmaify\":%d,\"warps_per_smsp\":%.2f,\"skipped\":\"regs %d, "
               "%d CTAs/SM\"}\n", SR, NS, (int)F, warps_per_sm / 4.0, fa.numRegs, occ);
        cudaFree(d);
        return;
    }
    g_grid = g_sms * warps_per_sm / 4;
    const int iters = 2000;
    float ms = time_ms([](double *o, int it) { k_mix<SR, NS, F><<<g_grid, g_thr>>>(o, it, 1.0, 0.0); }, d, iters);
    double ops = (double)g_grid * g_thr * iters * SR * NS * 21;  // FP64 lane-instructions
    printf("{\"kind\":\"mix\",\"SR\":%d,\"NS\":%d,\"fmaify\":%d,\"warps_per_smsp\":%.2f,\"regs\":%d,\"pct_of_64\":%.1f}\n",
           SR, NS, (int)F, warps_per_sm / 4.0, fa.numRegs, 100.0 * ops / (ms * 1e-3) / g_sms / 1.965e9 / 64);
    cudaFree(d);
}

int main() {
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0);
    for (int w : {8, 16}) {
        chain<2, 8>(w);
        chain<3, 8>(w);
        chain<4, 8>(w);
        chain<5, 8>(w);
        chain<3, 16>(w);
    }
    if (getenv("MIX2_CHAINS_ONLY")) return 0;
    for (int w : {8, 12, 16}) {
        mix<8, 2, false>(w);
        mix<8, 2, true>(w);
        mix<4, 2, false>(w);
        mix<4, 2, true>(w);
        mix<4, 4, false>(w);
        mix<4, 4, true>(w);
        mix<2, 4, true>(w);
    }
    return 0;
}
