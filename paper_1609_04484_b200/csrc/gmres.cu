// gmres.cu -- left-preconditioned full GMRES on one GPU (A8, A9).
//
// P:l.596-601 (GMRES, tol 1e-8 on the relative residual), P:l.661-663 (left
// preconditioning P^{-1} A sigma = P^{-1} f), P:l.678-686 (the residual pair).
// Reading C13: x0 = 0, no restart, CGS2, Givens, happy breakdown when
// H[k+1,k] <= 1e-14 ||P^{-1} A v_k||, strict "<" on the estimate.
//
// The Krylov basis V[0..max_iter] lives in HBM ([max_iter+1][2N]).  Vector
// kernels are deterministic two-stage reductions (fixed chunking, fixed order):
//   k_multidot  : partial[chunk][j] = V[j, chunk] . w[chunk], j = 0..k   (reads V once)
//   k_reduce    : h[j] = sum_chunk partial[chunk][j]
//   k_multiaxpy : w -= V[0..k]^T h   (or x = V^T y)                     (reads V once)
//   k_givens    : Hessenberg column update + new rotation on one thread
// The host reads each iteration's estimate 3 iterations behind the enqueue
// front (speculative iterations touch only entries the finish never reads), and
// the workspace is cached on the geometry (no allocation per solve).  The same
// driver serves the SLP system (kOpSLP) and batched multi-RHS solves.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <cmath>
#include <mutex>
#include <unordered_map>
#include <utility>
#include <vector>

#include "internal.cuh"

namespace bie {

constexpr int kChunk = 4096;      // elements of the 2N dimension per multidot CTA
constexpr int kDotThreads = 128;  // 4 basis vectors share one staged w chunk (batched kernels)
constexpr int kDotThreads1 = 256;  // k_multidot: 8 warps share the staged chunk (occupancy, round 2)

struct GmState {
    double *H;      // column-major: H[k * ldh + j], ldh = max_iter + 1
    double *cs, *sn, *g;
    double *h, *h2; // CGS passes
    double *scal;   // [0] beta, [1] w0^2 -> w0, [2] hk1^2 -> hk1, [3] est, [4] breakdown flag, [5] tmp
};

// sqrt(a^2 + b^2) correctly rounded (reading C28): a^2 + b^2 exactly as a
// double-double, a correctly rounded sqrt of its head, one Newton correction
// in double-double, one final rounding.  Library hypot() implementations
// differ by an ulp (glibc vs CUDA), which left the Givens recurrence of the
// two GMRES implementations not uniquely defined.
__device__ __forceinline__ double hypot_cr(double a, double b) {
    const double p = a * a, pe = fma(a, a, -p);
    const double q = b * b, qe = fma(b, b, -q);
    const double sh = p + q, t = sh - p;
    double se = (p - (sh - t)) + (q - t);
    se += pe + qe;
    const double s1 = sh + se, s1e = se - (s1 - sh);
    if (s1 == 0.0) return 0.0;
    const double r = __dsqrt_rn(s1);
    const double rr = r * r, rre = fma(r, r, -rr);
    return r + (((s1 - rr) - rre) + s1e) / (2.0 * r);
}

// One Givens step of GMRES (reading C13): H[:,k] = h + h2, H[k+1,k] = hk1,
// old rotations, new rotation, g, estimate, breakdown flag.  Every operation is
// the oracle's, in its order, without contraction (_rn intrinsics) and with a
// correctly rounded hypot, so equal inputs give bit-identical outputs.
__device__ __forceinline__ void givens_step(double *Hk, double *cs, double *sn, double *g, const double *h,
                                            const double *h2, double *scal, int k) {
    for (int j = 0; j <= k; ++j) Hk[j] = __dadd_rn(h[j], h2[j]);
    const double hk1 = scal[2];
    Hk[k + 1] = hk1;
    for (int j = 0; j < k; ++j) {
        const double a = Hk[j], b = Hk[j + 1];
        Hk[j] = __dadd_rn(__dmul_rn(cs[j], a), __dmul_rn(sn[j], b));
        Hk[j + 1] = __dadd_rn(__dmul_rn(-sn[j], a), __dmul_rn(cs[j], b));
    }
    const double a = Hk[k], b = Hk[k + 1];
    const double d = hypot_cr(a, b);
    cs[k] = __ddiv_rn(a, d);
    sn[k] = __ddiv_rn(b, d);
    Hk[k] = d;
    Hk[k + 1] = 0.0;
    g[k + 1] = __dmul_rn(-sn[k], g[k]);
    g[k] = __dmul_rn(cs[k], g[k]);
    scal[3] = __ddiv_rn(fabs(g[k + 1]), scal[0]);
    scal[4] = (hk1 <= __dmul_rn(1e-14, scal[1])) ? 1.0 : 0.0;
}

// Tail of a fused kernel (GMRES iteration): after the thread that
// finishes h_{k+1,k} = ||w|| has stored it, it runs the Givens step of
// iteration k = ctl[0] (k_givens_dev's work: hist[k + 1], ctl[1] = converged,
// ctl[0] = k + 1 and, in the CUDA-graph solve, the while-loop condition).
struct GivensTail {
    GmState s;
    int *ctl = nullptr;
    int ldh = 0, max_iter = 0;
    double tol = 0.0;
    double *hist = nullptr;
    cudaGraphConditionalHandle cond = 0;
    int use_cond = 0;
    int on = 0;
};
__device__ __forceinline__ void givens_tail(const GivensTail &t) {
    const int k = t.ctl[0];
    unsigned cont = 0;
    if (k < t.max_iter) {
        givens_step(t.s.H + (long long)k * t.ldh, t.s.cs, t.s.sn, t.s.g, t.s.h, t.s.h2, t.s.scal, k);
        const double est = t.s.scal[3];
        const int conv = (est < t.tol || t.s.scal[4] != 0.0) ? 1 : 0;
        t.hist[k + 1] = est;
        t.ctl[1] = conv;
        t.ctl[0] = k + 1;
        cont = (!conv && k + 1 < t.max_iter) ? 1u : 0u;
    }
    if (t.use_cond) cudaGraphSetConditional(t.cond, cont);
}

// partial[c * ldp + j] = sum_{e in chunk c} V[j][e] * w[e] for j in [0, nv).
// Grid (chunks, Gy); warp wid of CTA y owns basis vectors j = 4y + wid + 4 Gy q
// and reduces the whole 4096-element chunk for each (fixed lane order ->
// deterministic; the j loop does not change any per-j sum).  kdev != nullptr
// (GMRES iteration): nv = min(*kdev + 1, nv), the iteration count read on the
// device.  sq: store sqrt of the dot (a norm; single-chunk case only).
// xv != nullptr: one more vector, xv itself, is dotted with w as column nv
// (its chunk sum is computed by the same code, so the result is bitwise that
// of a separate norm launch); single chunk: sqrt of it goes to xout.
// gt.on (single chunk, nv = 1): the thread that stores the norm then runs the
// Givens step (givens_tail).
__global__ void __launch_bounds__(kDotThreads1, 3) k_multidot(const double *__restrict__ V, long long ldv, int nv,
                                                          const int *kdev, const double *__restrict__ w, long long n,
                                                          double *partial, int ldp, int sq, const double *xv,
                                                          double *xout, GivensTail gt) {
    pdl_wait();
    if (kdev) nv = min(*kdev + 1, nv);
    const int ntot = nv + (xv ? 1 : 0);
    if ((int)blockIdx.y * (kDotThreads1 / 32) >= ntot) return;
    __shared__ double ws[kChunk];
    const long long e0 = (long long)blockIdx.x * kChunk;
    const int len = (int)std::min<long long>(kChunk, n - e0);
    for (int q = threadIdx.x; q < kChunk; q += kDotThreads1) ws[q] = q < len ? w[e0 + q] : 0.0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int j = blockIdx.y * (kDotThreads1 / 32) + wid; j < ntot; j += gridDim.y * (kDotThreads1 / 32)) {
        const bool extra = j == nv;
        const double *vj = (extra ? xv : V + (long long)j * ldv) + e0;
        // eight independent streams per lane: ~16 warps per SM with 4 loads each
        // in flight left the kernel latency-bound at 0.70 of the HBM bandwidth
        // (ncu, profiles/round2/gmres_vec_r2_summary.txt)
        double ac[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        int q = lane;
        for (; q + 224 < len; q += 256) {
            double a[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) a[u] = __ldcs(vj + q + 32 * u);
#pragma unroll
            for (int u = 0; u < 8; ++u) ac[u] = fma(a[u], ws[q + 32 * u], ac[u]);
        }
        for (; q < len; q += 32) ac[0] = fma(vj[q], ws[q], ac[0]);
        double acc = ((ac[0] + ac[1]) + (ac[2] + ac[3])) + ((ac[4] + ac[5]) + (ac[6] + ac[7]));
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        BIE_DCHECK(j < ldp || gridDim.x == 1);
        if (lane == 0) {
            if (extra && gridDim.x == 1) {
                *xout = sqrt(acc);
            } else {
                partial[(long long)blockIdx.x * ldp + j] = sq ? sqrt(acc) : acc;
                if (gt.on && j == 0 && gridDim.x == 1) givens_tail(gt);
            }
        }
    }
}

// Small vectors (one chunk, n <= kChunk: configs 1-2): one CTA of 256 threads
// per basis vector (grid-stride over j) and a fixed-order block reduction.
// k_multidot's one warp per vector streamed a config-2 vector (3584 doubles)
// with 4 loads in flight per lane: 11 us per launch, latency-bound.  Same
// operands and outputs as k_multidot's single-chunk case (extra column xv ->
// sqrt into xout; Givens tail).
__global__ void __launch_bounds__(256) k_multidot_small(const double *__restrict__ V, long long ldv, int nv,
                                                        const int *kdev, const double *__restrict__ w, int n,
                                                        double *out, int sq, const double *xv, double *xout,
                                                        GivensTail gt) {
    pdl_wait();
    if (kdev) nv = min(*kdev + 1, nv);
    const int ntot = nv + (xv ? 1 : 0);
    __shared__ double red[8];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (int j = blockIdx.x; j < ntot; j += gridDim.x) {
        const bool extra = j == nv;
        const double *vj = extra ? xv : V + (long long)j * ldv;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int e = tid;
        for (; e + 768 < n; e += 1024) {
            const double v0 = vj[e], v1 = vj[e + 256], v2 = vj[e + 512], v3 = vj[e + 768];
            a0 = fma(v0, w[e], a0);
            a1 = fma(v1, w[e + 256], a1);
            a2 = fma(v2, w[e + 512], a2);
            a3 = fma(v3, w[e + 768], a3);
        }
        for (; e < n; e += 256) a0 = fma(vj[e], w[e], a0);
        double acc = (a0 + a1) + (a2 + a3);
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) red[wid] = acc;
        __syncthreads();
        if (tid == 0) {
            double t = red[0];
            for (int q = 1; q < 8; ++q) t += red[q];
            if (extra) {
                *xout = sqrt(t);
            } else {
                out[j] = sq ? sqrt(t) : t;
                if (gt.on && j == 0) givens_tail(gt);
            }
        }
        __syncthreads();
    }
}

// out[j] = (accumulate ? out[j] : 0) + sum_c partial[c * ldp + j]  (fixed order)
// Sum of column j over the chunks in chunk order.  The loads are issued in
// batches of 16 ahead of the (still sequential, so bitwise unchanged) adds: the
// serial load-add loop was latency-bound (8.9 us per launch at 67 chunks).
__device__ __forceinline__ double sum_chunks(const double *__restrict__ p, long long ldp, int nchunks) {
    double t = 0.0;
    int c = 0;
    for (; c + 16 <= nchunks; c += 16) {
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = p[(long long)(c + u) * ldp];
#pragma unroll
        for (int u = 0; u < 16; ++u) t += v[u];
    }
    for (; c < nchunks; ++c) t += p[(long long)c * ldp];
    return t;
}

// xout != nullptr: column nv (the extra vector of k_multidot) -> sqrt into
// *xout.  gt.on: thread 0 runs the Givens step after storing out[0].
__global__ void k_reduce(const double *__restrict__ partial, int ldp, int nchunks, int nv, const int *kdev,
                         double *out, int accumulate, int sq, double *xout, GivensTail gt) {
    pdl_wait();
    if (kdev) nv = min(*kdev + 1, nv);
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nv + (xout ? 1 : 0)) return;
    const double t = sum_chunks(partial + j, ldp, nchunks);
    if (j == nv) {
        *xout = sqrt(t);
        return;
    }
    const double r = accumulate ? out[j] + t : t;
    out[j] = sq ? sqrt(r) : r;
    if (gt.on && j == 0) givens_tail(gt);
}

// y[e] = beta * y[e] + alpha * sum_j V[j][e] * c[j]   (c in device memory, any nv).
// The coefficients are staged through shared memory in tiles of kAxpyTile
// (static 16 KB, so no dynamic-smem limit on nv = k + 1); the sum over j stays
// one sequential FMA chain per element, so results do not depend on the tiling.
constexpr int kAxpyTile = 2048;
__device__ __forceinline__ double axpy_chain(const double *__restrict__ V, long long ldv, int j0, int j1,
                                             const double *cs, long long e, double acc) {
    int j = j0;
    for (; j + 4 <= j1; j += 4) {
        const double a0 = V[(long long)j * ldv + e], a1 = V[(long long)(j + 1) * ldv + e];
        const double a2 = V[(long long)(j + 2) * ldv + e], a3 = V[(long long)(j + 3) * ldv + e];
        acc = fma(a0, cs[j - j0], acc);
        acc = fma(a1, cs[j + 1 - j0], acc);
        acc = fma(a2, cs[j + 2 - j0], acc);
        acc = fma(a3, cs[j + 3 - j0], acc);
    }
    for (; j < j1; ++j) acc = fma(V[(long long)j * ldv + e], cs[j - j0], acc);
    return acc;
}

__global__ void __launch_bounds__(256) k_multiaxpy(const double *__restrict__ V, long long ldv, int nv,
                                                   const int *kdev, const double *__restrict__ c, double alpha,
                                                   double beta, double *y, long long n) {
    pdl_wait();
    if (kdev) nv = min(*kdev + 1, nv);
    __shared__ double cs[kAxpyTile];
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const bool act = e < n;
    double acc = 0.0;
    for (int j0 = 0; j0 < nv; j0 += kAxpyTile) {
        const int j1 = min(nv, j0 + kAxpyTile);
        __syncthreads();
        for (int q = threadIdx.x; q < j1 - j0; q += blockDim.x) cs[q] = c[j0 + q];
        __syncthreads();
        if (act) acc = axpy_chain(V, ldv, j0, j1, cs, e, acc);
    }
    if (act) y[e] = (beta == 0.0 ? 0.0 : beta * y[e]) + alpha * acc;
}

// Small vectors (n <= kChunk): 32 elements per CTA, warp w sums the vectors
// j = w, w + 8, ... for its lane's element, the 8 partials are added in warp
// order (fixed; 8x the memory-level parallelism of one chain per element).
__global__ void __launch_bounds__(256) k_multiaxpy_small(const double *__restrict__ V, long long ldv, int nv,
                                                         const int *kdev, const double *__restrict__ c, double alpha,
                                                         double beta, double *y, long long n) {
    pdl_wait();
    if (kdev) nv = min(*kdev + 1, nv);
    __shared__ double part[8][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long long e = (long long)blockIdx.x * 32 + lane;
    double acc = 0.0;
    if (e < n) {
        int j = wid;
        for (; j + 24 < nv; j += 32) {
            const double v0 = V[(long long)j * ldv + e], v1 = V[(long long)(j + 8) * ldv + e];
            const double v2 = V[(long long)(j + 16) * ldv + e], v3 = V[(long long)(j + 24) * ldv + e];
            acc = fma(v0, c[j], acc);
            acc = fma(v1, c[j + 8], acc);
            acc = fma(v2, c[j + 16], acc);
            acc = fma(v3, c[j + 24], acc);
        }
        for (; j < nv; j += 8) acc = fma(V[(long long)j * ldv + e], c[j], acc);
    }
    part[wid][lane] = acc;
    __syncthreads();
    if (wid == 0 && e < n) {
        double t = part[0][lane];
        for (int q = 1; q < 8; ++q) t += part[q][lane];
        y[e] = (beta == 0.0 ? 0.0 : beta * y[e]) + alpha * t;
    }
}

__global__ void k_sqrt(const double *in, double *out) { *out = sqrt(*in); }

// y = x / (*s)
__global__ void k_scale_div(const double *x, const double *s, double *y, long long n) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n) y[e] = x[e] / *s;
}

__global__ void k_sub(const double *a, const double *b, double *y, long long n) {
    pdl_wait();
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n) y[e] = a[e] - b[e];
}

// Hessenberg column k: H[:,k] = h + h2, H[k+1,k] = hk1; apply old rotations, new rotation.
__global__ void k_givens(GmState s, int k, int ldh) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    givens_step(s.H + (long long)k * ldh, s.cs, s.sn, s.g, s.h, s.h2, s.scal, k);
}

// v = x / (*s) into the current-vector buffer and into V[ctl[0]] (when
// ctl[0] < max_iter): the next Krylov vector, at the device-side index.
__global__ void k_scale_store(const double *x, const double *s, double *V, long long n, const int *ctl,
                              int max_iter, double *vcur) {
    pdl_wait();
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    const double y = x[e] / *s;
    vcur[e] = y;
    const int k = *ctl;
    if (k < max_iter) V[(long long)k * n + e] = y;
}

// y = H^{-1} g (upper triangular, iters x iters), one CTA
__global__ void k_trisolve(const double *H, int ldh, const double *g, double *y, int iters) {
    pdl_wait();
    __shared__ double red[32];
    __shared__ double yi_s;
    for (int i = iters - 1; i >= 0; --i) {
        double acc = 0.0;
        for (int j = i + 1 + threadIdx.x; j < iters; j += blockDim.x) acc = fma(H[(long long)j * ldh + i], y[j], acc);
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += red[q];
            yi_s = (g[i] - t) / H[(long long)i * ldh + i];
            y[i] = yi_s;
        }
        __syncthreads();
    }
}

struct Dot {
    double *partial = nullptr;
    int nchunks = 0;
    int ldp = 0;
};

// out[0..nv) = V[0..nv)^T w (deterministic).  kdev: nv = min(*kdev + 1, nv) on
// the device (graph body; the grid is sized for the cap nv).  sq: out = sqrt.
static int multidot(const double *V, long long ldv, int nv, const double *w, long long n, Dot &d, double *out,
                    cudaStream_t st, const int *kdev = nullptr, int sq = 0, const double *xv = nullptr,
                    double *xout = nullptr, const GivensTail &gt = GivensTail{}) {
    const int ncap = nv + (xv ? 1 : 0);
    const int gy_full = (ncap + kDotThreads1 / 32 - 1) / (kDotThreads1 / 32);
    // device-side nv: cap the y extent (each warp loops over its vectors) so
    // that the mostly idle tail of a max_iter-sized grid stays small
    const int gy = kdev ? std::max(1, std::min(gy_full, (8 * 148 + d.nchunks - 1) / d.nchunks)) : gy_full;
    if (d.nchunks == 1) {  // one chunk (2N <= 4096): one CTA per vector, no reduction launch
        BIE_LAUNCH(k_multidot_small, std::min(ncap, 2 * 148), 256, 0, st, V, ldv, nv, kdev, w, (int)n, out, sq, xv,
                   xout, gt);
        count_launch();
        BIE_CUDA_TRY(cudaGetLastError());
        return BIE_OK;
    }
    BIE_LAUNCH(k_multidot, dim3(d.nchunks, gy), kDotThreads1, 0, st, V, ldv, nv, kdev, w, n, d.partial, d.ldp, 0, xv,
               xout, GivensTail{});
    BIE_LAUNCH(k_reduce, (ncap + 127) / 128, 128, 0, st, d.partial, d.ldp, d.nchunks, nv, kdev, out, 0, sq, xout, gt);
    count_launch(2);
    BIE_CUDA_TRY(cudaGetLastError());
    return BIE_OK;
}

static int multiaxpy(const double *V, long long ldv, int nv, const double *c, double alpha, double beta, double *y,
                     long long n, cudaStream_t st, const int *kdev = nullptr) {
    if (n <= kChunk)
        BIE_LAUNCH(k_multiaxpy_small, (unsigned)((n + 31) / 32), 256, 0, st, V, ldv, nv, kdev, c, alpha, beta, y, n);
    else
        BIE_LAUNCH(k_multiaxpy, (unsigned)((n + 255) / 256), 256, 0, st, V, ldv, nv, kdev, c, alpha, beta, y, n);
    count_launch();
    BIE_CUDA_TRY(cudaGetLastError());
    return BIE_OK;
}

__global__ void k_sqrt_n(const double *in, double *out, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = sqrt(in[i]);
}

// ---------------------------------------------------------------------------
// Batched (multi-RHS) forms of the vector kernels: blockIdx.z = active slot q,
// system r = act[q].  System r's basis is V + r * sysV, its small state (cs, sn,
// g, h, h2, scal) at small + r * smallper; slot q's work vector at W + q * n.
// Per system the arithmetic and the reduction order are those of the single-
// system kernels, so results are bitwise identical to looping over systems.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kDotThreads) k_multidot_b(const double *__restrict__ V, long long sysV, long long ldv,
                                                            int nv, const double *__restrict__ W, long long n,
                                                            double *partial, int ldp, long long psys,
                                                            const int *__restrict__ act, int self) {
    __shared__ double ws[kChunk];
    const int qs = blockIdx.z;
    const double *w = W + (long long)qs * n;
    const double *Vb = self ? w : V + (long long)act[qs] * sysV;  // self: the norm of w itself
    const long long e0 = (long long)blockIdx.x * kChunk;
    const int len = (int)std::min<long long>(kChunk, n - e0);
    for (int q = threadIdx.x; q < kChunk; q += kDotThreads) ws[q] = q < len ? w[e0 + q] : 0.0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int j = blockIdx.y * (kDotThreads / 32) + wid;
    if (j >= nv) return;
    const double *vj = Vb + (long long)j * ldv + e0;
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
    int q = lane;
    for (; q + 96 < len; q += 128) {
        const double a0 = __ldcs(vj + q), a1 = __ldcs(vj + q + 32), a2 = __ldcs(vj + q + 64), a3 = __ldcs(vj + q + 96);
        acc0 = fma(a0, ws[q], acc0);
        acc1 = fma(a1, ws[q + 32], acc1);
        acc2 = fma(a2, ws[q + 64], acc2);
        acc3 = fma(a3, ws[q + 96], acc3);
    }
    for (; q < len; q += 32) acc0 = fma(vj[q], ws[q], acc0);
    double acc = (acc0 + acc1) + (acc2 + acc3);
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) partial[(long long)qs * psys + (long long)blockIdx.x * ldp + j] = acc;
}

// small[act[q]] + off [j] = sum_c partial_q[c][j] (fixed order); sqrt_out: then
// the square root (norms)
__global__ void k_reduce_b(const double *__restrict__ partial, int ldp, long long psys, int nchunks, int nv,
                           double *small, long long smallper, long long off, const int *__restrict__ act,
                           int sqrt_out) {
    const int q = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nv) return;
    const double *pq = partial + (long long)q * psys;
    const double t = sum_chunks(pq + j, ldp, nchunks);
    small[(long long)act[q] * smallper + off + j] = sqrt_out ? sqrt(t) : t;
}

// W_q[e] = beta * W_q[e] + alpha * sum_j V_r[j][e] * c_r[j]  (coefficients tiled as in k_multiaxpy)
__global__ void __launch_bounds__(256) k_multiaxpy_b(const double *__restrict__ V, long long sysV, long long ldv,
                                                     int nv, const double *small, long long smallper, long long coff,
                                                     double alpha, double beta, double *W, long long n,
                                                     const int *__restrict__ act) {
    __shared__ double cs[kAxpyTile];
    const int qs = blockIdx.y, r = act[qs];
    const double *c = small + (long long)r * smallper + coff;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const bool on = e < n;
    const double *Vb = V + (long long)r * sysV;
    double acc = 0.0;
    for (int j0 = 0; j0 < nv; j0 += kAxpyTile) {
        const int j1 = min(nv, j0 + kAxpyTile);
        __syncthreads();
        for (int q = threadIdx.x; q < j1 - j0; q += blockDim.x) cs[q] = c[j0 + q];
        __syncthreads();
        if (on) acc = axpy_chain(Vb, ldv, j0, j1, cs, e, acc);
    }
    if (!on) return;
    double *y = W + (long long)qs * n;
    y[e] = (beta == 0.0 ? 0.0 : beta * y[e]) + alpha * acc;
}

// one thread per active slot: the Givens update of system act[q]; estimate and
// breakdown flag also to est[2 q], est[2 q + 1] for one D2H copy
__global__ void k_givens_b(double *Hbase, long long Hsys, double *small, long long smallper, int ldh, int k,
                           const int *__restrict__ act, int na, double *est) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= na) return;
    const int r = act[q];
    double *b = small + (long long)r * smallper;
    GmState s{Hbase + (long long)r * Hsys, b, b + ldh, b + 2 * ldh, b + 3 * ldh, b + 4 * ldh, b + 5 * ldh};
    givens_step(s.H + (long long)k * ldh, s.cs, s.sn, s.g, s.h, s.h2, s.scal, k);
    est[2 * q] = s.scal[3];
    est[2 * q + 1] = s.scal[4];
}

// V_r[k + 1] = W_q / scal_r[2]  (blockIdx.y = slot; scal at small + r * smallper + scal_off)
__global__ void k_scale_b(const double *W, long long n, double *V, long long sysV, long long koff,
                          const double *small, long long smallper, long long scal_off, const int *__restrict__ act) {
    const int qs = blockIdx.y, r = act[qs];
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n) V[(long long)r * sysV + koff + e] = W[(long long)qs * n + e] / small[(long long)r * smallper + scal_off + 2];
}

// Win_q = V_r[k]  (blockIdx.y = slot)
__global__ void k_gather_b(const double *V, long long sysV, long long koff, double *W, long long n,
                           const int *__restrict__ act) {
    const int qs = blockIdx.y;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n) W[(long long)qs * n + e] = V[(long long)act[qs] * sysV + koff + e];
}

}  // namespace bie

using namespace bie;

// ---------------------------------------------------------------------------
// Krylov building blocks (row-sharded GMRES): the same kernels
// bie_gmres_solve uses, exposed so a multi-rank driver keeps every vector
// operation in this library and only adds the collectives.
// ---------------------------------------------------------------------------
extern "C" {

int bie_krylov_dots(const double *V, long long ldv, int nv, const double *w, long long n, double *out,
                    void *stream) {
    if (!V || !w || !out || nv < 1 || n < 0) {
        set_error("bie_krylov_dots: null pointer, nv < 1 or n < 0");
        return BIE_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (n == 0) {
        BIE_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double) * nv, st));
        return BIE_OK;
    }
    Dot d;
    d.nchunks = (int)((n + kChunk - 1) / kChunk);
    d.ldp = nv;
    if (d.nchunks > 1) {
        // grow-only scratch per stream (work on one stream is ordered, so reuse is
        // safe); a cudaMallocAsync per call cost ~10 us in the sharded driver
        static std::mutex mu;
        static std::unordered_map<cudaStream_t, std::pair<double *, size_t>> scratch;
        const size_t need = (size_t)d.nchunks * nv;
        std::lock_guard<std::mutex> lock(mu);
        auto &e = scratch[st];
        if (e.second < need) {
            if (e.first) BIE_CUDA_TRY(cudaFreeAsync(e.first, st));
            const size_t cap = std::max(need, 2 * e.second);
            BIE_CUDA_TRY(cudaMallocAsync(&e.first, sizeof(double) * cap, st));
            e.second = cap;
        }
        d.partial = e.first;
    }
    return multidot(V, ldv, nv, w, n, d, out, st);
}

int bie_krylov_axpy(const double *V, long long ldv, int nv, const double *c, double alpha, double beta, double *y,
                    long long n, void *stream) {
    if (!V || !c || !y || nv < 0 || n < 0) {
        set_error("bie_krylov_axpy: null pointer, nv < 0 or n < 0");
        return BIE_EINVAL;
    }
    if (n == 0) return BIE_OK;
    return multiaxpy(V, ldv, nv, c, alpha, beta, y, n, (cudaStream_t)stream);
}

int bie_krylov_scale(const double *x, const double *s, double *y, long long n, void *stream) {
    if (!x || !s || !y || n < 0) {
        set_error("bie_krylov_scale: null pointer or n < 0");
        return BIE_EINVAL;
    }
    if (n == 0) return BIE_OK;
    k_scale_div<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(x, s, y, n);
    count_launch();
    BIE_CUDA_TRY(cudaGetLastError());
    return BIE_OK;
}

int bie_krylov_sqrt(const double *in, double *out, int n, void *stream) {
    if (!in || !out || n < 1) {
        set_error("bie_krylov_sqrt: null pointer or n < 1");
        return BIE_EINVAL;
    }
    k_sqrt_n<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(in, out, n);
    count_launch();
    BIE_CUDA_TRY(cudaGetLastError());
    return BIE_OK;
}

int bie_krylov_givens(double *H, int ldh, double *cs, double *sn, double *g, const double *h, const double *h2,
                      int k, double *scal, void *stream) {
    if (!H || !cs || !sn || !g || !h || !h2 || !scal || k < 0 || ldh < k + 2) {
        set_error("bie_krylov_givens: null pointer or bad k / ldh");
        return BIE_EINVAL;
    }
    GmState s{H, cs, sn, g, const_cast<double *>(h), const_cast<double *>(h2), scal};
    k_givens<<<1, 1, 0, (cudaStream_t)stream>>>(s, k, ldh);
    count_launch();
    BIE_CUDA_TRY(cudaGetLastError());
    return BIE_OK;
}

int bie_krylov_trisolve(const double *H, int ldh, const double *g, double *y, int iters, void *stream) {
    if (!H || !g || !y || iters < 0 || ldh < iters) {
        set_error("bie_krylov_trisolve: null pointer or bad iters / ldh");
        return BIE_EINVAL;
    }
    if (iters == 0) return BIE_OK;
    k_trisolve<<<1, 256, 0, (cudaStream_t)stream>>>(H, ldh, g, y, iters);
    count_launch();
    BIE_CUDA_TRY(cudaGetLastError());
    return BIE_OK;
}

}  // extern "C"

// opf: BIE_FULL (the completed DLP) or kOpSLP (the single-layer operator, NEXT-1)
//
// One GMRES iteration is a fixed sequence of launches whose only varying
// argument, the iteration index k, lives on the device (ctl[0]): operator apply
// on v_k (kept in vcur), CGS2 over V[0..k] (its first dot launch also gives
// ||w||), hk1 with the Givens step in the same kernel's tail (givens_tail)
// and v_{k+1} (k_scale_store).  The solve captures that sequence ONCE into the
// body of a CUDA-graph conditional WHILE node; givens_tail sets the loop
// condition, so a whole solve is one graph launch with no host round trip per
// iteration.  The instantiated graph is cached on the geometry and reused while
// the operator, BD handle, tol, max_iter and the workspace are unchanged.  With
// profiling on (bie_profile_begin: per-apply events, which a graph body cannot
// hold) or BIE_GMRES_GRAPH=0 the same sequence is enqueued from the host with a
// kLook-iteration lookahead instead.  Both forms launch the same kernels with the
// same arguments, so results are bitwise identical.
static int gmres_solve_impl(const char *fn, unsigned opf, bie_geometry_t gh, bie_blockdiag_t bdh, const double *f,
                            double *x, double tol, int max_iter, double *hist_host, int *iters, double *res_pc,
                            double *res_true, int *converged, void *stream) {
    Geometry *g = as_geom(gh);
    BlockDiag *bd = bdh ? as_bd(bdh) : nullptr;
    if (!g || (bdh && !bd) || !f || !x || !hist_host || !iters || !res_pc || !res_true || !converged ||
        max_iter < 1 || !(tol > 0.0) || f == x) {
        set_error(std::string(fn) + ": invalid handle, null pointer, f == x, max_iter < 1 or tol <= 0");
        return BIE_EINVAL;
    }
    if (bd && bd->g != g) {
        set_error(std::string(fn) + ": blockdiag was built from another geometry");
        return BIE_EINVAL;
    }
    if (bd && (bd->b0 != 0 || bd->b1 != g->M + 1)) {
        set_error(std::string(fn) + ": blockdiag covers a body range, not the whole geometry");
        return BIE_EINVAL;
    }
    if (bd && bd->op != ((opf & kOpSLP) ? 1 : 0)) {
        set_error(std::string(fn) + ": blockdiag was factored for the other operator (DLP vs SLP)");
        return BIE_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const long long n = 2LL * g->N;
    const int ldh = max_iter + 1;
    GmState s{};
    Dot d;
    constexpr int kMaxLook = 7;
    int kLook = 3;                     // host-driven form: iterations enqueued ahead of the check
    if (const char *e = getenv("BIE_GMRES_LOOKAHEAD")) kLook = std::max(1, std::min(kMaxLook, atoi(e)));
    const int kRing = kLook + 1;
    bool use_graph = !g->prof;
    if (const char *e = getenv("BIE_GMRES_GRAPH")) use_graph = use_graph && atoi(e) != 0;
    d.nchunks = (int)((n + kChunk - 1) / kChunk);
    d.ldp = ldh;
    GmresWork &ws = g->gm;
    auto ensure = [&](double *&ptr, size_t &cap, size_t need) -> cudaError_t {
        if (need <= cap) return cudaSuccess;
        cudaFree(ptr);  // synchronises the device: no work in flight uses the old buffer
        ptr = nullptr;
        cap = 0;
        cudaError_t e = cudaMalloc(&ptr, sizeof(double) * need);
        if (e == cudaSuccess) cap = need;
        return e;
    };
    BIE_CUDA_TRY(ensure(ws.V, ws.V_cap, (size_t)ldh * n));
    BIE_CUDA_TRY(ensure(ws.w, ws.n_cap, 3 * (size_t)n));  // w | t | vcur
    BIE_CUDA_TRY(ensure(ws.H, ws.H_cap, (size_t)ldh * max_iter));
    BIE_CUDA_TRY(ensure(ws.small, ws.small_cap, 6 * (size_t)ldh + 16));
    BIE_CUDA_TRY(ensure(ws.partial, ws.partial_cap, (size_t)d.nchunks * ldh));
    if (!ws.pinned) BIE_CUDA_TRY(cudaMallocHost(&ws.pinned, sizeof(double) * (8 + 2 * (kMaxLook + 1))));
    for (int q = 0; q < kRing; ++q)
        if (!ws.evs[q]) BIE_CUDA_TRY(cudaEventCreateWithFlags(&ws.evs[q], cudaEventDisableTiming));
    double *V = ws.V, *w = ws.w, *t = ws.w + n, *vcur = ws.w + 2 * n;
    double *pinned = ws.pinned;
    cudaEvent_t *evs = ws.evs;
    s.H = ws.H;
    s.cs = ws.small;
    s.sn = ws.small + ldh;
    s.g = ws.small + 2 * ldh;
    s.h = ws.small + 3 * ldh;
    s.h2 = ws.small + 4 * ldh;
    s.scal = ws.small + 5 * ldh;                         // 8 scalars
    double *hist_d = ws.small + 5 * ldh + 8;             // [ldh] estimates
    int *ctl = reinterpret_cast<int *>(ws.small + 6 * ldh + 8);  // [0] k, [1] converged
    d.partial = ws.partial;
    BIE_CUDA_TRY(cudaMemsetAsync(s.g, 0, sizeof(double) * ldh, st));
    BIE_CUDA_TRY(cudaMemsetAsync(s.H, 0, sizeof(double) * (size_t)ldh * max_iter, st));
    BIE_CUDA_TRY(cudaMemsetAsync(ctl, 0, 2 * sizeof(int), st));

    auto apply_op = [&](const double *in, double *out, cudaStream_t q) -> int {  // out = P^{-1} A in
        if (bd) {
            int r = dlp_apply_impl(g, in, t, 1, opf, 0, g->N, q);
            if (r) return r;
            return blockdiag_apply_impl(bd, t, out, 1, q);
        }
        return dlp_apply_impl(g, in, out, 1, opf, 0, g->N, q);
    };
    auto norm_to = [&](const double *v, double *dst, cudaStream_t q) -> int {  // dst = ||v|| (device)
        return multidot(v, 0, 1, v, n, d, dst, q, nullptr, 1);
    };
    const unsigned eb = (unsigned)((n + 255) / 256);
    // one iteration at the device-side index k = ctl[0]
    auto body = [&](cudaStream_t q, cudaGraphConditionalHandle cond, int use_cond) -> int {
        int r;
        if ((r = apply_op(vcur, w, q))) return r;
        // CGS2 over V[0..k]; the first pass also yields w0 = ||P^{-1} A v_k|| (w as
        // the extra column), the final norm hk1 runs the Givens step in its tail
        if ((r = multidot(V, n, ldh - 1, w, n, d, s.h, q, ctl, 0, w, s.scal + 1))) return r;
        if ((r = multiaxpy(V, n, ldh, s.h, -1.0, 1.0, w, n, q, ctl))) return r;
        if ((r = multidot(V, n, ldh, w, n, d, s.h2, q, ctl))) return r;
        if ((r = multiaxpy(V, n, ldh, s.h2, -1.0, 1.0, w, n, q, ctl))) return r;
        GivensTail gt;
        gt.s = s;
        gt.ctl = ctl;
        gt.ldh = ldh;
        gt.max_iter = max_iter;
        gt.tol = tol;
        gt.hist = hist_d;
        gt.cond = cond;
        gt.use_cond = use_cond;
        gt.on = 1;
        if ((r = multidot(w, 0, 1, w, n, d, s.scal + 2, q, nullptr, 1, nullptr, nullptr, gt))) return r;  // hk1
        BIE_LAUNCH(k_scale_store, eb, 256, 0, q, w, s.scal + 2, V, n, ctl, max_iter, vcur);
        count_launch(1);
        BIE_CUDA_TRY(cudaGetLastError());
        return BIE_OK;
    };

    // r0 = P^{-1} f, beta = ||r0||, v0 = r0 / beta
    if (bd) {
        BIE_RC_TRY(blockdiag_apply_impl(bd, f, w, 1, st));
    } else {
        BIE_CUDA_TRY(cudaMemcpyAsync(w, f, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    }
    BIE_RC_TRY(norm_to(w, s.scal + 0, st));
    BIE_CUDA_TRY(cudaMemcpyAsync(pinned, s.scal, sizeof(double), cudaMemcpyDeviceToHost, st));
    BIE_CUDA_TRY(cudaStreamSynchronize(st));
    const double beta = pinned[0];
    hist_host[0] = 1.0;
    *iters = 0;
    *converged = 0;
    BIE_CUDA_TRY(cudaMemsetAsync(x, 0, sizeof(double) * n, st));
    if (beta == 0.0) {
        *converged = 1;
        *res_pc = 0.0;
        *res_true = 0.0;
        return BIE_OK;
    }
    k_scale_store<<<eb, 256, 0, st>>>(w, s.scal + 0, V, n, ctl, max_iter, vcur);  // ctl[0] = 0: V[0]
    count_launch();
    BIE_CUDA_TRY(cudaMemcpyAsync(s.g, s.scal + 0, sizeof(double), cudaMemcpyDeviceToDevice, st));
    int it = 0;
    bool conv = false;
    use_graph = use_graph && !ws.graph_off;
    if (use_graph) {
        const GmGraphKey key{bd, bd ? bd->serial : 0, opf, max_iter, tol, V, w, ws.small, ws.partial, g->partial,
                             g->slp_s};
        if (!ws.gexec || !(ws.gkey == key)) {
            if (ws.gexec) cudaGraphExecDestroy(ws.gexec);
            if (ws.graph) cudaGraphDestroy(ws.graph);
            ws.gexec = nullptr;
            ws.graph = nullptr;
            // buffers the apply allocates lazily must exist before the capture
            BIE_RC_TRY(apply_op(vcur, w, st));
            if (!ws.cap) BIE_CUDA_TRY(cudaStreamCreateWithFlags(&ws.cap, cudaStreamNonBlocking));
            // a driver without conditional graph nodes (or any capture failure)
            // falls back to the host-enqueued loop for this geometry: same kernels
            bool capturing = false;
            auto capture = [&]() -> cudaError_t {
                cudaError_t e = cudaGraphCreate(&ws.graph, 0);
                if (e != cudaSuccess) return e;
                cudaGraphConditionalHandle cond;
                if ((e = cudaGraphConditionalHandleCreate(&cond, ws.graph, 1, cudaGraphCondAssignDefault))) return e;
                cudaGraphNodeParams cp{};
                cp.type = cudaGraphNodeTypeConditional;
                cp.conditional.handle = cond;
                cp.conditional.type = cudaGraphCondTypeWhile;
                cp.conditional.size = 1;
                cudaGraphNode_t node;
                if ((e = cudaGraphAddNode(&node, ws.graph, nullptr, 0, &cp))) return e;
                cudaGraph_t bg = cp.conditional.phGraph_out[0];
                if ((e = cudaStreamBeginCaptureToGraph(ws.cap, bg, nullptr, nullptr, 0,
                                                       cudaStreamCaptureModeRelaxed)))
                    return e;
                capturing = true;
                const long long c0 = bie_launch_count();
                const int rb = body(ws.cap, cond, 1);
                cudaGraph_t cap_out = nullptr;
                e = cudaStreamEndCapture(ws.cap, &cap_out);
                capturing = false;
                ws.body_launches = bie_launch_count() - c0;
                count_launch(-(int)ws.body_launches);  // counted per executed iteration below
                if (rb != BIE_OK) return cudaErrorUnknown;
                if (e != cudaSuccess) return e;
                return cudaGraphInstantiate(&ws.gexec, ws.graph, 0);
            };
            if (capture() != cudaSuccess) {
                if (capturing) {
                    cudaGraph_t dummy = nullptr;
                    cudaStreamEndCapture(ws.cap, &dummy);
                }
                (void)cudaGetLastError();
                if (ws.gexec) cudaGraphExecDestroy(ws.gexec);
                if (ws.graph) cudaGraphDestroy(ws.graph);
                ws.gexec = nullptr;
                ws.graph = nullptr;
                ws.graph_off = true;
                use_graph = false;
            } else {
                ws.gkey = key;
            }
        }
    }
    if (use_graph) {
        BIE_CUDA_TRY(cudaGraphLaunch(ws.gexec, st));
        BIE_CUDA_TRY(cudaMemcpyAsync(pinned + 1, ctl, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
        BIE_CUDA_TRY(cudaStreamSynchronize(st));
        const int *hc = reinterpret_cast<const int *>(pinned + 1);
        it = hc[0];
        conv = hc[1] != 0;
        count_launch((int)(ws.body_launches * it));
    } else {
        // host-driven: iteration k is enqueued before the host reads the state of
        // iteration k - kLook (so the device queue holds ~kLook iterations of
        // work).  Iterations after the converged one are speculative: they touch
        // only H[:,k], g[k..k+1], cs/sn[k], hist[k+1] and V[k+1], none of which
        // the finish reads (after a happy breakdown possibly NaNs, unused).
        bool done = false;
        auto check = [&](int kk) -> int {
            BIE_CUDA_TRY(cudaEventSynchronize(evs[kk % kRing]));
            const int *hc = reinterpret_cast<const int *>(pinned + 8 + 2 * (kk % kRing));
            it = kk + 1;
            if (hc[1]) {
                conv = true;
                done = true;
            }
            return BIE_OK;
        };
        for (int k = 0; k < max_iter && !done; ++k) {
            BIE_RC_TRY(body(st, cudaGraphConditionalHandle{}, 0));
            BIE_CUDA_TRY(cudaMemcpyAsync(pinned + 8 + 2 * (k % kRing), ctl, 2 * sizeof(int),
                                         cudaMemcpyDeviceToHost, st));
            BIE_CUDA_TRY(cudaEventRecord(evs[k % kRing], st));
            if (k >= kLook) BIE_RC_TRY(check(k - kLook));
        }
        while (!done && it < max_iter) BIE_RC_TRY(check(it));  // the iterations still in flight
    }
    *iters = it;
    *converged = conv ? 1 : 0;
    // y = H^{-1} g, x = V y
    k_trisolve<<<1, 256, 0, st>>>(s.H, ldh, s.g, s.h, it);
    count_launch();
    BIE_CUDA_TRY(cudaGetLastError());
    BIE_RC_TRY(multiaxpy(V, n, it, s.h, 1.0, 0.0, x, n, st));
    // residual pair (P:l.678-686): r = f - A x
    BIE_RC_TRY(dlp_apply_impl(g, x, t, 1, opf, 0, g->N, st));
    k_sub<<<eb, 256, 0, st>>>(f, t, w, n);
    count_launch();
    BIE_RC_TRY(norm_to(w, s.scal + 6, st));
    BIE_RC_TRY(norm_to(f, s.scal + 7, st));
    if (bd) {
        BIE_RC_TRY(blockdiag_apply_impl(bd, w, t, 1, st));
        BIE_RC_TRY(norm_to(t, s.scal + 5, st));
        BIE_CUDA_TRY(cudaMemcpyAsync(pinned + 5, s.scal + 5, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
    } else {
        BIE_CUDA_TRY(cudaMemcpyAsync(pinned + 6, s.scal + 6, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    }
    if (it > 0)
        BIE_CUDA_TRY(cudaMemcpyAsync(hist_host + 1, hist_d + 1, sizeof(double) * it, cudaMemcpyDeviceToHost, st));
    BIE_CUDA_TRY(cudaStreamSynchronize(st));
    *res_true = pinned[6] / pinned[7];
    *res_pc = bd ? pinned[5] / beta : *res_true;
    return BIE_OK;
}

extern "C" int bie_gmres_solve(bie_geometry_t gh, bie_blockdiag_t bdh, const double *f, double *x, double tol,
                               int max_iter, double *hist_host, int *iters, double *res_pc, double *res_true,
                               int *converged, void *stream) {
    return gmres_solve_impl("bie_gmres_solve", BIE_FULL, gh, bdh, f, x, tol, max_iter, hist_host, iters, res_pc,
                            res_true, converged, stream);
}

// End-to-end form with HOST buffers: f is copied to the
// geometry's device staging buffer, solved there, and x copied back; the call
// returns after the D2H copy has completed.  Pinned host memory makes both
// copies DMA transfers on `stream`; pageable memory works (driver-staged).
extern "C" int bie_gmres_solve_host(bie_geometry_t gh, bie_blockdiag_t bdh, const double *f_host, double *x_host,
                                    double tol, int max_iter, double *hist_host, int *iters, double *res_pc,
                                    double *res_true, int *converged, void *stream) {
    Geometry *g = as_geom(gh);
    if (!g || !f_host || !x_host || f_host == x_host) {
        set_error("bie_gmres_solve_host: invalid handle, null host buffer or f == x");
        return BIE_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const size_t bytes = sizeof(double) * 2 * (size_t)g->N;
    BIE_CUDA_TRY(cudaMemcpyAsync(g->stage_in, f_host, bytes, cudaMemcpyHostToDevice, st));
    int rc = gmres_solve_impl("bie_gmres_solve_host", BIE_FULL, gh, bdh, g->stage_in, g->stage_out, tol, max_iter,
                              hist_host, iters, res_pc, res_true, converged, stream);
    if (rc) return rc;
    BIE_CUDA_TRY(cudaMemcpyAsync(x_host, g->stage_out, bytes, cudaMemcpyDeviceToHost, st));
    BIE_CUDA_TRY(cudaStreamSynchronize(st));
    return BIE_OK;
}

extern "C" int bie_gmres_solve_slp(bie_geometry_t gh, bie_blockdiag_t bdh, const double *f, double *x, double tol,
                                   int max_iter, double *hist_host, int *iters, double *res_pc, double *res_true,
                                   int *converged, void *stream) {
    return gmres_solve_impl("bie_gmres_solve_slp", kOpSLP, gh, bdh, f, x, tol, max_iter, hist_host, iters, res_pc,
                            res_true, converged, stream);
}

// ---------------------------------------------------------------------------
// NEXT-3: batched multi-RHS GMRES.  Identical per-system algorithm (reading
// C13); the operator applications of all active systems share one nvec-wide
// bie_dlp_apply / bie_blockdiag_apply per iteration (chunks of 16).
// ---------------------------------------------------------------------------
namespace bie {
static int batched_op(Geometry *g, BlockDiag *bd, const double *in, double *tmp, double *out, int nv,
                      cudaStream_t st, unsigned opf) {
    const long long n = 2LL * g->N;
    // Operator: groups of 4 / 8 / 16 vectors through the one-sided multi-vector
    // kernels (11 + 2 + 4 nvec FP64 instructions per pair: 7.25 per vector at
    // nvec = 4), a remainder of 1-3 vectors one at a time through the symmetric
    // kernel (10.5 per vector; the one-sided nvec = 1 / 2 / 3 forms cost 16 / 10.5
    // / 9.7 plus a second launch).  The BD apply takes the whole chunk.
    for (int v0 = 0; v0 < nv; v0 += BIE_MAX_NVEC) {
        const int c = std::min(BIE_MAX_NVEC, nv - v0);
        const int cw = c - c % 4;
        double *dst = bd ? tmp : out;
        if (cw > 0) {
            int rc = dlp_apply_impl(g, in + v0 * n, dst + v0 * n, cw, opf, 0, g->N, st);
            if (rc) return rc;
        }
        for (int v = v0 + cw; v < v0 + c; ++v) {
            int rc = dlp_apply_impl(g, in + v * n, dst + v * n, 1, opf, 0, g->N, st);
            if (rc) return rc;
        }
        if (bd) {
            int rc = blockdiag_apply_impl(bd, tmp + v0 * n, out + v0 * n, c, st);
            if (rc) return rc;
        }
    }
    return BIE_OK;
}
}  // namespace bie

static int gmres_batch_impl(const char *fn, unsigned opf, bie_geometry_t gh, bie_blockdiag_t bdh, const double *F,
                            double *X, int nrhs, double tol, int max_iter, double *hist_host, int *iters,
                            double *res_pc, double *res_true, int *converged, void *stream) {
    Geometry *g = as_geom(gh);
    BlockDiag *bd = bdh ? as_bd(bdh) : nullptr;
    if (!g || (bdh && !bd) || !F || !X || !hist_host || !iters || !res_pc || !res_true || !converged ||
        max_iter < 1 || !(tol > 0.0) || F == X || nrhs < 1 || nrhs > 64) {
        set_error(std::string(fn) + ": invalid handle, null pointer, F == X, nrhs not in [1,64], max_iter < 1 "
                                    "or tol <= 0");
        return BIE_EINVAL;
    }
    if (bd && bd->g != g) {
        set_error(std::string(fn) + ": blockdiag was built from another geometry");
        return BIE_EINVAL;
    }
    if (bd && (bd->b0 != 0 || bd->b1 != g->M + 1)) {
        set_error(std::string(fn) + ": blockdiag covers a body range, not the whole geometry");
        return BIE_EINVAL;
    }
    if (bd && bd->op != ((opf & kOpSLP) ? 1 : 0)) {
        set_error(std::string(fn) + ": blockdiag was factored for the other operator (DLP vs SLP)");
        return BIE_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const long long n = 2LL * g->N;
    const int ldh = max_iter + 1;
    const unsigned eb = (unsigned)((n + 255) / 256);
    Dot d;
    d.nchunks = (int)((n + kChunk - 1) / kChunk);
    d.ldp = ldh;
    int rc = BIE_OK;
    auto cleanup = [&]() {};  // the workspace stays cached on the geometry
#define GB_TRY(expr)                   \
    do {                               \
        cudaError_t _e = (expr);       \
        if (_e != cudaSuccess) {       \
            rc = cuda_fail(_e, #expr); \
            cleanup();                 \
            return rc;                 \
        }                              \
    } while (0)
#define GB_RC(expr)          \
    do {                     \
        rc = (expr);         \
        if (rc != BIE_OK) {  \
            cleanup();       \
            return rc;       \
        }                    \
    } while (0)
    // per-system small state: cs, sn, g, h, h2 [ldh each] + scal [8]
    const long long smallper = 5LL * ldh + 8;
    GmresWork &ws = g->gmb;
    auto ensure = [&](double *&ptr, size_t &cap, size_t need) -> cudaError_t {
        if (need <= cap) return cudaSuccess;
        cudaFree(ptr);  // synchronises the device: no work in flight uses the old buffer
        ptr = nullptr;
        cap = 0;
        cudaError_t e = cudaMalloc(&ptr, sizeof(double) * need);
        if (e == cudaSuccess) cap = need;
        return e;
    };
    GB_TRY(ensure(ws.V, ws.V_cap, (size_t)nrhs * ldh * n));
    GB_TRY(ensure(ws.w, ws.n_cap, 3 * (size_t)nrhs * n));
    GB_TRY(ensure(ws.H, ws.H_cap, (size_t)nrhs * ldh * max_iter));
    GB_TRY(ensure(ws.small, ws.small_cap, (size_t)nrhs * smallper));
    // partials of all active systems + est[2][64] + act[64] (as ints)
    const long long psys = (long long)d.nchunks * ldh;
    GB_TRY(ensure(ws.partial, ws.partial_cap, (size_t)(nrhs * psys + 256)));
    // host lookahead (as bie_gmres_solve's host-enqueued form): iteration k is
    // enqueued before the estimates of iteration k - kLookB are read; each of the
    // kRingB in-flight iterations has its own active list / estimate slots
    constexpr int kLookB = 3, kRingB = kLookB + 1;
    GB_TRY(ensure(ws.partial, ws.partial_cap, (size_t)(nrhs * psys + kRingB * 192)));
    // pinned: 64 x 8 per-system scalars + kRingB x (est [128] + act [64 ints])
    if (!ws.pinned) GB_TRY(cudaMallocHost(&ws.pinned, sizeof(double) * (512 + kRingB * 192)));
    for (int q = 0; q < kRingB; ++q)
        if (!ws.evs[q]) GB_TRY(cudaEventCreateWithFlags(&ws.evs[q], cudaEventDisableTiming));
    double *V = ws.V, *Win = ws.w, *Wt = ws.w + (size_t)nrhs * n, *Wout = ws.w + 2 * (size_t)nrhs * n;
    double *H = ws.H, *small = ws.small, *pinned = ws.pinned;
    d.partial = ws.partial;
    auto d_est_slot = [&](int q) { return ws.partial + nrhs * psys + (long long)q * 192; };
    auto d_act_slot = [&](int q) { return reinterpret_cast<int *>(d_est_slot(q) + 128); };
    auto h_est_slot = [&](int q) { return pinned + 512 + (long long)q * 192; };
    auto h_act_slot = [&](int q) { return reinterpret_cast<int *>(h_est_slot(q) + 128); };
    const long long sysV = (long long)ldh * n, Hsys = (long long)ldh * max_iter, scal_off = 5LL * ldh;
    GB_TRY(cudaMemsetAsync(H, 0, sizeof(double) * (size_t)nrhs * ldh * max_iter, st));
    GB_TRY(cudaMemsetAsync(small, 0, sizeof(double) * (size_t)nrhs * smallper, st));
    std::vector<GmState> S(nrhs);
    for (int r = 0; r < nrhs; ++r) {
        double *b = small + r * smallper;
        S[r] = GmState{H + (size_t)r * ldh * max_iter, b, b + ldh, b + 2 * ldh, b + 3 * ldh, b + 4 * ldh, b + 5 * ldh};
    }
    auto Vr = [&](int r, int k) { return V + ((size_t)r * ldh + k) * n; };
    auto norm_to = [&](const double *v, double *tmp, double *dst) -> int {
        (void)tmp;
        return multidot(v, 0, 1, v, n, d, dst, st, nullptr, 1);
    };
    // r0 = P^{-1} f for all systems at once
    if (bd) {
        for (int v0 = 0; v0 < nrhs; v0 += BIE_MAX_NVEC)
            GB_RC(blockdiag_apply_impl(bd, F + v0 * n, Wout + v0 * n, std::min(BIE_MAX_NVEC, nrhs - v0), st));
    } else {
        GB_TRY(cudaMemcpyAsync(Wout, F, sizeof(double) * (size_t)nrhs * n, cudaMemcpyDeviceToDevice, st));
    }
    for (int r = 0; r < nrhs; ++r) GB_RC(norm_to(Wout + r * n, S[r].scal + 5, S[r].scal + 0));
    for (int r = 0; r < nrhs; ++r)
        GB_TRY(cudaMemcpyAsync(pinned + 8 * r, S[r].scal, sizeof(double), cudaMemcpyDeviceToHost, st));
    GB_TRY(cudaStreamSynchronize(st));
    GB_TRY(cudaMemsetAsync(X, 0, sizeof(double) * (size_t)nrhs * n, st));
    std::vector<double> beta(nrhs);
    std::vector<int> it(nrhs, 0), active;
    for (int r = 0; r < nrhs; ++r) {
        beta[r] = pinned[8 * r];
        hist_host[(size_t)r * ldh] = 1.0;
        converged[r] = 0;
        iters[r] = 0;
        res_pc[r] = res_true[r] = 0.0;
        if (beta[r] == 0.0) {
            converged[r] = 1;
            continue;
        }
        active.push_back(r);
        k_scale_div<<<eb, 256, 0, st>>>(Wout + r * n, S[r].scal + 0, Vr(r, 0), n);
        count_launch();
        GB_TRY(cudaMemcpyAsync(S[r].g, S[r].scal + 0, sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    // Iteration: every vector operation of all active systems in one batched
    // launch (blockIdx.z / y = slot), one D2H of the estimates.  The host reads
    // iteration k's estimates after iteration k + kLookB is enqueued; a system
    // found converged then has run up to kLookB speculative iterations, which
    // touch only its entries beyond the ones its finish reads (as in the single
    // solve), and leaves the active set from the next enqueued iteration on.
    std::vector<std::vector<int>> ring_act(kRingB);
    int processed = 0;  // iterations whose estimates have been read
    auto process = [&](int kk) -> int {
        const int sl = kk % kRingB;
        GB_TRY(cudaEventSynchronize(ws.evs[sl]));
        const double *he = h_est_slot(sl);
        std::vector<int> keep;
        for (size_t q = 0; q < ring_act[sl].size(); ++q) {
            const int r = ring_act[sl][q];
            if (converged[r]) continue;  // detected at an earlier iteration: speculative entry
            const double est = he[2 * q];
            const bool brk = he[2 * q + 1] != 0.0;
            hist_host[(size_t)r * ldh + kk + 1] = est;
            it[r] = kk + 1;
            if (est < tol || brk) converged[r] = 1;
        }
        for (int r : active)
            if (!converged[r]) keep.push_back(r);
        active.swap(keep);
        processed = kk + 1;
        return BIE_OK;
    };
    int k = 0;
    for (; k < max_iter && !active.empty(); ++k) {
        const int sl = k % kRingB;
        ring_act[sl] = active;
        const int na = (int)active.size();
        int *h_act = h_act_slot(sl), *d_act = d_act_slot(sl);
        double *d_est = d_est_slot(sl);
        for (int q = 0; q < na; ++q) h_act[q] = active[q];
        GB_TRY(cudaMemcpyAsync(d_act, h_act, sizeof(int) * na, cudaMemcpyHostToDevice, st));
        k_gather_b<<<dim3(eb, na), 256, 0, st>>>(V, sysV, (long long)k * n, Win, n, d_act);
        count_launch();
        GB_RC(batched_op(g, bd, Win, Wt, Wout, na, st, opf));
        const int nv = k + 1;
        const unsigned gy = (unsigned)((nv + kDotThreads / 32 - 1) / (kDotThreads / 32));
        // w0 = ||w||
        k_multidot_b<<<dim3(d.nchunks, 1, na), kDotThreads, 0, st>>>(nullptr, 0, 0, 1, Wout, n, d.partial, d.ldp,
                                                                      psys, d_act, 1);
        k_reduce_b<<<dim3(1, na), 128, 0, st>>>(d.partial, d.ldp, psys, d.nchunks, 1, small, smallper, scal_off + 1,
                                                d_act, 1);
        // CGS2: two passes h = V^T w, w -= V h
        for (int pass = 0; pass < 2; ++pass) {
            const long long hoff = (3LL + pass) * ldh;
            k_multidot_b<<<dim3(d.nchunks, gy, na), kDotThreads, 0, st>>>(V, sysV, n, nv, Wout, n, d.partial, d.ldp,
                                                                           psys, d_act, 0);
            k_reduce_b<<<dim3((nv + 127) / 128, na), 128, 0, st>>>(d.partial, d.ldp, psys, d.nchunks, nv, small,
                                                                   smallper, hoff, d_act, 0);
            k_multiaxpy_b<<<dim3(eb, na), 256, 0, st>>>(V, sysV, n, nv, small, smallper, hoff, -1.0,
                                                                          1.0, Wout, n, d_act);
        }
        // hk1 = ||w||
        k_multidot_b<<<dim3(d.nchunks, 1, na), kDotThreads, 0, st>>>(nullptr, 0, 0, 1, Wout, n, d.partial, d.ldp,
                                                                      psys, d_act, 1);
        k_reduce_b<<<dim3(1, na), 128, 0, st>>>(d.partial, d.ldp, psys, d.nchunks, 1, small, smallper, scal_off + 2,
                                                d_act, 1);
        k_givens_b<<<(na + 63) / 64, 64, 0, st>>>(H, Hsys, small, smallper, ldh, k, d_act, na, d_est);
        count_launch(11);
        GB_TRY(cudaMemcpyAsync(h_est_slot(sl), d_est, sizeof(double) * 2 * na, cudaMemcpyDeviceToHost, st));
        if (k + 1 < max_iter) {
            k_scale_b<<<dim3(eb, na), 256, 0, st>>>(Wout, n, V, sysV, (long long)(k + 1) * n, small, smallper,
                                                     scal_off, d_act);
            count_launch();
        }
        GB_TRY(cudaGetLastError());
        GB_TRY(cudaEventRecord(ws.evs[sl], st));
        if (k >= kLookB) GB_RC(process(k - kLookB));
    }
    while (processed < k) GB_RC(process(processed));  // the iterations still in flight
    // finish: y = H^{-1} g, x = V y per system; residual pair with batched operators
    for (int r = 0; r < nrhs; ++r) {
        iters[r] = it[r];
        if (it[r] == 0) continue;
        k_trisolve<<<1, 256, 0, st>>>(S[r].H, ldh, S[r].g, S[r].h, it[r]);
        count_launch();
        GB_RC(multiaxpy(Vr(r, 0), n, it[r], S[r].h, 1.0, 0.0, X + r * n, n, st));
    }
    for (int v0 = 0; v0 < nrhs; v0 += BIE_MAX_NVEC)
        GB_RC(dlp_apply_impl(g, X + v0 * n, Wt + v0 * n, std::min(BIE_MAX_NVEC, nrhs - v0), opf, 0, g->N, st));
    for (int r = 0; r < nrhs; ++r) {
        k_sub<<<eb, 256, 0, st>>>(F + r * n, Wt + r * n, Win + r * n, n);
        count_launch();
    }
    if (bd)
        for (int v0 = 0; v0 < nrhs; v0 += BIE_MAX_NVEC)
            GB_RC(blockdiag_apply_impl(bd, Win + v0 * n, Wout + v0 * n, std::min(BIE_MAX_NVEC, nrhs - v0), st));
    for (int r = 0; r < nrhs; ++r) {
        GB_RC(norm_to(Win + r * n, S[r].scal + 5, S[r].scal + 6));
        GB_RC(norm_to(F + r * n, S[r].scal + 5, S[r].scal + 7));
        if (bd) GB_RC(norm_to(Wout + r * n, S[r].scal + 4, S[r].scal + 5));
        GB_TRY(cudaMemcpyAsync(pinned + 8 * r + 5, S[r].scal + 5, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
    }
    GB_TRY(cudaStreamSynchronize(st));
    for (int r = 0; r < nrhs; ++r) {
        if (beta[r] == 0.0) continue;
        res_true[r] = pinned[8 * r + 6] / pinned[8 * r + 7];
        res_pc[r] = bd ? pinned[8 * r + 5] / beta[r] : res_true[r];
    }
#undef GB_TRY
#undef GB_RC
    cleanup();
    return BIE_OK;
}

extern "C" int bie_gmres_solve_batch(bie_geometry_t gh, bie_blockdiag_t bdh, const double *F, double *X, int nrhs,
                                     double tol, int max_iter, double *hist_host, int *iters, double *res_pc,
                                     double *res_true, int *converged, void *stream) {
    return gmres_batch_impl("bie_gmres_solve_batch", BIE_FULL, gh, bdh, F, X, nrhs, tol, max_iter, hist_host, iters,
                            res_pc, res_true, converged, stream);
}

extern "C" int bie_gmres_solve_batch_slp(bie_geometry_t gh, bie_blockdiag_t bdh, const double *F, double *X,
                                         int nrhs, double tol, int max_iter, double *hist_host, int *iters,
                                         double *res_pc, double *res_true, int *converged, void *stream) {
    return gmres_batch_impl("bie_gmres_solve_batch_slp", kOpSLP, gh, bdh, F, X, nrhs, tol, max_iter, hist_host,
                            iters, res_pc, res_true, converged, stream);
}

BIE_DCHECK_TU(gmres)
