// dlp.cu -- the completed double-layer matvec (A2-A5 of SURVEY.md s8(a)) and
// the paper's single-layer operator with the Kapur-Rokhlin correction (NEXT-1).
//
//   k_moments   (A2)  per-pore lambda_k, mu_k and the wall scalar nu     O(N)
//   k_dlp_sym   (A3)  symmetric all-pairs sum, nvec = 1 (each unordered
//                     pair once, dynamic segments)                       O(N^2)  <- hot
//   k_dlp_diag  (A3)  pairs inside a 512-node block (one-sided)         O(512 N)
//   k_dlp_pairs (A3)  one-sided all-pairs sum: nvec > 1, row ranges,
//                     field targets                                      O(N^2)
//   k_epilogue  (A4+A5) fixed-order partial sums, -1/2 sigma, self term, N0,
//                       Stokeslet/rotlet completion (SLP: KR correction) O(N M)
// Every pair kernel takes OP = 0 (completed DLP) or OP = 1 (SLP); all sums are
// in a fixed order, so results are bitwise repeatable.
//
// Operator (P:l.243-248 with trapezoid weights P:l.310-319; readings C3-C5):
//   y_i = -1/2 s_i + sum_{j != i} (r.nw_j)(r.s_j) r / rho^4 + selfc_i (t_i.s_i) t_i
//         + [i in Gamma_0] nu n_i + sum_k S(x_i - c_k) lambda_k + r_k R(x_i - c_k) mu_k
//   nw_j = w_j n_j / pi,  r = x_i - x_j,  selfc_i = w_i kappa_n,i / (2 pi).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <string>
#include <type_traits>

#include "internal.cuh"

namespace bie {

constexpr int kPairThreads = 128;

// Pair-kernel variants: vectors per launch, targets per thread, sources per tile.
struct Variant {
    int nv, R, TS;
};
static const Variant kVariants[5] = {{1, 4, 256}, {2, 2, 256}, {4, 4, 256}, {8, 1, 128}, {16, 1, 64}};

__device__ __forceinline__ double rcp_approx(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    return r;
}

// Branch-free log for the pair loops (the library log() carries special-case
// branches that keep ptxas from interleaving independent pairs): a Tang-style
// table reduction.  d = 2^e m, m in [1, 2); k = top 8 mantissa bits;
// tab[k] = (rc_k, 1/2 log rc_k) with rc_k = RN(1 / (1 + (k + 1/2)/256)).
// r = m rc_k - 1 (one FMA, |r| < 2^-9), log m = log1p(r) - log rc_k with
// log1p(r) = r (1 - r/2 + ... + r^4/5) (truncation r^6/6 < 2^-56.6, below the
// rounding of e ln2 + 1/2 log rc_k; offline check against 40-digit logs: the
// same worst-case error as round 1's form).  Returns hl = -1/2 log d directly
// (scaled coefficients): 7 FP64 instructions, one shared-memory lookup and an
// I2F.F64 for the exponent.  (Round 1: 64 entries and a degree-7 series, 9
// instructions; the 256-entry table saves two FMAs per pair in every SLP pair
// loop and completion field.)  With EX the
// exponent comes as a double from a second table indexed by the biased exponent
// bits (an LDS instead of the I2F, which occupies the FP64 pipe; 16 KiB more
// shared memory, worth it in the symmetric SLP kernel, but not in the one-sided
// kernels, where it costs occupancy).  Both forms give bit-identical results.
// d must be positive and normal (pair distances are).
template <bool EX>
struct LogTabT {
    double2 e[256];
    double ex[EX ? 2048 : 1];  // b - 1023 for biased exponent b
};
using LogTab = LogTabT<false>;
using LogTabX = LogTabT<true>;
template <bool EX>
__device__ __forceinline__ void log_tab_init(LogTabT<EX> &t, int tid, int nthreads) {
    for (int k = tid; k < 256; k += nthreads) {
        const double rc = 1.0 / (1.0 + (k + 0.5) / 256.0);
        t.e[k] = make_double2(rc, 0.5 * log(rc));  // -1/2 log(1/rc) = 1/2 log rc
    }
    if constexpr (EX)
        for (int k = tid; k < 2048; k += nthreads) t.ex[k] = (double)(k - 1023);
}
template <bool EX>
__device__ __forceinline__ double neg_half_log_tab(double d, const LogTabT<EX> &t) {
    const int hi = __double2hiint(d), lo = __double2loint(d);
    // (hi & 0x000fffff) | 0x3ff00000 as one LOP3 (the constant in a register)
    int mhi;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(mhi) : "r"(hi), "r"(0x000fffff), "r"(0x3ff00000));
    const double m = __hiloint2double(mhi, lo);
    const double2 tk = t.e[(hi >> 12) & 255];
    const double r = fma(m, tk.x, -1.0);
    double q = -0.5 / 5.0;  // -1/2 (1 - r/2 + r^2/3 - r^3/4 + r^4/5); the r^5 term is < 2^-56.6
    q = fma(q, r, 0.5 / 4.0);
    q = fma(q, r, -0.5 / 3.0);
    q = fma(q, r, 0.5 / 2.0);
    q = fma(q, r, -0.5);
    // e ln2 with ln2 rounded to double: the error |e| 2.3e-17 stays below half an
    // ulp of e ln2 itself for every exponent a pair distance can have
    // d > 0: hi >> 20 is the biased exponent (no sign bit to mask)
    const double e = EX ? t.ex[hi >> 20] : (double)((hi >> 20) - 1023);
    const double base = fma(e, -0.5 * 0.69314718055994528623, tk.y);
    return fma(r, q, base);
}

// Single-layer pair factor (NEXT-1; P:l.270-276): for r = x_i - x_j returns
// hl = -1/2 log rho^2 and inv = 1/rho^2, so that
//   G(x_i, x_j) (w_j sigma_j) = hl S_j + (r . S_j) inv r,   S_j = w_j sigma_j / (4 pi).
// r = 0 (the self pair, or zero-padded slots that coincide) maps rho^2 -> 1:
// hl = 0 and the dyadic term vanishes with r, so no branch is needed.
__device__ __forceinline__ void slp_factors(double rx, double ry, double &hl, double &inv, const LogTab &lt) {
    double d = fma(rx, rx, ry * ry);
    d = d == 0.0 ? 1.0 : d;
    double i = rcp_approx(d);
    const double e = fma(-d, i, 1.0);
    inv = fma(i, fma(e, e, e), i);
    hl = neg_half_log_tab(d, lt);
}

__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gmem_src, int src_bytes) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem_src), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// CTA that owns work unit u under the static partition u0(p) = floor(p U / P).
__host__ __device__ __forceinline__ int unit_owner(long long u, long long U, int P) {
    return (int)(((u + 1) * (long long)P - 1) / U);
}

// Segment of unit u in a unit list (or slice) starting at ub.  Both all-pairs
// kernels hand out fixed segments of Useg units through an atomic counter; a
// target block's partial for segment s goes to slot s - seg_of(first unit of
// the block), so the sums do not depend on which CTA ran which segment.
__host__ __device__ __forceinline__ long long seg_of(long long u, long long ub, long long Useg) {
    return (u - ub) / Useg;
}

struct PairArgs {
    const double2 *tpos;  // [Nt] target positions (pos + row_begin, or off-surface points)
    const double2 *pos;   // [N] source positions
    const double2 *nw;    // [N] w n / pi
    const double *sigma;  // first vector of this chunk; vector v at sigma + v * sig_stride
    long long sig_stride; // 2N
    double *partial;      // [S][nvec_total][2 Nt]
    int nvec_total, v0;   // total vectors of the call, first vector of this chunk
    int N, row_begin, Nt; // sources, first target, number of targets
    int nTS;
    long long U;
    long long Useg, nseg;          // dynamic segments (see seg_of)
    unsigned long long *counter;   // zeroed before the launch
    long long partial_len = 0;     // doubles in partial (checked build: BIE_DCHECK on stores)
};

// A3: all-pairs DLP sum.  Each persistent CTA walks a contiguous range of
// (target block, source tile) units; sources are staged in shared memory by
// cp.async double buffering and read as warp-broadcast LDS.128; each thread
// keeps R targets and their NV accumulators in registers.  The self pair
// (r = 0) needs no branch: rho^2 gets +1e-300 (below one ulp of any real
// pair distance), so 1/rho^2 stays finite and r.nw = 0 zeroes the term.
// 1/rho^2: MUFU.RCP64H seed + one cubic Newton step (3 DFMA, rel. err ~2^-60).
// OP = 1: the single-layer operator instead (NEXT-1).  sigma then holds the
// pre-scaled S_j = w_j sigma_j / (4 pi) and nw is unused.
template <int NV, int R, int TS, int OP = 0, int MINB = 1>
__global__ void __launch_bounds__(kPairThreads, MINB) k_dlp_pairs(PairArgs a) {
    extern __shared__ double2 smem[];  // [2][(2 + NV) * TS]
    constexpr int NT = kPairThreads;
    constexpr int TB = NT * R;
    constexpr int STAGE = (2 + NV) * TS;
    static_assert(STAGE % NT == 0, "stage must be a multiple of the CTA size");
    const int tid = threadIdx.x;
    const long long U = a.U, Useg = a.Useg;
    const int N = a.N, nTS = a.nTS;
    __shared__ long long s_seg;
    __shared__ LogTab s_log;  // OP = 1 only; visible after the first segment barrier
    if constexpr (OP == 1) log_tab_init(s_log, tid, kPairThreads);

    auto load_tile = [&](int buf, int ts) {
        double2 *s = smem + buf * STAGE;
        const int j0 = ts * TS;
#pragma unroll
        for (int q0 = 0; q0 < STAGE; q0 += NT) {
            const int q = q0 + tid;
            const int arr = q / TS;
            const int j = j0 + (q - arr * TS);
            const bool ok = j < N;
            const double2 *src;
            if (arr == 0)
                src = a.pos + (ok ? j : 0);
            else if (arr == 1)
                src = a.nw + (ok ? j : 0);
            else
                src = reinterpret_cast<const double2 *>(a.sigma + (long long)(arr - 2) * a.sig_stride) + (ok ? j : 0);
            cp_async16(s + q, src, ok ? 16 : 0);
        }
        cp_async_commit();
    };

    double tx[R], ty[R];
    double2 acc[R][NV];
    auto load_targets = [&](int tb) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            int it = tb * TB + r * NT + tid;
            double2 x = make_double2(0.0, 0.0);
            if (it < a.Nt) x = a.tpos[it];
            tx[r] = x.x;
            ty[r] = x.y;
#pragma unroll
            for (int v = 0; v < NV; ++v) acc[r][v] = make_double2(0.0, 0.0);
        }
    };

    for (;;) {  // claim segments of Useg units (see seg_of)
    if (tid == 0) s_seg = (long long)atomicAdd(a.counter, 1ULL);
    __syncthreads();
    const long long sg = s_seg;
    __syncthreads();
    if (sg >= a.nseg) break;
    const long long u0 = sg * Useg, u1 = min(u0 + Useg, U);
    long long u = u0;
    int tb = (int)(u / nTS);
    load_targets(tb);
    load_tile(0, (int)(u % nTS));
    int buf = 0;
    for (; u < u1; ++u) {
        if (u + 1 < u1)
            load_tile(buf ^ 1, (int)((u + 1) % nTS));
        else
            cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        const double2 *sp = smem + buf * STAGE;
#pragma unroll 2
        for (int j = 0; j < TS; ++j) {
            const double2 xj = sp[j];
            const double2 nj = sp[TS + j];
            double2 sj[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) sj[v] = sp[(2 + v) * TS + j];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if constexpr (OP == 1) {
                    const double rx = tx[r] - xj.x;
                    const double ry = ty[r] - xj.y;
                    double hl, inv;
                    slp_factors(rx, ry, hl, inv, s_log);
                    if constexpr (NV >= 2) {
                        // r / rho^2 once per pair: 6 FP64 instructions per vector instead of 7
                        const double ix = inv * rx, iy = inv * ry;
#pragma unroll
                        for (int v = 0; v < NV; ++v) {
                            const double rs = fma(rx, sj[v].x, ry * sj[v].y);
                            acc[r][v].x = fma(rs, ix, fma(hl, sj[v].x, acc[r][v].x));
                            acc[r][v].y = fma(rs, iy, fma(hl, sj[v].y, acc[r][v].y));
                        }
                    } else {
#pragma unroll
                        for (int v = 0; v < NV; ++v) {
                            const double c = inv * fma(rx, sj[v].x, ry * sj[v].y);
                            acc[r][v].x = fma(c, rx, fma(hl, sj[v].x, acc[r][v].x));
                            acc[r][v].y = fma(c, ry, fma(hl, sj[v].y, acc[r][v].y));
                        }
                    }
                    continue;
                }
                const double rx = tx[r] - xj.x;
                const double ry = ty[r] - xj.y;
                const double rho2 = fma(rx, rx, fma(ry, ry, 1e-300));
                const double rn = fma(rx, nj.x, ry * nj.y);
                double inv = rcp_approx(rho2);
                const double e = fma(-rho2, inv, 1.0);
                inv = fma(inv, fma(e, e, e), inv);
                const double q = (rn * inv) * inv;  // (r.nw)/rho^4
                if constexpr (NV >= 2) {
                    // g = q r once per pair (2 DMUL), then (r.sigma) g: 4 FP64
                    // instructions per vector (11 + 2 + 4 nvec per pair; the round-1
                    // forms took 11 + 5 nvec, or 16 + 4 nvec with P = q r r^T)
                    const double gx = q * rx, gy = q * ry;
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        const double rs = fma(rx, sj[v].x, ry * sj[v].y);
                        acc[r][v].x = fma(rs, gx, acc[r][v].x);
                        acc[r][v].y = fma(rs, gy, acc[r][v].y);
                    }
                } else {
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        const double c = q * fma(rx, sj[v].x, ry * sj[v].y);
                        acc[r][v].x = fma(c, rx, acc[r][v].x);
                        acc[r][v].y = fma(c, ry, acc[r][v].y);
                    }
                }
            }
        }
        __syncthreads();
        buf ^= 1;
        const bool seg_end = (u + 1 == u1) || ((u + 1) % nTS == 0);
        if (seg_end) {
            const int slot = (int)(sg - seg_of((long long)tb * nTS, 0, Useg));
#pragma unroll
            for (int r = 0; r < R; ++r) {
                int it = tb * TB + r * NT + tid;
                if (it < a.Nt) {
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        const long long o = ((long long)slot * a.nvec_total + a.v0 + v) * 2LL * a.Nt;
                        BIE_DCHECK(slot >= 0 && o + 2LL * it + 1 < a.partial_len);
                        double2 *dst = reinterpret_cast<double2 *>(a.partial + o);
                        dst[it] = acc[r][v];
                    }
                }
            }
            if (u + 1 < u1) {
                tb = (int)((u + 1) / nTS);
                load_targets(tb);
            }
        }
    }
    }  // segments
}

// A2: moments (reading C5).  Block b < M: pore b; block M: Gamma_0.
// Deterministic fixed-shape tree reduction.
__global__ void k_moments(const double2 *__restrict__ pos, const double2 *__restrict__ nrm,
                          const double *__restrict__ w, const double4 *__restrict__ pore, const double *sigma,
                          long long sig_stride, int nvec, int M, int n_pore, int wall_lo, int N, double wall_len,
                          double *moments /* [nvec][M][3], then [nvec] nu */) {
    pdl_wait();
    __shared__ double red[3][256];
    const int b = blockIdx.x, tid = threadIdx.x;
    for (int v = 0; v < nvec; ++v) {
        const double2 *s = reinterpret_cast<const double2 *>(sigma + (long long)v * sig_stride);
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        if (b < M) {
            double4 pk = pore[b];
            for (int j = b * n_pore + tid; j < (b + 1) * n_pore; j += blockDim.x) {
                double2 sj = s[j], xj = pos[j];
                double px = xj.y - pk.y, py = -(xj.x - pk.x);  // (x - c)^perp
                a0 += w[j] * sj.x;
                a1 += w[j] * sj.y;
                a2 += w[j] * (sj.x * px + sj.y * py);
            }
        } else {
            for (int j = wall_lo + tid; j < N; j += blockDim.x) {
                double2 sj = s[j], nj = nrm[j];
                a0 += w[j] * (nj.x * sj.x + nj.y * sj.y);
            }
        }
        red[0][tid] = a0;
        red[1][tid] = a1;
        red[2][tid] = a2;
        __syncthreads();
        for (int h = blockDim.x / 2; h > 0; h >>= 1) {
            if (tid < h) {
                red[0][tid] += red[0][tid + h];
                red[1][tid] += red[1][tid + h];
                red[2][tid] += red[2][tid + h];
            }
            __syncthreads();
        }
        if (tid == 0) {
            if (b < M) {
                double4 pk = pore[b];
                double *m = moments + ((long long)v * M + b) * 3;
                m[0] = red[0][0] / pk.w;
                m[1] = red[1][0] / pk.w;
                m[2] = red[2][0] / (pk.w * pk.z);
            } else {
                moments[(long long)nvec * M * 3 + v] = red[0][0] / wall_len;
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Symmetric all-pairs path (nvec = 1, full rows).  Pair (i, j) and (j, i) share
// r (up to sign), rho^2 and 1/rho^4.  With per-node quadratic forms
//   Q_j = (nwx sx, nwx sy + nwy sx, nwy sy)   (nw = w n / pi, s = sigma)
// (r.nw_j)(r.s_j) = Qxx rx^2 + Qxy rx ry + Qyy ry^2, so
//   u_i += Q_j(r) r / rho^4      and      u_j -= Q_i(r) r / rho^4.
// Each unordered pair is evaluated once: 21 FP64 instructions for both
// directions (10.5 per directed pair vs 16; see k_quad for the Q' form).  Blocks of TB = 512 nodes; block A
// pairs with every 32-node chunk after its end ("units"), handled by a
// persistent grid over the triangular unit list.  Inside a warp the 32-source
// chunk rotates through the lanes (__shfl) together with its accumulator, so
// each source collects the contributions of the warp's 128 targets without a
// reduction; the 4 warps' source sums are added in fixed order through shared
// memory and stored as src_partial[A][j].  Target accumulators are flushed per
// CTA segment (slot = CTA - first owner).  Pairs inside a block (A, A) are
// done by k_dlp_diag with the one-sided kernel.  All sums have a fixed order.
// ---------------------------------------------------------------------------
constexpr int kSymR = 4;
constexpr int kSymWarps = 4;
constexpr int kSymTB = 32 * kSymR * kSymWarps;  // 512
constexpr int kSymChunk = 32;

// ---------------------------------------------------------------------------
// Order-independent exact accumulation (symmetric path).  A pair-sum
// contribution v (one unit's 512-target sum for a source, or one segment's
// sum for a target) is scaled by 2^-E (E = exponent of max |Q|, so the window
// follows the data) and split exactly into three integer limbs
//   v 2^-E = x2 + x1 2^-32 + x0 2^-64 - t,  x2 = floor, x1, x0 in [0, 2^32),
// (truncation t < 2^-64), each added with a 64-bit integer RED to its own
// accumulator.  Integer addition is associative, so the totals -- and the
// double the epilogue forms from them -- do not depend on which CTA added
// what when: bitwise deterministic results with O(N) memory (3 x 2N words)
// and no ordering waits.  The round-1 form kept one FP64 partial per
// (512-node block, node): N x nTB doubles, 35 GB at config 5.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void fx_add(unsigned long long *acc, long long limb_stride, double v) {
    const double f2 = floor(v);
    const double t1 = (v - f2) * 4294967296.0;  // both steps exact
    const double f1 = floor(t1);
    const double f0 = floor((t1 - f1) * 4294967296.0);
    atomicAdd(acc, (unsigned long long)(long long)f2);
    atomicAdd(acc + limb_stride, (unsigned long long)f1);
    atomicAdd(acc + 2 * limb_stride, (unsigned long long)f0);
}
// sum of the three limb totals (carry-normalised, exact) as a double, times 2^E
__device__ __forceinline__ double fx_value(const unsigned long long *acc, long long limb_stride, double scale_back) {
    unsigned long long x2 = acc[0], x1 = acc[limb_stride], x0 = acc[2 * limb_stride];
    x1 += x0 >> 32;
    x0 &= 0xffffffffull;
    x2 += x1 >> 32;
    x1 &= 0xffffffffull;
    const double frac = __ull2double_rn((x1 << 32) | x0) * 0x1p-64;
    return ((double)(long long)x2 + frac) * scale_back;
}
// 2^-E and 2^E for the accumulation window (E = exponent of max |Q|, 0 if Q = 0)
__device__ __forceinline__ void fx_scales(const unsigned long long *qmax_bits, double &scale, double &scale_back) {
    const double qm = __longlong_as_double((long long)*qmax_bits);
    const int E = qm > 0.0 ? ilogb(qm) : 0;
    scale = ldexp(1.0, -E);
    scale_back = ldexp(1.0, E);
}
__device__ __forceinline__ void qmax_update(double m, unsigned long long *qmax_bits) {
    // m >= 0: IEEE order of non-negative doubles is their integer order
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(qmax_bits, (unsigned long long)__double_as_longlong(m));
}

// node j's three limb pairs of the symmetric kernel's accumulators (zeroed
// here, in the O(N) kernel that precedes every symmetric launch, instead of a
// separate memset per apply)
__device__ __forceinline__ void zero_limbs(unsigned long long *acc, int j, int N) {
#pragma unroll
    for (int q = 0; q < 3; ++q)
        reinterpret_cast<ulonglong2 *>(acc + 2LL * N * q)[j] = make_ulonglong2(0ull, 0ull);
}

__global__ void k_quad(const double2 *__restrict__ nw, const double *__restrict__ sigma, double4 *Q, int N,
                       unsigned long long *qmax_bits, unsigned long long *acc) {
    pdl_wait();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    double m = 0.0;
    if (j < N) zero_limbs(acc, j, N);
    if (j < N) {
        const double2 a = nw[j];
        const double2 b = reinterpret_cast<const double2 *>(sigma)[j];
        // (Qxx, Qxy, Qyy - Qxx): with d = rx^2 + ry^2,
        //   Qxx rx^2 + Qxy rx ry + Qyy ry^2 = Qxx d + Qxy rx ry + (Qyy - Qxx) ry^2,
        // so the pair loop never forms rx^2 (21 instead of 22 FP64 instructions)
        const double qxx = a.x * b.x;
        const double4 q = make_double4(qxx, fma(a.x, b.y, a.y * b.x), fma(a.y, b.y, -qxx), 0.0);
        Q[j] = q;
        m = fmax(fabs(q.x), fmax(fabs(q.y), fabs(q.z)));
    }
    qmax_update(m, qmax_bits);
}

// One unordered pair (target t, source s) of the symmetric kernels: the target
// accumulates the source's contribution and vice versa (DLP: odd in r, so the
// source side takes -b; SLP: even in r).
__device__ __forceinline__ void dlp_pairpair(double tx, double ty, double tqa, double tqb, double tqc, double sx,
                                             double sy, double sqa, double sqb, double sqc, double &ax, double &ay,
                                             double &bx, double &by) {
    const double rx = tx - sx, ry = ty - sy;
    // + 1e-150: below one ulp of any real pair distance^2, and keeps
    // q = 1/d^2 <= 1e300 finite for coincident points (zero padding at a target
    // that sits at the origin: cs q then stays finite and r = 0 zeroes it)
    const double yy = fma(ry, ry, 1e-150), xy = rx * ry;
    const double d = fma(rx, rx, yy);
    double i = rcp_approx(d);
    const double cs = fma(sqa, d, fma(sqb, xy, sqc * yy));  // target <- source (Q' form, k_quad)
    const double ct = fma(tqa, d, fma(tqb, xy, tqc * yy));  // source <- target
    const double e = fma(-d, i, 1.0);
    i = fma(i, fma(e, e, e), i);
    const double q = i * i;
    const double a = cs * q, b = ct * q;
    ax = fma(a, rx, ax);
    ay = fma(a, ry, ay);
    bx = fma(-b, rx, bx);
    by = fma(-b, ry, by);
}

__device__ __forceinline__ void slp_pairpair(double tx, double ty, double tsx, double tsy, double sx, double sy,
                                             double ssx, double ssy, double &ax, double &ay, double &bx,
                                             double &by, const LogTabX &lt) {
    const double rx = tx - sx, ry = ty - sy;
    // no self pairs here; coincident zero padding gets d = 1e-300 (finite hl and
    // 1/rho^2, multiplied by a zero density and r = 0)
    const double d = fma(rx, rx, fma(ry, ry, 1e-300));
    double i = rcp_approx(d);
    const double ee = fma(-d, i, 1.0);
    i = fma(i, fma(ee, ee, ee), i);
    const double hl = neg_half_log_tab(d, lt);
    const double ct = i * fma(rx, ssx, ry * ssy), cs = i * fma(rx, tsx, ry * tsy);
    ax = fma(ct, rx, fma(hl, ssx, ax));
    ay = fma(ct, ry, fma(hl, ssy, ay));
    bx = fma(cs, rx, fma(hl, tsx, bx));
    by = fma(cs, ry, fma(hl, tsy, by));
}

struct SymArgs {
    const double2 *pos;
    const double4 *Q;
    const long long *off;  // [nTB + 1] prefix of units per block
    unsigned long long *acc;        // [3][2N] fixed-point limbs of the pair sums (fx_add; zeroed per launch)
    const unsigned long long *qmax; // max |Q| (bits) from k_quad / k_slp_scale: accumulation window
    int N, nTB;
    long long U;           // units in this launch's slice [ub, ub + U) of the triangular list
    long long ub;          // 0 for the single-GPU matvec; a rank's slice start when sharded
    unsigned long long *trace;  // optional [P][2] CTA start/end %globaltimer (BIE_SYM_TRACE diagnostics)
    long long Useg;        // units per segment (dynamic work distribution)
    long long nseg;        // segments in the slice
    unsigned long long *counter;  // next free segment (zeroed before each launch)
};

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ double shfl_d(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }

// A3, nvec = 1: symmetric all-pairs kernel.  SR targets per lane, SW warps
// (SR SW 32 = 512-node blocks), NS sources per step: at step t lane l pairs
// each of its targets with sources (l + t + k 32/NS) mod 32, k < NS, so every
// step carries SR x NS independent pair chains and NS rotating source
// accumulators (NS = 2 is the round-1 "dual-source" form).
// Both sides flush into the fixed-point limb accumulators (fx_add): a unit's
// 32 source sums (added over the warps in fixed order) at the unit's end, the
// targets' register sums at a segment's end or block change.  The totals are
// exact integers, so results are bitwise deterministic however the dynamic
// segments were scheduled.
// OP = 1: single-layer operator (NEXT-1); Q holds (S_x, S_y, 0, 0) with
// S = w sigma / (4 pi) and both directions add hl S + (r.S) r / rho^2.
// GR > 0 (DLP only): the pairs of GR targets x NS sources are written stage by
// stage in lockstep (all differences, then all rho^2, all seeds, ...), which
// changes the order ptxas's list scheduler starts from.
template <int SR, int SW, int NS, int MINB = 1, int OP = 0, int UNR = (OP == 1 ? 2 : 1), int GR = 0>
__global__ void __launch_bounds__(32 * SW, MINB) k_dlp_sym(SymArgs a) {
    pdl_wait();
    static_assert(SR * SW * 32 == kSymTB, "block size fixed at 512");
    static_assert(NS == 2 || NS == 4, "2 or 4 sources per step");
    constexpr int STEPS = 32 / NS;
    __shared__ __align__(16) double2 s_src[2][SW][3][32];  // [buf][warp][(x,y) | (qa,qb) | (qc,-)][lane]
    __shared__ LogTabT<OP == 1> s_log;  // OP = 1 only
    if constexpr (OP == 1) log_tab_init(s_log, threadIdx.x, 32 * SW);  // visible after the first segment barrier
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int p = blockIdx.x;
    const long long U = a.U, Useg = a.Useg;
    if (a.trace && threadIdx.x == 0) a.trace[2 * p] = global_ns();
    const int N = a.N;
    __shared__ long long s_seg;
    int A = 0;
    long long offA = 0, offA1 = 0;
    double fxs, fxb;
    fx_scales(a.qmax, fxs, fxb);
    const long long L = 2LL * N;  // limb stride

    double tx[SR], ty[SR], tqa[SR], tqb[SR], tqc[SR], ax[SR], ay[SR];
    auto load_targets = [&](int blk) {
#pragma unroll
        for (int r = 0; r < SR; ++r) {
            const int i = blk * kSymTB + w * (32 * SR) + r * 32 + lane;
            double2 x = make_double2(0.0, 0.0);
            double4 q = make_double4(0.0, 0.0, 0.0, 0.0);
            if (i < N) {
                x = a.pos[i];
                q = a.Q[i];
            }
            tx[r] = x.x;
            ty[r] = x.y;
            tqa[r] = q.x;
            tqb[r] = q.y;
            tqc[r] = q.z;
            ax[r] = 0.0;
            ay[r] = 0.0;
        }
    };
    const int src_lane = (lane + 1) & 31;
    // The chunk's sources sit in this warp's shared-memory slice (double
    // buffered; the next unit's chunk is fetched by cp.async while this one is
    // computed); only the accumulators rotate by __shfl.
    auto fetch = [&](int buf, int blk, long long uoff) {  // chunk of unit uoff within block blk
        const int cc = (blk + 1) * (kSymTB / kSymChunk) + (int)uoff;
        const int jj = cc * kSymChunk + lane;
        const bool ok = jj < N;
        const double2 *q2 = reinterpret_cast<const double2 *>(a.Q + (ok ? jj : 0));
        cp_async16(&s_src[buf][w][0][lane], a.pos + (ok ? jj : 0), ok ? 16 : 0);
        cp_async16(&s_src[buf][w][1][lane], q2, ok ? 16 : 0);
        cp_async16(&s_src[buf][w][2][lane], q2 + 1, ok ? 16 : 0);
        cp_async_commit();
    };
    for (;;) {
    if (threadIdx.x == 0) s_seg = (long long)atomicAdd(a.counter, 1ULL);
    __syncthreads();
    const long long sg = s_seg;
    __syncthreads();
    if (sg >= a.nseg) break;
    const long long u0 = a.ub + sg * Useg, u1 = min(u0 + Useg, a.ub + U);
    if (a.off[A + 1] <= u0) {  // segments are claimed in increasing order: search forward
        int lo = A + 1, hi = a.nTB;
        while (hi - lo > 1) {
            int mid = (lo + hi) >> 1;
            if (a.off[mid] <= u0) lo = mid; else hi = mid;
        }
        A = lo;
    }
    BIE_DCHECK(A >= 0 && A < a.nTB);
    offA = a.off[A];
    offA1 = a.off[A + 1];
    load_targets(A);
    fetch(0, A, u0 - offA);
    for (long long u = u0; u < u1; ++u) {
        const int buf = (int)((u - u0) & 1);
        const int c = (A + 1) * (kSymTB / kSymChunk) + (int)(u - offA);
        const int j = c * kSymChunk + lane;
        if (u + 1 < u1) {
            if (u + 1 == offA1)
                fetch(buf ^ 1, A + 1, 0);
            else
                fetch(buf ^ 1, A, u + 1 - offA);
        } else {
            cp_async_commit();
        }
        cp_async_wait<1>();
        __syncwarp();
        double bx[NS], by[NS];
#pragma unroll
        for (int k = 0; k < NS; ++k) bx[k] = by[k] = 0.0;
        // UNR: the step loop unrolled by two for the single layer (19.84 -> 19.73 ms
        // at config 4, round 1); the DLP is faster rolled
#pragma unroll(UNR)
        for (int t = 0; t < STEPS; ++t) {
            double2 xs[NS], qs[NS];
            double cq[NS];
#pragma unroll
            for (int k = 0; k < NS; ++k) {
                const int l = (lane + t + k * STEPS) & 31;
                xs[k] = s_src[buf][w][0][l];
                qs[k] = s_src[buf][w][1][l];
                cq[k] = s_src[buf][w][2][l].x;
            }
            if constexpr (GR > 0 && OP == 0) {
                constexpr int G = GR * NS;
#pragma unroll
                for (int r0 = 0; r0 < SR; r0 += GR) {
                    double rx[G], ry[G], yy[G], xy[G], d[G], iv[G], cs[G], ct[G];
#pragma unroll
                    for (int q = 0; q < G; ++q) {
                        const int r = r0 + q / NS, k = q % NS;
                        rx[q] = tx[r] - xs[k].x;
                        ry[q] = ty[r] - xs[k].y;
                    }
#pragma unroll
                    for (int q = 0; q < G; ++q) {
                        yy[q] = fma(ry[q], ry[q], 1e-150);
                        xy[q] = rx[q] * ry[q];
                    }
#pragma unroll
                    for (int q = 0; q < G; ++q) {
                        d[q] = fma(rx[q], rx[q], yy[q]);
                        iv[q] = rcp_approx(d[q]);
                    }
#pragma unroll
                    for (int q = 0; q < G; ++q) {
                        const int r = r0 + q / NS, k = q % NS;
                        cs[q] = fma(qs[k].x, d[q], fma(qs[k].y, xy[q], cq[k] * yy[q]));
                        ct[q] = fma(tqa[r], d[q], fma(tqb[r], xy[q], tqc[r] * yy[q]));
                    }
#pragma unroll
                    for (int q = 0; q < G; ++q) {
                        const double e = fma(-d[q], iv[q], 1.0);
                        iv[q] = fma(iv[q], fma(e, e, e), iv[q]);
                    }
#pragma unroll
                    for (int q = 0; q < G; ++q) {
                        const int r = r0 + q / NS, k = q % NS;
                        const double qq = iv[q] * iv[q];
                        const double av = cs[q] * qq, bv = ct[q] * qq;
                        ax[r] = fma(av, rx[q], ax[r]);
                        ay[r] = fma(av, ry[q], ay[r]);
                        bx[k] = fma(-bv, rx[q], bx[k]);
                        by[k] = fma(-bv, ry[q], by[k]);
                    }
                }
            } else {
#pragma unroll
            for (int r = 0; r < SR; ++r) {
#pragma unroll
                for (int k = 0; k < NS; ++k) {
                    if constexpr (OP == 1)
                        slp_pairpair(tx[r], ty[r], tqa[r], tqb[r], xs[k].x, xs[k].y, qs[k].x, qs[k].y, ax[r], ay[r],
                                     bx[k], by[k], s_log);
                    else
                        dlp_pairpair(tx[r], ty[r], tqa[r], tqb[r], tqc[r], xs[k].x, xs[k].y, qs[k].x, qs[k].y, cq[k],
                                     ax[r], ay[r], bx[k], by[k]);
                }
            }
            }
#pragma unroll
            for (int k = 0; k < NS; ++k) {
                bx[k] = shfl_d(bx[k], src_lane);
                by[k] = shfl_d(by[k], src_lane);
            }
        }
        // after STEPS rotations, lane l's accumulator k belongs to source
        // l + (k + 1) STEPS (mod 32): gather source l's NS parts in fixed order
        double sx = 0.0, sy = 0.0;
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            const int from = (lane - (k + 1) * STEPS) & 31;
            sx += shfl_d(bx[k], from);
            sy += shfl_d(by[k], from);
        }
        // each warp adds its own 32 source sums: the limb totals do not depend on
        // the order, so no cross-warp reduction (and no block barrier) per unit
        if (j < N) {
            fx_add(a.acc + 2LL * j, L, sx * fxs);
            fx_add(a.acc + 2LL * j + 1, L, sy * fxs);
        }
        if (u + 1 == u1 || u + 1 == offA1) {
#pragma unroll
            for (int r = 0; r < SR; ++r) {
                const int i = A * kSymTB + w * (32 * SR) + r * 32 + lane;
                if (i < N) {
                    fx_add(a.acc + 2LL * i, L, ax[r] * fxs);
                    fx_add(a.acc + 2LL * i + 1, L, ay[r] * fxs);
                }
            }
            if (u + 1 < u1) {
                ++A;
                offA = offA1;
                offA1 = a.off[A + 1];
                load_targets(A);
            }
        }
    }
    }  // segments
    if (a.trace && threadIdx.x == 0) a.trace[2 * p + 1] = global_ns();
}

// Pairs inside one 512-node block (one-sided, all ordered pairs, self pair
// zeroed by the rho^2 + 1e-300 rule).  Two CTAs per block (one per half of its
// targets, 128 threads x 2 targets; all 512 sources staged): a config-4 launch
// is 532 CTAs instead of 266 -- 3.6 instead of 1.8 CTAs per SM evens out the
// partial last wave.  Per-target sums are unchanged (same sources, same order).
// OP = 1: single-layer pairs (sigma = pre-scaled S, nw unused; the self pair
// vanishes through slp_factors).
// split > 1 (few blocks, small N): the sources of a block are cut into `split`
// ranges handled by separate CTAs, writing partial sums to diag + part * 2N (the
// epilogue adds the parts in order), so small problems fill more SMs.
template <int OP = 0>
__global__ void __launch_bounds__(128) k_dlp_diag(const double2 *__restrict__ pos, const double2 *__restrict__ nw,
                                                  const double *__restrict__ sigma, double *diag, int N,
                                                  int blk0 = 0, int split = 1) {
    pdl_wait();
    __shared__ double2 sp[3][kSymTB];
    __shared__ LogTab s_log;  // OP = 1 only; visible after the staging barrier
    if constexpr (OP == 1) log_tab_init(s_log, threadIdx.x, 128);
    const int part = blockIdx.x % split, bh = blockIdx.x / split;
    const int A = blk0 + (bh >> 1), half = bh & 1, tid = threadIdx.x;
    const int base = A * kSymTB;
    constexpr int RT = kSymTB / 256;  // targets per thread
    for (int q = tid; q < kSymTB; q += 128) {
        const int j = base + q;
        const bool ok = j < N;
        sp[0][q] = ok ? pos[j] : make_double2(0.0, 0.0);
        sp[1][q] = (ok && OP == 0) ? nw[j] : make_double2(0.0, 0.0);
        sp[2][q] = ok ? reinterpret_cast<const double2 *>(sigma)[j] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    double tx[RT], ty[RT], ax[RT], ay[RT];
#pragma unroll
    for (int r = 0; r < RT; ++r) {
        const double2 x = sp[0][half * 256 + r * 128 + tid];
        tx[r] = x.x;
        ty[r] = x.y;
        ax[r] = 0.0;
        ay[r] = 0.0;
    }
    const int nsrc = min(kSymTB, N - base);
    const int j0 = part * (kSymTB / split);
    const int j1 = part == split - 1 ? nsrc : min(nsrc, (part + 1) * (kSymTB / split));
#pragma unroll 2
    for (int jj = j0; jj < j1; ++jj) {
        const double2 xj = sp[0][jj], nj = sp[1][jj], sj = sp[2][jj];
#pragma unroll
        for (int r = 0; r < RT; ++r) {
            if constexpr (OP == 1) {
                const double rx = tx[r] - xj.x;
                const double ry = ty[r] - xj.y;
                double hl, inv;
                slp_factors(rx, ry, hl, inv, s_log);
                const double c = inv * fma(rx, sj.x, ry * sj.y);
                ax[r] = fma(c, rx, fma(hl, sj.x, ax[r]));
                ay[r] = fma(c, ry, fma(hl, sj.y, ay[r]));
                continue;
            }
            const double rx = tx[r] - xj.x;
            const double ry = ty[r] - xj.y;
            const double rho2 = fma(rx, rx, fma(ry, ry, 1e-300));
            const double rn = fma(rx, nj.x, ry * nj.y);
            double inv = rcp_approx(rho2);
            const double e = fma(-rho2, inv, 1.0);
            inv = fma(inv, fma(e, e, e), inv);
            const double c = ((rn * inv) * inv) * fma(rx, sj.x, ry * sj.y);
            ax[r] = fma(c, rx, ax[r]);
            ay[r] = fma(c, ry, ay[r]);
        }
    }
#pragma unroll
    for (int r = 0; r < RT; ++r) {
        const int i = base + half * 256 + r * 128 + tid;
        if (i < N) reinterpret_cast<double2 *>(diag + (long long)part * 2LL * N)[i] = make_double2(ax[r], ay[r]);
    }
}

// acc += sum_{q < n} p[q * stride + 2i .. 2i+1] in order q = 0, 1, ..., with
// the loads issued 8 at a time (the adds stay sequential, so the order and the
// result are unchanged; the loop was latency-bound on one load per add).
__device__ __forceinline__ void sum_strided(double2 &acc, const double *p, long long stride, int n, int i) {
    // SUM_ILP loads in flight per thread (16 measured no faster: the sum runs at
    // ~4.2 TB/s over ~415 MB of partials at config 4)
    constexpr int SUM_ILP = 8;
    int q = 0;
    for (; q + SUM_ILP <= n; q += SUM_ILP) {
        double2 v[SUM_ILP];
#pragma unroll
        for (int t = 0; t < SUM_ILP; ++t) v[t] = reinterpret_cast<const double2 *>(p + (long long)(q + t) * stride)[i];
#pragma unroll
        for (int t = 0; t < SUM_ILP; ++t) {
            acc.x += v[t].x;
            acc.y += v[t].y;
        }
    }
    for (; q < n; ++q) {
        const double2 v = reinterpret_cast<const double2 *>(p + (long long)q * stride)[i];
        acc.x += v.x;
        acc.y += v.y;
    }
}

struct Chunk {
    int v0, nv, TB, nTS, P;
    long long U, Useg;
};
struct SymEpi {
    int on;                    // 1: partials come from the symmetric path (nvec = 1)
    const unsigned long long *acc;   // [3][2N] fixed-point limbs of the pair sums (fx_add)
    const unsigned long long *qmax;  // accumulation window (fx_scales)
    const double *diag;        // [dsplit][2N] in-block pair sums (k_dlp_diag)
    int dsplit;                // in-block sums come in dsplit parts [dsplit][2N]
};
// A5 completion field of every pore at one target (nvec = 1; readings C5/C6):
// sum over pores k of the Stokeslet (lambda_k / 4 pi) and rotlet (r_k mu_k)
// terms, pore records staged through shared memory in tiles of 128
// (warp-broadcast reads); 1/rho^2 by seed + cubic Newton.  Every thread of the
// CTA must call it (barriers); accumulators c[q mod 4] break the serial add chain.
struct PoreStage {
    double4 pc[128];  // (cx, cy, r, -)
    double4 pm[128];  // (lambda_x / 4 pi, lambda_y / 4 pi, r mu, -)
    LogTabX lt;       // table log (visible after the first tile barrier)
};
__device__ __forceinline__ double2 pore_completion(double2 xi, const double4 *__restrict__ pore,
                                                   const double *__restrict__ moments, int M, PoreStage &ps,
                                                   int tid, int nthreads) {
    constexpr double k4pi = 1.0 / (4.0 * kPi);
    constexpr int ILP = 4;
    log_tab_init(ps.lt, tid, nthreads);
    double2 c[ILP];
#pragma unroll
    for (int u2 = 0; u2 < ILP; ++u2) c[u2] = make_double2(0.0, 0.0);
    for (int k0 = 0; k0 < M; k0 += 128) {
        const int nk = min(128, M - k0);
        __syncthreads();
        for (int q = tid; q < nk; q += nthreads) {
            const int k = k0 + q;
            const double4 pk = pore[k];
            ps.pc[q] = pk;
            const double *m = moments + (long long)k * 3;
            ps.pm[q] = make_double4(k4pi * m[0], k4pi * m[1], pk.z * m[2], 0.0);
        }
        __syncthreads();
        auto pore_term = [&](int q, double2 &cc) {
            const double4 pk = ps.pc[q], pm = ps.pm[q];
            const double rx = xi.x - pk.x, ry = xi.y - pk.y;
            const double rho2 = fma(rx, rx, ry * ry);
            double ir = rcp_approx(rho2);
            const double e = fma(-rho2, ir, 1.0);
            ir = fma(ir, fma(e, e, e), ir);
            const double nlg = neg_half_log_tab(rho2, ps.lt);  // -log rho
            const double rl = fma(rx, pm.x, ry * pm.y) * ir;    // (r . lambda/4pi) / rho^2
            const double mr = pm.z * ir;                         // r_k mu / rho^2
            // accumulated term by term (3 FMA per component, no DMUL/DADD)
            cc.x = fma(mr, ry, fma(rl, rx, fma(nlg, pm.x, cc.x)));
            cc.y = fma(-mr, rx, fma(rl, ry, fma(nlg, pm.y, cc.y)));
        };
        int q = 0;
        for (; q + ILP <= nk; q += ILP) {
#pragma unroll
            for (int u2 = 0; u2 < ILP; ++u2) pore_term(q + u2, c[u2]);
        }
        for (; q < nk; ++q) pore_term(q, c[0]);
    }
    return make_double2((c[0].x + c[1].x) + (c[2].x + c[3].x), (c[0].y + c[1].y) + (c[2].y + c[3].y));
}

struct EpiArgs {
    const double2 *pos, *nrm, *tan;
    const double *selfc;
    const double4 *pore;
    const double *sigma;
    long long sig_stride;
    const double *partial;
    const double *moments;
    double *out;
    int nvec, N, M, wall_lo, row_begin, Nt;
    unsigned flags;
    int nchunks;
    Chunk ch[5];
    SymEpi sym;
    const double *presum;  // nvec = 1: pair sums already reduced (sharded path), local rows [2 Nt]
    int op;                // 0: completed DLP; 1: single-layer operator + Kapur-Rokhlin correction
    int n_pore;
    const double *slp_s;   // op 1: S = w sigma / (4 pi), [nvec][2N]
    double kr[6];          // op 1: gamma_1..gamma_6
};

// A4 + A5: reduce the split partials in fixed slot order, then add the local
// terms and the completion field of every pore.
// NVC > 0: nvec is the compile-time constant NVC (accumulators stay in
// registers); NVC == 0: generic nvec.
template <int NVC>
__global__ void __launch_bounds__(128) k_epilogue(EpiArgs a) {
    pdl_wait();
    const int it_raw = blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = it_raw < a.Nt;  // inactive threads still join the block barriers
    const int it = active ? it_raw : a.Nt - 1;
    const int nvec = NVC > 0 ? NVC : a.nvec;
    const int i = a.row_begin + it;
    const double2 xi = a.pos[i];
    const double2 ti = a.tan[i];
    const double sc = a.selfc[i];
    const bool full = !(a.flags & BIE_D_ONLY);
    constexpr double k4pi = 1.0 / (4.0 * kPi);
    double2 u[NVC > 0 ? NVC : BIE_MAX_NVEC];
    // nvec = 1: odd CTAs compute the (FP64-bound) completion field before the
    // (memory-bound) partial sums, even CTAs after, so that the two phases
    // overlap across the wave; the field is added at the same place either way
    __shared__ std::conditional_t<NVC == 1, PoreStage, char> s_ps;
    const bool pore_phase = NVC == 1 && full && a.op == 0;
    const bool pore_first = pore_phase && (blockIdx.x & 1);
    double2 pc = make_double2(0.0, 0.0);
    if constexpr (NVC == 1) {
        if (pore_first) pc = pore_completion(xi, a.pore, a.moments, a.M, s_ps, threadIdx.x, blockDim.x);
    }
    if (a.presum) u[0] = reinterpret_cast<const double2 *>(a.presum)[it];
    if (a.sym.on) {
        // exact limb totals of the symmetric kernel, then the in-block parts in order
        double fxs, fxb;
        fx_scales(a.sym.qmax, fxs, fxb);
        double2 acc = make_double2(fx_value(a.sym.acc + 2LL * i, 2LL * a.N, fxb),
                                   fx_value(a.sym.acc + 2LL * i + 1, 2LL * a.N, fxb));
        for (int q = 0; q < a.sym.dsplit; ++q) {
            const double2 pv = reinterpret_cast<const double2 *>(a.sym.diag + (long long)q * 2LL * a.N)[i];
            acc.x += pv.x;
            acc.y += pv.y;
        }
        u[0] = acc;
    }
    for (int c = 0; c < a.nchunks; ++c) {
        const Chunk ch = a.ch[c];
        const int tb = it / ch.TB;
        const int first = (int)seg_of((long long)tb * ch.nTS, 0, ch.Useg);
        const int last = (int)seg_of((long long)(tb + 1) * ch.nTS - 1, 0, ch.Useg);
        // NVC in {1, 4, 16}: nvec is one variant size -> a single chunk at v0 = 0
        const int nv = NVC > 0 ? NVC : ch.nv;
#pragma unroll
        for (int vv = 0; vv < nv; ++vv) {
            const int v = NVC > 0 ? vv : ch.v0 + vv;
            double2 acc = make_double2(0.0, 0.0);
            for (int sl = 0; sl <= last - first; ++sl) {
                const double2 pv = reinterpret_cast<const double2 *>(
                    a.partial + ((long long)sl * nvec + v) * 2LL * a.Nt)[it];
                acc.x += pv.x;
                acc.y += pv.y;
            }
            u[v] = acc;
        }
    }
    if (a.op == 1) {
        // Kapur-Rokhlin correction (reading C25): the all-pairs sum used w_j for
        // every j != i; the 12 periodic neighbours on i's own curve carry
        // w_j (1 + gamma_k), i.e. + gamma_k G(x_i, x_j) (w_j sigma_j).
        int lo, n;
        if (i < a.wall_lo) {
            lo = (i / a.n_pore) * a.n_pore;
            n = a.n_pore;
        } else {
            lo = a.wall_lo;
            n = a.N - a.wall_lo;
        }
        const int li = i - lo;
#pragma unroll
        for (int k = 1; k <= 6; ++k) {
            const double gk = a.kr[k - 1];
            for (int sg = 0; sg < 2; ++sg) {
                int lj = sg == 0 ? li + k : li - k;
                lj = lj >= n ? lj - n : (lj < 0 ? lj + n : lj);
                const int j = lo + lj;
                const double2 xj = a.pos[j];
                const double rx = xi.x - xj.x, ry = xi.y - xj.y;
                const double d = rx * rx + ry * ry;
                const double hl = -0.5 * log(d), inv = 1.0 / d;
                for (int v = 0; v < nvec; ++v) {
                    const double2 sj = reinterpret_cast<const double2 *>(a.slp_s + (long long)v * 2LL * a.N)[j];
                    const double c = inv * (rx * sj.x + ry * sj.y);
                    u[v].x += gk * (hl * sj.x + c * rx);
                    u[v].y += gk * (hl * sj.y + c * ry);
                }
            }
        }
        if (!active) return;
        for (int v = 0; v < nvec; ++v)
            reinterpret_cast<double2 *>(a.out + (long long)v * 2LL * a.Nt)[it] = u[v];
        return;
    }
    for (int v = 0; v < nvec; ++v) {
        const double2 si = reinterpret_cast<const double2 *>(a.sigma + (long long)v * a.sig_stride)[i];
        const double ts = sc * (ti.x * si.x + ti.y * si.y);
        u[v].x += ts * ti.x;
        u[v].y += ts * ti.y;
        if (full) {
            u[v].x += -0.5 * si.x;
            u[v].y += -0.5 * si.y;
            if (i >= a.wall_lo) {
                const double nu = a.moments[(long long)nvec * a.M * 3 + v];
                const double2 ni = a.nrm[i];
                u[v].x += nu * ni.x;
                u[v].y += nu * ni.y;
            }
        }
    }
    if (full && NVC == 1) {
        if constexpr (NVC == 1) {
            if (!pore_first) pc = pore_completion(xi, a.pore, a.moments, a.M, s_ps, threadIdx.x, blockDim.x);
        }
        u[0].x += pc.x;
        u[0].y += pc.y;
    } else if (full) {
        __shared__ LogTab s_log2;
        log_tab_init(s_log2, threadIdx.x, blockDim.x);
        __syncthreads();
        for (int k = 0; k < a.M; ++k) {
            const double4 pk = a.pore[k];
            const double rx = xi.x - pk.x, ry = xi.y - pk.y;
            const double rho2 = rx * rx + ry * ry;
            const double ir = 1.0 / rho2;
            const double lg = -neg_half_log_tab(rho2, s_log2);  // log rho
            const double rk = pk.z * ir;
            for (int v = 0; v < nvec; ++v) {
                const double *m = a.moments + ((long long)v * a.M + k) * 3;
                const double lx = m[0], ly = m[1], mu = m[2];
                const double rl = (rx * lx + ry * ly) * ir;
                u[v].x += k4pi * (-lg * lx + rx * rl) + rk * ry * mu;
                u[v].y += k4pi * (-lg * ly + ry * rl) - rk * rx * mu;
            }
        }
    }
    if (!active) return;
    for (int v = 0; v < nvec; ++v)
        reinterpret_cast<double2 *>(a.out + (long long)v * 2LL * a.Nt)[it] = u[v];
}

template <int NV, int R, int TS>
static void *pair_kernel_ptr(int op) {
    // nvec = 16: register cap of 4 CTAs per SM (128 registers, no spills; was 142 at
    // 3 CTAs/SM): config-4 DLP nvec-16 kernel 100.9 -> 95.7 ms
    return op ? reinterpret_cast<void *>(&k_dlp_pairs<NV, R, TS, 1, (NV == 16 ? 4 : 1)>)
              : reinterpret_cast<void *>(&k_dlp_pairs<NV, R, TS, 0, (NV == 16 ? 4 : 1)>);
}

static void *variant_kernel(int idx, int op = 0) {
    switch (idx) {
        case 0: return pair_kernel_ptr<1, 4, 256>(op);
        case 1: return pair_kernel_ptr<2, 2, 256>(op);
        case 2: return pair_kernel_ptr<4, 4, 256>(op);
        case 3: return pair_kernel_ptr<8, 1, 128>(op);
        default: return pair_kernel_ptr<16, 1, 64>(op);
    }
}

static int variant_index(int nv) {
    switch (nv) {
        case 1: return 0;
        case 2: return 1;
        case 4: return 2;
        case 8: return 3;
        default: return 4;
    }
}

// Fill the schedule of one variant for Nt targets and N sources.
static void make_sched(const Geometry *g, int vi, int Nt, PairSched &s, int op = 0) {
    const Variant &V = kVariants[vi];
    s.nv = V.nv;
    s.R = V.R;
    s.TS = V.TS;
    s.TB = kPairThreads * V.R;
    s.nTB = (Nt + s.TB - 1) / s.TB;
    s.nTS = (g->N + s.TS - 1) / s.TS;
    s.U = (long long)s.nTB * s.nTS;
    s.smem = 2 * (2 + V.nv) * V.TS * (int)sizeof(double2);
    long long Pmax = (long long)g->num_sms * std::max(1, op ? g->occ_slp[vi] : g->occ[vi]);
    s.P = (int)std::min<long long>(Pmax, s.U);
    // max slots per target block: ceil(P / nTB) + 1 bounds it; compute exactly
    // ~16 segments per CTA: tail <= one segment, few slots per target block
    s.Useg = std::max<long long>(std::max<long long>(1, std::min<long long>(4, s.U / s.P)),
                                 (s.U + 16LL * s.P - 1) / (16LL * s.P));
    int S = 1;
    for (int tb = 0; tb < s.nTB; ++tb) {
        const long long f = seg_of((long long)tb * s.nTS, 0, s.Useg);
        const long long l = seg_of((long long)(tb + 1) * s.nTS - 1, 0, s.Useg);
        S = std::max(S, (int)(l - f + 1));
    }
    s.S = S;
}

int build_schedules(Geometry *g) {
    size_t need = 0;
    for (int vi = 0; vi < 5; ++vi) {
        const Variant &V = kVariants[vi];
        int smem = 2 * (2 + V.nv) * V.TS * (int)sizeof(double2);
        for (int op = 0; op < 2; ++op) {  // completed DLP, single-layer (NEXT-1)
            cudaError_t e =
                cudaFuncSetAttribute(variant_kernel(vi, op), cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(k_dlp_pairs)");
            int occ = 0;
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, variant_kernel(vi, op), kPairThreads, smem);
            if (e != cudaSuccess) return cuda_fail(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
            (op ? g->occ_slp : g->occ)[vi] = std::max(1, occ);
            PairSched s;
            make_sched(g, vi, g->N, s, op);
            (op ? g->sched_slp : g->sched)[vi] = s;
            need = std::max(need, (size_t)s.S * V.nv * 2 * (size_t)g->N);  // grows on demand in dlp_apply_impl
        }
    }
    cudaError_t e = cudaMalloc(&g->partial, need * sizeof(double));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(partial)");
    e = cudaMalloc(&g->pair_counter, sizeof(unsigned long long) * 8);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(pair counters)");
    g->partial_elems = need;
    return BIE_OK;
}

// Symmetric DLP kernel variants (BIE_SYM_VARIANT, A/B only; the default is
// chosen by size in sym_prepare): 0 = (8 targets per lane, 2 warps, 2 sources
// per step in lockstep groups of 4 targets) register-capped at 6 CTAs per SM
// (170 registers, no spills: 3 warps per SMSP) -- N >= 65536, 12.71 ms at
// config 4; 2 = the same uncapped (249 registers, 2 warps per SMSP, step loop
// unrolled by two) -- smaller N, where the capped form's 888 CTAs share too
// few work units (config 2 BD-GMRES 3.77 vs 3.95 ms, config 3 127.5 vs
// 129.2 ms; config 4 12.79 ms); 1 = (4, 4, 2) capped at 3 CTAs of 4 warps per
// SM.  Round 1-2 sweeps of the other shapes: DESIGN.md s5.
static const int kNumSymVar = 3;
static void *sym_kernel(int v) {
    if (v == 1) return reinterpret_cast<void *>(&k_dlp_sym<4, 4, 2, 3>);
    if (v == 2) return reinterpret_cast<void *>(&k_dlp_sym<8, 2, 2, 1, 0, 2, 4>);
    return reinterpret_cast<void *>(&k_dlp_sym<8, 2, 2, 6, 0, 1, 4>);
}
static int sym_warps(int v) { return v == 1 ? 4 : 2; }
static void launch_sym(int v, int P, const SymArgs &sa, cudaStream_t st) {
    if (v == 1)
        BIE_LAUNCH((k_dlp_sym<4, 4, 2, 3>), P, 128, 0, st, sa);
    else if (v == 2)
        BIE_LAUNCH((k_dlp_sym<8, 2, 2, 1, 0, 2, 4>), P, 64, 0, st, sa);
    else
        BIE_LAUNCH((k_dlp_sym<8, 2, 2, 6, 0, 1, 4>), P, 64, 0, st, sa);
}
static void *slp_sym_kernel(int v) {
    if (v == 1) return reinterpret_cast<void *>(&k_dlp_sym<4, 4, 2, 3, 1>);
    return reinterpret_cast<void *>(&k_dlp_sym<8, 2, 2, 1, 1>);
}
static void launch_sym_slp(int v, int P, const SymArgs &sa, cudaStream_t st) {
    if (v == 1)
        BIE_LAUNCH((k_dlp_sym<4, 4, 2, 3, 1>), P, 128, 0, st, sa);
    else
        BIE_LAUNCH((k_dlp_sym<8, 2, 2, 1, 1>), P, 64, 0, st, sa);
}

// Segment size of the dynamic work distribution: about 8 segments per CTA
// (tail <= one segment), at least 8 units so a segment amortises its start.
// Below 8 units per CTA (small N), smaller segments so every CTA gets work
// (config 2: 92 -> 44 us per matvec); measured at config 3, segments under 8
// units cost more in per-segment start-up than they save in tail.
static long long sym_useg(long long U, int P) {
    long long lo = std::max<long long>(1, std::min<long long>(8, U / P));
    if (const char *e = getenv("BIE_SYM_USEG_MIN")) lo = std::max(1, atoi(e));  // tuning knob
    // segments per CTA (knob BIE_SYM_SEGS_PER_CTA); config 4, ms per matvec (round 1):
    // 8: 13.170, 12: 13.172, 16: 13.173, 24: 13.185, 32: 13.193, 48: 13.237.
    // Each segment writes one 512-node slot of target partials, so fewer
    // segments also mean fewer slots (DRAM traffic ~ segments x 8 KB).
    long long per = 8;
    if (const char *e = getenv("BIE_SYM_SEGS_PER_CTA")) per = std::max(1, atoi(e));
    return std::max<long long>(lo, (U + per * P - 1) / (per * P));
}

// Schedule of one launch over the slice [ub, ub + U) of the unit list for
// operator op: persistent CTAs P and units per segment Useg.
struct SymPlan {
    int P = 1;
    long long Useg = 1;
};
static SymPlan sym_plan(const Geometry *g, long long U, int op) {
    SymPlan pl;
    pl.P = (int)std::max<long long>(1, std::min<long long>((long long)g->num_sms * g->sym_occ[op], U));
    pl.Useg = sym_useg(U, pl.P);
    return pl;
}

// Lazily allocate the symmetric path's schedule and buffers (nvec = 1 only):
// O(N) memory -- the fixed-point limb accumulators [3][2N] (fx_add), the
// in-block parts [4][2N], the per-node quadratic forms and the block table.
static int sym_prepare(Geometry *g) {
    if (g->sym_state != 0) return BIE_OK;
    const int N = g->N;
    const int nTB = (N + kSymTB - 1) / kSymTB;
    const long long nC = (N + kSymChunk - 1) / kSymChunk;
    g->sym_variant = N >= 65536 ? 0 : 2;  // see sym_kernel
    if (const char *e = getenv("BIE_SYM_VARIANT")) g->sym_variant = std::max(0, std::min(kNumSymVar - 1, atoi(e)));  // tuning knob
    if (const char *e = getenv("BIE_SLP_SYM_VARIANT")) g->slp_sym_variant = std::max(0, std::min(1, atoi(e)));
    std::vector<long long> off(nTB + 1, 0);
    for (int A = 0; A < nTB; ++A) {
        long long n = nC - (long long)(A + 1) * (kSymTB / kSymChunk);
        off[A + 1] = off[A] + std::max(0LL, n);
    }
    const long long U = off[nTB];
    for (int op = 0; op < 2; ++op) {
        int occ = 0;
        void *k = op ? slp_sym_kernel(g->slp_sym_variant) : sym_kernel(g->sym_variant);
        const int threads = op ? (g->slp_sym_variant == 1 ? 128 : 64) : 32 * sym_warps(g->sym_variant);
        BIE_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, 0));
        g->sym_occ[op] = std::max(1, occ);
    }
    // in-block pairs: split each block's sources over up to 16 CTAs when there are
    // too few blocks to fill the SMs (2 CTAs per block before splitting; config 2:
    // 4 blocks x 2 x 16 = 128 CTAs of 32 sources each)
    g->sym_dsplit = (int)std::max<long long>(1, std::min<long long>(16, (2LL * g->num_sms + 2LL * nTB - 1) / (2LL * nTB)));
    g->sym_nTB = nTB;
    g->sym_U = U;
    g->sym_state = -1;  // stays -1 (one-sided path) if an allocation fails
    if (cudaMalloc(&g->sym_counter, sizeof(unsigned long long) * 2) != cudaSuccess ||
        cudaMalloc(&g->sym_Q, sizeof(double4) * (size_t)N) != cudaSuccess ||
        cudaMalloc(&g->sym_off, sizeof(long long) * (size_t)(nTB + 1)) != cudaSuccess ||
        cudaMalloc(&g->sym_acc, sizeof(unsigned long long) * 6 * (size_t)N) != cudaSuccess ||
        cudaMalloc(&g->sym_diag, sizeof(double) * 2 * (size_t)N * g->sym_dsplit) != cudaSuccess) {
        (void)cudaGetLastError();  // clear the (non-sticky) allocation error
        return BIE_OK;
    }
    BIE_CUDA_TRY(cudaMemcpy(g->sym_off, off.data(), sizeof(long long) * (size_t)(nTB + 1), cudaMemcpyHostToDevice));
    const SymPlan p0 = sym_plan(g, U, 0), p1 = sym_plan(g, U, 1);
    if (getenv("BIE_SYM_TRACE"))
        cudaMalloc(&g->sym_trace, sizeof(unsigned long long) * 2 * (size_t)std::max(p0.P, p1.P));
    g->sym_P = p0.P;
    g->sym_Useg = p0.Useg;
    g->sym_state = 1;
    return BIE_OK;
}

// The max |Q| word (sym_counter[1]) must be zero before k_quad / k_slp_scale.
static int sym_pre(Geometry *g, cudaStream_t st) {
    BIE_CUDA_TRY(cudaMemsetAsync(g->sym_counter, 0, sizeof(unsigned long long) * 2, st));
    return BIE_OK;
}

// Launch the symmetric kernel on the slice [ub, ub + U).  The limb accumulators
// were zeroed by k_quad / k_slp_scale, the segment counter and max |Q| by sym_pre.
static int sym_launch(Geometry *g, long long ub, long long U, int op, cudaStream_t st) {
    if (U <= 0) return BIE_OK;
    const SymPlan pl = sym_plan(g, U, op);
    SymArgs sa{g->pos, g->sym_Q, g->sym_off, g->sym_acc, g->sym_counter + 1, g->N, g->sym_nTB, U, ub,
               (ub == 0 && U == g->sym_U) ? g->sym_trace : nullptr, pl.Useg, (U + pl.Useg - 1) / pl.Useg,
               g->sym_counter};
    if (op)
        launch_sym_slp(g->slp_sym_variant, pl.P, sa, st);
    else
        launch_sym(g->sym_variant, pl.P, sa, st);
    count_launch();
    BIE_CUDA_TRY(cudaGetLastError());
    return BIE_OK;
}

static void launch_pairs(int vi, const PairSched &s, const PairArgs &a, cudaStream_t st, int op = 0) {
    if (op) {
        switch (vi) {
            case 0: k_dlp_pairs<1, 4, 256, 1><<<s.P, kPairThreads, s.smem, st>>>(a); break;
            case 1: k_dlp_pairs<2, 2, 256, 1><<<s.P, kPairThreads, s.smem, st>>>(a); break;
            case 2: k_dlp_pairs<4, 4, 256, 1><<<s.P, kPairThreads, s.smem, st>>>(a); break;
            case 3: k_dlp_pairs<8, 1, 128, 1><<<s.P, kPairThreads, s.smem, st>>>(a); break;
            default: k_dlp_pairs<16, 1, 64, 1, 4><<<s.P, kPairThreads, s.smem, st>>>(a); break;
        }
        return;
    }
    switch (vi) {
        case 0: k_dlp_pairs<1, 4, 256><<<s.P, kPairThreads, s.smem, st>>>(a); break;
        case 1: k_dlp_pairs<2, 2, 256><<<s.P, kPairThreads, s.smem, st>>>(a); break;
        case 2: k_dlp_pairs<4, 4, 256><<<s.P, kPairThreads, s.smem, st>>>(a); break;
        case 3: k_dlp_pairs<8, 1, 128><<<s.P, kPairThreads, s.smem, st>>>(a); break;
        default: k_dlp_pairs<16, 1, 64, 0, 4><<<s.P, kPairThreads, s.smem, st>>>(a); break;
    }
}

// NEXT-1: S = w sigma / (4 pi) for every vector (the single-layer source
// strength), and for the symmetric path also the (S_x, S_y, 0, 0) records.
__global__ void k_slp_scale(const double *__restrict__ w, const double *__restrict__ sigma, long long stride,
                            int nvec, int N, double *S, double4 *Q, unsigned long long *qmax_bits = nullptr,
                            unsigned long long *acc = nullptr) {
    pdl_wait();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    double m = 0.0;
    if (acc && j < N) zero_limbs(acc, j, N);
    if (j < N) {
        const double f = w[j] * (1.0 / (4.0 * kPi));
        for (int v = 0; v < nvec; ++v) {
            const double2 sj = reinterpret_cast<const double2 *>(sigma + (long long)v * stride)[j];
            const double2 o = make_double2(f * sj.x, f * sj.y);
            reinterpret_cast<double2 *>(S + (long long)v * 2LL * N)[j] = o;
            if (Q && v == 0) {
                Q[j] = make_double4(o.x, o.y, 0.0, 0.0);
                m = fmax(fabs(o.x), fabs(o.y));
            }
        }
    }
    if (qmax_bits) qmax_update(m, qmax_bits);
}

static int slp_prepare(Geometry *g) {
    if (g->slp_s) return BIE_OK;
    BIE_CUDA_TRY(cudaMalloc(&g->slp_s, sizeof(double) * BIE_MAX_NVEC * 2 * (size_t)g->N));
    return BIE_OK;
}

int dlp_apply_impl(Geometry *g, const double *sigma, double *out, int nvec, unsigned flags, int row_begin,
                   int row_end, cudaStream_t st) {
    const int N = g->N;
    const int Nt = row_end - row_begin;
    if (Nt <= 0) return BIE_OK;
    const long long stride = 2LL * N;
    const int op = (flags & kOpSLP) ? 1 : 0;
    const bool full = !(flags & BIE_D_ONLY) && !op;
    const double *sigma_in = sigma;  // the caller's density (epilogue local terms)
    if (op) {
        int rc = slp_prepare(g);
        if (rc != BIE_OK) return rc;
    }
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    if (g->prof) {
        while (g->prof_ev.size() < g->prof_used + 4) {
            cudaEvent_t e;
            BIE_CUDA_TRY(cudaEventCreate(&e));
            g->prof_ev.push_back(e);
        }
        for (int q = 0; q < 4; ++q) ev[q] = g->prof_ev[g->prof_used + q];
        g->prof_used += 4;
        BIE_CUDA_TRY(cudaEventRecord(ev[0], st));
    }
    EpiArgs ea{};
    const bool sym = nvec == 1 && row_begin == 0 && row_end == N && !(flags & BIE_ONE_SIDED) &&
                     sym_prepare(g) == BIE_OK && g->sym_state == 1;
    if (full && !sym) {  // (symmetric path: on the side stream with the in-block kernel, below)
        count_launch();
        BIE_LAUNCH(k_moments, g->M + 1, 256, 0, st, g->pos, g->nrm, g->w, g->pore, sigma, stride, nvec, g->M,
                   g->n_pore, g->wall_lo, N, g->wall_len, g->moments);
        BIE_CUDA_TRY(cudaGetLastError());
    }
    if (sym) {
        int rc = sym_pre(g, st);
        if (rc) return rc;
    }
    if (op) {
        BIE_LAUNCH(k_slp_scale, (N + 255) / 256, 256, 0, st, g->w, sigma, stride, nvec, N, g->slp_s,
                   sym ? g->sym_Q : nullptr, sym ? g->sym_counter + 1 : nullptr, sym ? g->sym_acc : nullptr);
        count_launch();
        sigma = g->slp_s;  // the pair kernels read S
    }
    if (sym) {
        if (!op) {
            BIE_LAUNCH(k_quad, (N + 255) / 256, 256, 0, st, g->nw, sigma, g->sym_Q, N, g->sym_counter + 1,
                       g->sym_acc);
            count_launch();
        }
        // The in-block pairs (k_dlp_diag) depend only on sigma / S: they run on a
        // side stream forked here and joined before the epilogue, so their CTAs
        // fill the SMs that the persistent pair kernel's tail leaves idle
        // (fork/join events; inside the GMRES graph this becomes a parallel branch).
        BIE_RC_TRY(ensure_side_stream(g));
        BIE_CUDA_TRY(cudaEventRecord(g->ev_fork, st));
        if (ev[1]) BIE_CUDA_TRY(cudaEventRecord(ev[1], st));
        int rc = sym_launch(g, 0, g->sym_U, op, st);
        if (rc) return rc;
        BIE_CUDA_TRY(cudaStreamWaitEvent(g->side, g->ev_fork, 0));
        if (full) {  // the completion moments, read only by the epilogue
            k_moments<<<g->M + 1, 256, 0, g->side>>>(g->pos, g->nrm, g->w, g->pore, sigma_in, stride, nvec, g->M,
                                                       g->n_pore, g->wall_lo, N, g->wall_len, g->moments);
            count_launch();
        }
        if (op)
            k_dlp_diag<1><<<2 * g->sym_nTB * g->sym_dsplit, 128, 0, g->side>>>(g->pos, g->nw, sigma, g->sym_diag, N,
                                                                               0, g->sym_dsplit);
        else
            k_dlp_diag<0><<<2 * g->sym_nTB * g->sym_dsplit, 128, 0, g->side>>>(g->pos, g->nw, sigma, g->sym_diag, N,
                                                                               0, g->sym_dsplit);
        count_launch();
        BIE_CUDA_TRY(cudaGetLastError());
        BIE_CUDA_TRY(cudaEventRecord(g->ev_join, g->side));
        BIE_CUDA_TRY(cudaStreamWaitEvent(st, g->ev_join, 0));
        if (ev[2]) BIE_CUDA_TRY(cudaEventRecord(ev[2], st));
        ea.sym = SymEpi{1, g->sym_acc, g->sym_counter + 1, g->sym_diag, g->sym_dsplit};
    }
    // decompose nvec into variant chunks (16, 8, 4, 2, 1)
    int v = sym ? nvec : 0;
    PairSched sch[5];
    int vis[5];
    int nch = 0;
    size_t need = 0;
    while (v < nvec) {
        int rem = nvec - v;
        int nv = rem >= 16 ? 16 : rem >= 8 ? 8 : rem >= 4 ? 4 : rem >= 2 ? 2 : 1;
        int vi = variant_index(nv);
        PairSched s;
        if (row_begin == 0 && row_end == N)
            s = op ? g->sched_slp[vi] : g->sched[vi];
        else
            make_sched(g, vi, Nt, s, op);
        need = std::max(need, (size_t)s.S * nvec * 2 * (size_t)Nt);
        sch[nch] = s;
        vis[nch] = vi;
        ea.ch[nch] = Chunk{v, nv, s.TB, s.nTS, s.P, s.U, s.Useg};
        ++nch;
        v += nv;
    }
    if (need > g->partial_elems) {
        BIE_CUDA_TRY(cudaStreamSynchronize(st));
        cudaFree(g->partial);
        g->partial = nullptr;
        g->partial_elems = 0;
        BIE_CUDA_TRY(cudaMalloc(&g->partial, need * sizeof(double)));
        g->partial_elems = need;
    }
    if (ev[1] && !sym) BIE_CUDA_TRY(cudaEventRecord(ev[1], st));
    if (nch > 0) BIE_CUDA_TRY(cudaMemsetAsync(g->pair_counter, 0, sizeof(unsigned long long) * nch, st));
    for (int c = 0; c < nch; ++c) {
        PairArgs a;

        a.partial_len = (long long)g->partial_elems;
        a.tpos = g->pos + row_begin;
        a.pos = g->pos;
        a.nw = g->nw;
        a.sigma = sigma + (long long)ea.ch[c].v0 * stride;
        a.sig_stride = stride;
        a.partial = g->partial;
        a.nvec_total = nvec;
        a.v0 = ea.ch[c].v0;
        a.N = N;
        a.row_begin = row_begin;
        a.Nt = Nt;
        a.nTS = sch[c].nTS;
        a.U = sch[c].U;
        a.Useg = sch[c].Useg;
        a.nseg = (a.U + a.Useg - 1) / a.Useg;
        a.counter = g->pair_counter + c;
        launch_pairs(vis[c], sch[c], a, st, op);
        count_launch();
        BIE_CUDA_TRY(cudaGetLastError());
    }
    if (ev[2] && !sym) BIE_CUDA_TRY(cudaEventRecord(ev[2], st));
    ea.pos = g->pos;
    ea.nrm = g->nrm;
    ea.tan = g->tan;
    ea.selfc = g->selfc;
    ea.pore = g->pore;
    ea.sigma = sigma_in;
    ea.sig_stride = stride;
    ea.op = op;
    ea.n_pore = g->n_pore;
    ea.slp_s = g->slp_s;
    for (int k = 0; k < 6; ++k) ea.kr[k] = g->kr[k];
    ea.partial = g->partial;
    ea.moments = g->moments;
    ea.out = out;
    ea.nvec = nvec;
    ea.N = N;
    ea.M = g->M;
    ea.wall_lo = g->wall_lo;
    ea.row_begin = row_begin;
    ea.Nt = Nt;
    ea.flags = flags;
    ea.nchunks = nch;
    if (nvec == 1)
        BIE_LAUNCH(k_epilogue<1>, (Nt + 127) / 128, 128, 0, st, ea);
    else if (nvec == 4)
        BIE_LAUNCH(k_epilogue<4>, (Nt + 127) / 128, 128, 0, st, ea);
    else if (nvec == 16)
        BIE_LAUNCH(k_epilogue<16>, (Nt + 127) / 128, 128, 0, st, ea);
    else
        BIE_LAUNCH(k_epilogue<0>, (Nt + 127) / 128, 128, 0, st, ea);
    count_launch();
    BIE_CUDA_TRY(cudaGetLastError());
    if (ev[3]) BIE_CUDA_TRY(cudaEventRecord(ev[3], st));
    return BIE_OK;
}

// NEXT-2 field evaluation epilogue: fixed-order slot sum + completion field.
__global__ void __launch_bounds__(128) k_field_epilogue(const double2 *__restrict__ tgt, const double *partial,
                                                        int Nt, Chunk ch, const double4 *__restrict__ pore,
                                                        const double *__restrict__ moments, int M, double *out) {
    __shared__ double4 s_pc[128], s_pm[128];
    const int it_raw = blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = it_raw < Nt;
    const int it = active ? it_raw : Nt - 1;
    const double2 xi = tgt[it];
    const int tb = it / ch.TB;
    const int first = (int)seg_of((long long)tb * ch.nTS, 0, ch.Useg);
    const int last = (int)seg_of((long long)(tb + 1) * ch.nTS - 1, 0, ch.Useg);
    double2 u = make_double2(0.0, 0.0);
    for (int sl = 0; sl <= last - first; ++sl) {
        const double2 pv = reinterpret_cast<const double2 *>(partial + (long long)sl * 2LL * Nt)[it];
        u.x += pv.x;
        u.y += pv.y;
    }
    constexpr double k4pi = 1.0 / (4.0 * kPi);
    __shared__ LogTab s_log;  // visible after the first tile barrier
    log_tab_init(s_log, threadIdx.x, blockDim.x);
    for (int k0 = 0; k0 < M; k0 += 128) {
        const int nk = min(128, M - k0);
        __syncthreads();
        if ((int)threadIdx.x < nk) {
            const int k = k0 + threadIdx.x;
            s_pc[threadIdx.x] = pore[k];
            s_pm[threadIdx.x] = make_double4(moments[3 * k], moments[3 * k + 1], moments[3 * k + 2], 0.0);
        }
        __syncthreads();
        for (int q = 0; q < nk; ++q) {
            const double4 pk = s_pc[q], pm = s_pm[q];
            const double rx = xi.x - pk.x, ry = xi.y - pk.y;
            const double rho2 = fma(rx, rx, ry * ry);
            const double ir = 1.0 / rho2;
            const double lg = -neg_half_log_tab(rho2, s_log);  // log rho
            const double rk = pk.z * ir;
            const double rl = (rx * pm.x + ry * pm.y) * ir;
            u.x += k4pi * (-lg * pm.x + rx * rl) + rk * ry * pm.z;
            u.y += k4pi * (-lg * pm.y + ry * rl) - rk * rx * pm.z;
        }
    }
    if (active) reinterpret_cast<double2 *>(out)[it] = u;
}

// ---------------------------------------------------------------------------
// Sharded symmetric path: a rank computes the pair sums of a
// slice [ub, ue) of the triangular unit list plus the in-block pairs of blocks
// [blk0, blk1) into a full-size vector; the ranks' vectors are reduce-scattered
// and each rank finishes its rows with bie_dlp_epilogue_rows.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_sym_gather(const unsigned long long *__restrict__ acc,
                                                    const unsigned long long *__restrict__ qmax,
                                                    const double *__restrict__ diag, int N, int blk0, int blk1,
                                                    double *out, int dsplit) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int B = i / kSymTB;
    double fxs, fxb;
    fx_scales(qmax, fxs, fxb);
    double2 v = make_double2(fx_value(acc + 2LL * i, 2LL * N, fxb), fx_value(acc + 2LL * i + 1, 2LL * N, fxb));
    if (B >= blk0 && B < blk1) {
        for (int q = 0; q < dsplit; ++q) {
            const double2 pv = reinterpret_cast<const double2 *>(diag + (long long)q * 2LL * N)[i];
            v.x += pv.x;
            v.y += pv.y;
        }
    }
    reinterpret_cast<double2 *>(out)[i] = v;
}

int pairs_partial_impl(Geometry *g, const double *sigma, double *out_full, long long ub, long long ue, int blk0,
                       int blk1, cudaStream_t st, int op = 0) {
    int rc = sym_prepare(g);
    if (rc) return rc;
    if (g->sym_state != 1) {
        set_error("bie_dlp_pairs_partial: symmetric path unavailable (memory cap)");
        return BIE_ENOMEM;
    }
    const int N = g->N;
    const long long U = ue - ub;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    if (g->prof) {  // same phase events as dlp_apply_impl (moments slot unused)
        while (g->prof_ev.size() < g->prof_used + 4) {
            cudaEvent_t e;
            BIE_CUDA_TRY(cudaEventCreate(&e));
            g->prof_ev.push_back(e);
        }
        for (int q = 0; q < 4; ++q) ev[q] = g->prof_ev[g->prof_used + q];
        g->prof_used += 4;
        BIE_CUDA_TRY(cudaEventRecord(ev[0], st));
    }
    rc = sym_pre(g, st);
    if (rc) return rc;
    if (op) {  // single layer (NEXT-1): S = w sigma / 4pi and its (S, 0, 0) records
        int rc2 = slp_prepare(g);
        if (rc2) return rc2;
        k_slp_scale<<<(N + 255) / 256, 256, 0, st>>>(g->w, sigma, 2LL * N, 1, N, g->slp_s, g->sym_Q,
                                                     g->sym_counter + 1, g->sym_acc);
    } else {
        k_quad<<<(N + 255) / 256, 256, 0, st>>>(g->nw, sigma, g->sym_Q, N, g->sym_counter + 1, g->sym_acc);
    }
    count_launch();
    if (ev[1]) BIE_CUDA_TRY(cudaEventRecord(ev[1], st));
    rc = sym_launch(g, ub, U, op, st);  // (k_quad / k_slp_scale zeroed the accumulators, even for an empty slice)
    if (rc) return rc;
    if (blk1 > blk0) {
        if (op)
            k_dlp_diag<1><<<2 * (blk1 - blk0) * g->sym_dsplit, 128, 0, st>>>(g->pos, g->nw, g->slp_s, g->sym_diag, N,
                                                                            blk0, g->sym_dsplit);
        else
            k_dlp_diag<0><<<2 * (blk1 - blk0) * g->sym_dsplit, 128, 0, st>>>(g->pos, g->nw, sigma, g->sym_diag, N, blk0,
                                                                            g->sym_dsplit);
        count_launch();
    }
    if (ev[2]) BIE_CUDA_TRY(cudaEventRecord(ev[2], st));
    k_sym_gather<<<(N + 255) / 256, 256, 0, st>>>(g->sym_acc, g->sym_counter + 1, g->sym_diag, N, blk0, blk1,
                                                  out_full, g->sym_dsplit);
    count_launch();
    BIE_CUDA_TRY(cudaGetLastError());
    if (ev[3]) BIE_CUDA_TRY(cudaEventRecord(ev[3], st));
    return BIE_OK;
}

int epilogue_rows_impl(Geometry *g, const double *sigma, const double *presum, double *out, int rb, int re,
                       unsigned flags, cudaStream_t st) {
    const int N = g->N;
    const int Nt = re - rb;
    if (Nt <= 0) return BIE_OK;
    const int op = (flags & kOpSLP) ? 1 : 0;
    if (op) {  // the KR correction needs S = w sigma / 4pi of the neighbours
        int rc = slp_prepare(g);
        if (rc) return rc;
        k_slp_scale<<<(N + 255) / 256, 256, 0, st>>>(g->w, sigma, 2LL * N, 1, N, g->slp_s, nullptr);
        count_launch();
    } else if (!(flags & BIE_D_ONLY)) {
        k_moments<<<g->M + 1, 256, 0, st>>>(g->pos, g->nrm, g->w, g->pore, sigma, 2LL * N, 1, g->M, g->n_pore,
                                            g->wall_lo, N, g->wall_len, g->moments);
        count_launch();
    }
    EpiArgs ea{};
    ea.pos = g->pos;
    ea.nrm = g->nrm;
    ea.tan = g->tan;
    ea.selfc = g->selfc;
    ea.pore = g->pore;
    ea.sigma = sigma;
    ea.sig_stride = 2LL * N;
    ea.partial = nullptr;
    ea.moments = g->moments;
    ea.out = out;
    ea.nvec = 1;
    ea.N = N;
    ea.M = g->M;
    ea.wall_lo = g->wall_lo;
    ea.row_begin = rb;
    ea.Nt = Nt;
    ea.flags = flags;
    ea.nchunks = 0;
    ea.presum = presum;
    ea.op = op;
    ea.n_pore = g->n_pore;
    ea.slp_s = g->slp_s;
    for (int k = 0; k < 6; ++k) ea.kr[k] = g->kr[k];
    k_epilogue<1><<<(Nt + 127) / 128, 128, 0, st>>>(ea);
    count_launch();
    BIE_CUDA_TRY(cudaGetLastError());
    return BIE_OK;
}

int field_eval_impl(Geometry *g, const double *sigma, const double2 *targets, int ntgt, double *out, cudaStream_t st) {
    if (ntgt == 0) return BIE_OK;
    const int N = g->N;
    k_moments<<<g->M + 1, 256, 0, st>>>(g->pos, g->nrm, g->w, g->pore, sigma, 2LL * N, 1, g->M, g->n_pore,
                                        g->wall_lo, N, g->wall_len, g->moments);
    count_launch();
    PairSched s;
    make_sched(g, 0, ntgt, s);
    const size_t need = (size_t)s.S * 2 * (size_t)ntgt;
    if (need > g->partial_elems) {
        BIE_CUDA_TRY(cudaStreamSynchronize(st));
        cudaFree(g->partial);
        g->partial = nullptr;
        g->partial_elems = 0;
        BIE_CUDA_TRY(cudaMalloc(&g->partial, need * sizeof(double)));
        g->partial_elems = need;
    }
    PairArgs a;

    a.partial_len = (long long)g->partial_elems;
    a.tpos = targets;
    a.pos = g->pos;
    a.nw = g->nw;
    a.sigma = sigma;
    a.sig_stride = 2LL * N;
    a.partial = g->partial;
    a.nvec_total = 1;
    a.v0 = 0;
    a.N = N;
    a.row_begin = 0;
    a.Nt = ntgt;
    a.nTS = s.nTS;
    a.U = s.U;
    a.Useg = s.Useg;
    a.nseg = (a.U + a.Useg - 1) / a.Useg;
    a.counter = g->pair_counter;
    BIE_CUDA_TRY(cudaMemsetAsync(g->pair_counter, 0, sizeof(unsigned long long), st));
    launch_pairs(0, s, a, st);
    count_launch();
    k_field_epilogue<<<(ntgt + 127) / 128, 128, 0, st>>>(targets, g->partial, ntgt, Chunk{0, 1, s.TB, s.nTS, s.P, s.U, s.Useg},
                                                         g->pore, g->moments, g->M, out);
    count_launch();
    BIE_CUDA_TRY(cudaGetLastError());
    return BIE_OK;
}

}  // namespace bie

using namespace bie;

extern "C" {

// NEXT-1 field evaluation with the single-layer density: the plain trapezoid
// sum of P:l.346-354 (eq. stokesSLP_discretized), no correction.
int slp_field_eval_impl(Geometry *g, const double *sigma, const double2 *targets, int ntgt, double *out,
                        cudaStream_t st) {
    if (ntgt == 0) return BIE_OK;
    const int N = g->N;
    int rc = slp_prepare(g);
    if (rc != BIE_OK) return rc;
    k_slp_scale<<<(N + 255) / 256, 256, 0, st>>>(g->w, sigma, 2LL * N, 1, N, g->slp_s, nullptr);
    count_launch();
    PairSched s;
    make_sched(g, 0, ntgt, s, 1);
    const size_t need = (size_t)s.S * 2 * (size_t)ntgt;
    if (need > g->partial_elems) {
        BIE_CUDA_TRY(cudaStreamSynchronize(st));
        cudaFree(g->partial);
        g->partial = nullptr;
        g->partial_elems = 0;
        BIE_CUDA_TRY(cudaMalloc(&g->partial, need * sizeof(double)));
        g->partial_elems = need;
    }
    PairArgs a;

    a.partial_len = (long long)g->partial_elems;
    a.tpos = targets;
    a.pos = g->pos;
    a.nw = g->nw;
    a.sigma = g->slp_s;
    a.sig_stride = 2LL * N;
    a.partial = g->partial;
    a.nvec_total = 1;
    a.v0 = 0;
    a.N = N;
    a.row_begin = 0;
    a.Nt = ntgt;
    a.nTS = s.nTS;
    a.U = s.U;
    a.Useg = s.Useg;
    a.nseg = (a.U + a.Useg - 1) / a.Useg;
    a.counter = g->pair_counter;
    BIE_CUDA_TRY(cudaMemsetAsync(g->pair_counter, 0, sizeof(unsigned long long), st));
    launch_pairs(0, s, a, st, 1);
    count_launch();
    k_field_epilogue<<<(ntgt + 127) / 128, 128, 0, st>>>(targets, g->partial, ntgt, Chunk{0, 1, s.TB, s.nTS, s.P, s.U, s.Useg},
                                                         nullptr, nullptr, 0, out);
    count_launch();
    BIE_CUDA_TRY(cudaGetLastError());
    return BIE_OK;
}

static int check_apply_args(Geometry *g, const double *sigma, double *out, int nvec, unsigned flags, const char *fn) {
    if (!g) {
        set_error(std::string(fn) + ": invalid geometry handle");
        return BIE_EINVAL;
    }
    if (!sigma || !out) {
        set_error(std::string(fn) + ": null sigma/out");
        return BIE_EINVAL;
    }
    if (nvec < 1 || nvec > BIE_MAX_NVEC) {
        set_error(std::string(fn) + ": nvec must be in [1, 16]");
        return BIE_EINVAL;
    }
    if (flags & ~(BIE_D_ONLY | BIE_ONE_SIDED)) {
        set_error(std::string(fn) + ": unknown flags");
        return BIE_EINVAL;
    }
    if ((const void *)sigma == (const void *)out) {
        /* aliasing */
        set_error(std::string(fn) + ": out must not alias sigma");
        return BIE_EINVAL;
    }
    return BIE_OK;
}

int bie_dlp_apply(bie_geometry_t gh, const double *sigma, double *out, int nvec, unsigned flags, void *stream) {
    Geometry *g = as_geom(gh);
    int rc = check_apply_args(g, sigma, out, nvec, flags, "bie_dlp_apply");
    if (rc) return rc;
    return dlp_apply_impl(g, sigma, out, nvec, flags, 0, g->N, (cudaStream_t)stream);
}

int bie_dlp_apply_rows(bie_geometry_t gh, const double *sigma, double *out, int nvec, unsigned flags, int row_begin,
                       int row_end, void *stream) {
    Geometry *g = as_geom(gh);
    int rc = check_apply_args(g, sigma, out, nvec, flags, "bie_dlp_apply_rows");
    if (rc) return rc;
    if (row_begin < 0 || row_end > g->N || row_begin > row_end) {
        set_error("bie_dlp_apply_rows: row range out of [0, N]");
        return BIE_EINVAL;
    }
    return dlp_apply_impl(g, sigma, out, nvec, flags, row_begin, row_end, (cudaStream_t)stream);
}

int bie_dlp_sym_info(bie_geometry_t gh, long long *units, int *blocks) {
    Geometry *g = as_geom(gh);
    if (!g || !units || !blocks) {
        set_error("bie_dlp_sym_info: invalid handle or null output");
        return BIE_EINVAL;
    }
    int rc = sym_prepare(g);
    if (rc) return rc;
    if (g->sym_state != 1) {
        set_error("bie_dlp_sym_info: symmetric path unavailable (memory cap)");
        return BIE_ENOMEM;
    }
    *units = g->sym_U;
    *blocks = g->sym_nTB;
    return BIE_OK;
}

int bie_dlp_pairs_partial(bie_geometry_t gh, const double *sigma, double *out_full, long long unit_begin,
                          long long unit_end, int block_begin, int block_end, void *stream) {
    Geometry *g = as_geom(gh);
    if (!g || !sigma || !out_full || sigma == out_full) {
        set_error("bie_dlp_pairs_partial: invalid handle, null pointer or aliasing");
        return BIE_EINVAL;
    }
    int rc = sym_prepare(g);
    if (rc) return rc;
    if (unit_begin < 0 || unit_end > g->sym_U || unit_begin > unit_end || block_begin < 0 ||
        block_end > g->sym_nTB || block_begin > block_end) {
        set_error("bie_dlp_pairs_partial: unit or block range out of bounds (see bie_dlp_sym_info)");
        return BIE_EINVAL;
    }
    return pairs_partial_impl(g, sigma, out_full, unit_begin, unit_end, block_begin, block_end, (cudaStream_t)stream);
}

int bie_slp_pairs_partial(bie_geometry_t gh, const double *sigma, double *out_full, long long unit_begin,
                          long long unit_end, int block_begin, int block_end, void *stream) {
    Geometry *g = as_geom(gh);
    if (!g || !sigma || !out_full || sigma == out_full) {
        set_error("bie_slp_pairs_partial: invalid handle, null pointer or aliasing");
        return BIE_EINVAL;
    }
    int rc = sym_prepare(g);
    if (rc) return rc;
    if (unit_begin < 0 || unit_end > g->sym_U || unit_begin > unit_end || block_begin < 0 ||
        block_end > g->sym_nTB || block_begin > block_end) {
        set_error("bie_slp_pairs_partial: unit or block range out of bounds (see bie_dlp_sym_info)");
        return BIE_EINVAL;
    }
    return pairs_partial_impl(g, sigma, out_full, unit_begin, unit_end, block_begin, block_end, (cudaStream_t)stream,
                              1);
}

int bie_slp_epilogue_rows(bie_geometry_t gh, const double *sigma, const double *pairsum_rows, double *out_rows,
                          int row_begin, int row_end, void *stream) {
    Geometry *g = as_geom(gh);
    if (!g || !sigma || !pairsum_rows || !out_rows || row_begin < 0 || row_end > g->N || row_begin > row_end) {
        set_error("bie_slp_epilogue_rows: invalid handle, pointer or row range");
        return BIE_EINVAL;
    }
    return epilogue_rows_impl(g, sigma, pairsum_rows, out_rows, row_begin, row_end, kOpSLP, (cudaStream_t)stream);
}

int bie_dlp_epilogue_rows(bie_geometry_t gh, const double *sigma, const double *pairsum_rows, double *out_rows,
                          int row_begin, int row_end, unsigned flags, void *stream) {
    Geometry *g = as_geom(gh);
    if (!g || !sigma || !pairsum_rows || !out_rows || (flags & ~BIE_D_ONLY) || row_begin < 0 || row_end > g->N ||
        row_begin > row_end) {
        set_error("bie_dlp_epilogue_rows: invalid handle, pointer, flags or row range");
        return BIE_EINVAL;
    }
    return epilogue_rows_impl(g, sigma, pairsum_rows, out_rows, row_begin, row_end, flags, (cudaStream_t)stream);
}

int bie_slp_apply(bie_geometry_t gh, const double *sigma, double *out, int nvec, unsigned flags, void *stream) {
    Geometry *g = as_geom(gh);
    int rc = check_apply_args(g, sigma, out, nvec, flags, "bie_slp_apply");
    if (rc) return rc;
    if (flags & BIE_D_ONLY) {
        set_error("bie_slp_apply: BIE_D_ONLY does not apply to the single-layer operator");
        return BIE_EINVAL;
    }
    return dlp_apply_impl(g, sigma, out, nvec, flags | kOpSLP, 0, g->N, (cudaStream_t)stream);
}

int bie_slp_apply_rows(bie_geometry_t gh, const double *sigma, double *out, int nvec, int row_begin, int row_end,
                       void *stream) {
    Geometry *g = as_geom(gh);
    int rc = check_apply_args(g, sigma, out, nvec, 0u, "bie_slp_apply_rows");
    if (rc) return rc;
    if (row_begin < 0 || row_end > g->N || row_begin > row_end) {
        set_error("bie_slp_apply_rows: row range out of [0, N]");
        return BIE_EINVAL;
    }
    return dlp_apply_impl(g, sigma, out, nvec, kOpSLP, row_begin, row_end, (cudaStream_t)stream);
}

int bie_slp_field_eval(bie_geometry_t gh, const double *sigma, const double *targets, int ntgt, double *out,
                       void *stream) {
    Geometry *g = as_geom(gh);
    if (!g || !sigma || (ntgt > 0 && (!targets || !out)) || ntgt < 0 || (const void *)out == (const void *)sigma) {
        set_error("bie_slp_field_eval: invalid handle, null pointer, ntgt < 0 or out aliasing sigma");
        return BIE_EINVAL;
    }
    return slp_field_eval_impl(g, sigma, reinterpret_cast<const double2 *>(targets), ntgt, out,
                               (cudaStream_t)stream);
}

int bie_field_eval(bie_geometry_t gh, const double *sigma, const double *targets, int ntgt, double *out,
                   void *stream) {
    Geometry *g = as_geom(gh);
    if (!g || !sigma || (ntgt > 0 && (!targets || !out)) || ntgt < 0 || (const void *)out == (const void *)sigma) {
        set_error("bie_field_eval: invalid handle, null pointer, ntgt < 0 or out aliasing sigma");
        return BIE_EINVAL;
    }
    return field_eval_impl(g, sigma, reinterpret_cast<const double2 *>(targets), ntgt, out, (cudaStream_t)stream);
}

int bie_dlp_apply_host(bie_geometry_t gh, const double *sigma_host, double *out_host, int nvec, unsigned flags,
                       void *stream) {
    Geometry *g = as_geom(gh);
    int rc = check_apply_args(g, sigma_host, out_host, nvec, flags, "bie_dlp_apply_host");
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    size_t bytes = sizeof(double) * 2 * (size_t)g->N * nvec;
    BIE_CUDA_TRY(cudaMemcpyAsync(g->stage_in, sigma_host, bytes, cudaMemcpyHostToDevice, st));
    rc = dlp_apply_impl(g, g->stage_in, g->stage_out, nvec, flags, 0, g->N, st);
    if (rc) return rc;
    BIE_CUDA_TRY(cudaMemcpyAsync(out_host, g->stage_out, bytes, cudaMemcpyDeviceToHost, st));
    BIE_CUDA_TRY(cudaStreamSynchronize(st));
    return BIE_OK;
}

}  // extern "C"

BIE_DCHECK_TU(dlp)
