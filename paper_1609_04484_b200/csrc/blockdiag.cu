// blockdiag.cu -- block-diagonal preconditioner (A6 factor, A7 apply).
//
// P:l.651-657: "a block-diagonal preconditioner (with the diagonal blocks
// corresponding to the self-interactions of the individual pores and the
// outer boundary) ... The diagonal blocks are assembled, factorized, and
// inverted exactly."  Block b = rows/cols of the completed operator on body b.
//
// Factor: every block is inverted in place by blocked Gauss-Jordan elimination
// with partial pivoting.  For a panel K of NB columns:
//   1. k_panel    : LU with partial pivoting of the panel rows >= k0 (one CTA per
//                   matrix) -> pivots; A11^{-1} from L11 U11.
//   2. k_swap     : apply the panel's row swaps to the whole matrix.
//   3. k_copy_T   : T = M[:, K];   k_make_G : G = A11^{-1} M[K, :], G[:, K] = A11^{-1}
//   4. k_update3  : M[i, :] = (i in K) ? G[i-k0, :] : base(i, :) - T[i, :] G
//                   (base = M off K, 0 on K)  -- the rank-NB sweep on the FP64 tensor cores (DMMA).
// Large single blocks (the wall, order >= 4096): super-panels of kSB = 4 NB columns with
// the delayed rank-kSB update of the columns outside the slab (k_make_Y,
// k_update_agg_async: cp.async double-buffered DMMA tiles) and a lookahead schedule:
// the next super-panel's cooperative panel LUs (k_panel_coop) run on a high-priority
// stream beside the sweep of the current one (k_swap_rng applies a super-panel's row
// swaps to the outside columns afterwards).  DESIGN.md s5.
// After the last panel, columns are unpermuted (A^{-1} = M P).  Batched over
// all blocks of one size class (pores share one size; Gamma_0 is its own class).
// Apply: one warp per row of the explicit inverses (HBM-bound batched GEMV).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include "internal.cuh"

namespace cg = cooperative_groups;

namespace bie {

constexpr int NB = 32;  // panel width
constexpr int kSB = 4 * NB;  // super-panel of the delayed update (large single blocks)

struct BDView {            // one size class
    double *mat;           // first matrix
    long long mstride;     // doubles between consecutive matrices
    int n2;                // matrix order
    int count;             // matrices in the class
    int body0;             // body index of the first matrix
};

struct BDScratch {
    double *W;      // [count][n2][NB]   panel LU workspace
    double *T;      // [count][n2][NB]
    double *G;      // [count][NB][n2]
    double *A11i;   // [count][NB][NB]
    int *piv;       // [count][n2]
    int *flag;      // [count]
};

// ------------------------------------------------------------------ assembly
// Entry (2x2 node block) for nodes i, j of body b (same formula as the operator):
//   i != j : c r r^T with c = (r . nw_j)/rho^4          (DLP, P:l.243-248)
//   i == j : selfc_i t t^T - 1/2 I                      (C4, C3)
//   pore k : + (w_j/|Gamma_k|) [S(x_i - c_k) + R(x_i - c_k) ((x_j - c_k)^perp)^T]   (C5)
//   wall   : + n_i n_j^T w_j / |Gamma_0|                (C5, N0)
__global__ void k_bd_assemble(BDView v, int lo0, int nodes, int is_wall, const double2 *__restrict__ pos,
                              const double2 *__restrict__ nw, const double2 *__restrict__ nrm,
                              const double2 *__restrict__ tan, const double *__restrict__ w,
                              const double *__restrict__ selfc, const double4 *__restrict__ pore, double wall_len) {
    const int m = blockIdx.y;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)nodes * nodes) return;
    const int li = (int)(e / nodes), lj = (int)(e % nodes);
    const int lo = lo0 + m * nodes;
    const int i = lo + li, j = lo + lj;
    double e00, e01, e10, e11;
    const double2 xi = pos[i], xj = pos[j];
    if (i != j) {
        const double rx = xi.x - xj.x, ry = xi.y - xj.y;
        const double rho2 = rx * rx + ry * ry;
        const double2 nj = nw[j];
        const double c = (rx * nj.x + ry * nj.y) / (rho2 * rho2);
        e00 = c * rx * rx;
        e01 = c * rx * ry;
        e10 = e01;
        e11 = c * ry * ry;
    } else {
        const double2 t = tan[i];
        const double a = selfc[i];
        e00 = a * t.x * t.x - 0.5;
        e01 = a * t.x * t.y;
        e10 = e01;
        e11 = a * t.y * t.y - 0.5;
    }
    if (!is_wall) {
        const double4 pk = pore[v.body0 + m];
        const double rx = xi.x - pk.x, ry = xi.y - pk.y;
        const double rho2 = rx * rx + ry * ry;
        const double lg = 0.5 * log(rho2);
        const double f = w[j] / pk.w;
        constexpr double k4pi = 1.0 / (4.0 * kPi);
        const double s00 = k4pi * (-lg + rx * rx / rho2);
        const double s01 = k4pi * (rx * ry / rho2);
        const double s11 = k4pi * (-lg + ry * ry / rho2);
        const double Rx = ry / rho2, Ry = -rx / rho2;
        const double qx = xj.y - pk.y, qy = -(xj.x - pk.x);
        e00 += f * (s00 + Rx * qx);
        e01 += f * (s01 + Rx * qy);
        e10 += f * (s01 + Ry * qx);
        e11 += f * (s11 + Ry * qy);
    } else {
        const double f = w[j] / wall_len;
        const double2 ni = nrm[i], nj = nrm[j];
        e00 += f * ni.x * nj.x;
        e01 += f * ni.x * nj.y;
        e10 += f * ni.y * nj.x;
        e11 += f * ni.y * nj.y;
    }
    double *M = v.mat + (long long)m * v.mstride;
    const long long n2 = v.n2;
    M[(2LL * li) * n2 + 2 * lj] = e00;
    M[(2LL * li) * n2 + 2 * lj + 1] = e01;
    M[(2LL * li + 1) * n2 + 2 * lj] = e10;
    M[(2LL * li + 1) * n2 + 2 * lj + 1] = e11;
}

// SLP blocks (NEXT-1; reading C25): node pair (i, j) of one closed curve of
// `nodes` nodes carries W_ij G(x_i, x_j) with G = (1/4pi)(-log rho I + r r^T/rho^2),
// W_ii = 0, W_ij = w_j (1 + gamma_k) at periodic offset +-k (k <= 6), else w_j.
struct KRWeights {
    double g[6];
};
__global__ void k_bd_assemble_slp(BDView v, int lo0, int nodes, const double2 *__restrict__ pos,
                                  const double *__restrict__ w, KRWeights kr) {
    const int m = blockIdx.y;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)nodes * nodes) return;
    const int li = (int)(e / nodes), lj = (int)(e % nodes);
    const int lo = lo0 + m * nodes;
    double e00 = 0.0, e01 = 0.0, e11 = 0.0;
    if (li != lj) {
        int d = lj - li;
        d = d < 0 ? d + nodes : d;
        const int k = min(d, nodes - d);
        double W = w[lo + lj];
        if (k <= 6) W *= 1.0 + kr.g[k - 1];
        const double2 xi = pos[lo + li], xj = pos[lo + lj];
        const double rx = xi.x - xj.x, ry = xi.y - xj.y;
        const double rho2 = rx * rx + ry * ry;
        const double lg = 0.5 * log(rho2);
        const double f = W * (1.0 / (4.0 * kPi));
        e00 = f * (-lg + rx * rx / rho2);
        e01 = f * (rx * ry / rho2);
        e11 = f * (-lg + ry * ry / rho2);
    }
    double *M = v.mat + (long long)m * v.mstride;
    const long long n2 = v.n2;
    M[(2LL * li) * n2 + 2 * lj] = e00;
    M[(2LL * li) * n2 + 2 * lj + 1] = e01;
    M[(2LL * li + 1) * n2 + 2 * lj] = e01;
    M[(2LL * li + 1) * n2 + 2 * lj + 1] = e11;
}

// ------------------------------------------------------------------ panel LU
// One CTA per matrix.  Rows [k0, n2) of panel columns [k0, k0+nbe).
// Pivot = max |value|, lowest row index on ties (as the oracle).
__global__ void __launch_bounds__(1024) k_panel(BDView v, BDScratch s, int k0, int nbe) {
    const int m = blockIdx.x;
    const int n2 = v.n2;
    const double *M = v.mat + (long long)m * v.mstride;
    // W column-major: W[c * n2 + r] (coalesced over rows r)
    double *W = s.W + (long long)m * n2 * NB;
#define WI(r, c) ((long long)(c) * n2 + (r))
    int *piv = s.piv + (long long)m * n2;
    __shared__ double red_v[32];
    __shared__ int red_i[32];
    __shared__ int s_p;
    __shared__ double s_d;
    __shared__ double s_row[NB];
    __shared__ double L11[NB][NB + 1], U11[NB][NB + 1];
    const int tid = threadIdx.x, nt = blockDim.x;
    for (long long q = tid; q < (long long)(n2 - k0) * nbe; q += nt) {
        int r = k0 + (int)(q / nbe), c = (int)(q % nbe);
        W[WI(r, c)] = M[(long long)r * n2 + k0 + c];
    }
    __syncthreads();
    for (int c = 0; c < nbe; ++c) {
        const int k = k0 + c;
        double best = -1.0;
        int bi = n2;
        for (int r = k + tid; r < n2; r += nt) {
            double a = fabs(W[WI(r, c)]);
            if (a > best) { best = a; bi = r; }
        }
        // warp argmax (lowest index on ties)
        for (int o = 16; o > 0; o >>= 1) {
            double ob = __shfl_down_sync(0xffffffffu, best, o);
            int oi = __shfl_down_sync(0xffffffffu, bi, o);
            if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        if ((tid & 31) == 0) { red_v[tid >> 5] = best; red_i[tid >> 5] = bi; }
        __syncthreads();
        if (tid < 32) {
            int nw = (nt + 31) >> 5;
            best = tid < nw ? red_v[tid] : -1.0;
            bi = tid < nw ? red_i[tid] : n2;
            for (int o = 16; o > 0; o >>= 1) {
                double ob = __shfl_down_sync(0xffffffffu, best, o);
                int oi = __shfl_down_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
            }
            if (tid == 0) {
                if (!(best > 0.0) || bi >= n2) {
                    s.flag[m] = 1;
                    bi = k;
                }
                s_p = bi;
                piv[k] = bi;
            }
        }
        __syncthreads();
        const int p = s_p;
        if (tid < nbe) {
            double t = W[WI(k, tid)];
            if (p != k) {
                double o = W[WI(p, tid)];
                W[WI(k, tid)] = o;
                W[WI(p, tid)] = t;
                t = o;
            }
            s_row[tid] = t;  // pivot row after the swap
        }
        __syncthreads();
        if (tid == 0) {
            double d = s_row[c];
            s_d = (d != 0.0) ? d : 1.0;
        }
        __syncthreads();
        const double d = s_d;
        // L column and trailing panel update, one thread per row below k
        for (int r = k + 1 + tid; r < n2; r += nt) {
            const double l = W[WI(r, c)] / d;
            W[WI(r, c)] = l;
            for (int cc = c + 1; cc < nbe; ++cc) W[WI(r, cc)] -= l * s_row[cc];
        }
        __syncthreads();
    }
    // A11 = L11 U11 (rows k0..k0+nbe); A11^{-1} by solving A11 X = I (column per thread)
    for (int q = tid; q < nbe * nbe; q += nt) {
        int r = q / nbe, c = q % nbe;
        double val = W[WI(k0 + r, c)];
        L11[r][c] = (c < r) ? val : (c == r ? 1.0 : 0.0);
        U11[r][c] = (c >= r) ? val : 0.0;
    }
    __syncthreads();
    if (tid < nbe) {
        const int col = tid;
        double z[NB];
        for (int r = 0; r < nbe; ++r) {
            double acc = (r == col) ? 1.0 : 0.0;
            for (int q = 0; q < r; ++q) acc -= L11[r][q] * z[q];
            z[r] = acc;
        }
        for (int r = nbe - 1; r >= 0; --r) {
            double acc = z[r];
            for (int q = r + 1; q < nbe; ++q) acc -= U11[r][q] * z[q];
            z[r] = acc / U11[r][r];
        }
        // note: the panel rows were permuted inside W; A11 here is P_panel * M[K, K]
        double *Ai = s.A11i + (long long)m * NB * NB;
        for (int r = 0; r < nbe; ++r) Ai[r * NB + col] = z[r];
    }
#undef WI
}

// Shared helper: A11^{-1} (nbe x nbe) from the LU'd pivot rows A (row-major,
// stride NB: strict lower = L (unit diagonal), upper = U), one thread per column.
__device__ void a11_inverse(const double *A, int nbe, double *Ai) {
    const int col = threadIdx.x;
    if (col >= nbe) return;
    double z[NB];
#pragma unroll
    for (int r = 0; r < NB; ++r) {
        if (r < nbe) {
            double acc = (r == col) ? 1.0 : 0.0;
            for (int q = 0; q < r; ++q) acc -= A[r * NB + q] * z[q];
            z[r] = acc;
        }
    }
#pragma unroll
    for (int r = NB - 1; r >= 0; --r) {
        if (r < nbe) {
            double acc = z[r];
            for (int q = r + 1; q < nbe; ++q) acc -= A[r * NB + q] * z[q];
            z[r] = acc / A[r * NB + r];
        }
    }
#pragma unroll
    for (int r = 0; r < NB; ++r)
        if (r < nbe) Ai[r * NB + col] = z[r];
}

// Small matrices (rows n2 - k0 <= kSmemPanelRows): the panel LU runs entirely in
// shared memory (column-major, rows k0..n2-1), one CTA per matrix.
constexpr int kSmemPanelRows = 768;
__global__ void __launch_bounds__(256) k_panel_smem(BDView v, BDScratch s, int k0, int nbe) {
    extern __shared__ double Ws[];  // [NB][R]
    __shared__ double red_v[8];
    __shared__ int red_i[8];
    __shared__ int s_p;
    __shared__ double s_row[NB];
    __shared__ double s_A[NB * NB];
    const int m = blockIdx.x;
    const int n2 = v.n2;
    const int R = n2 - k0;
    const double *M = v.mat + (long long)m * v.mstride;
    int *piv = s.piv + (long long)m * n2;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int q = tid; q < R * nbe; q += nt) {
        const int r = q / nbe, c = q % nbe;
        Ws[c * R + r] = M[(long long)(k0 + r) * n2 + k0 + c];
    }
    __syncthreads();
    for (int c = 0; c < nbe; ++c) {
        double best = -1.0;
        int bi = R;
        for (int r = c + tid; r < R; r += nt) {
            const double a = fabs(Ws[c * R + r]);
            if (a > best) { best = a; bi = r; }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_down_sync(0xffffffffu, best, o);
            const int oi = __shfl_down_sync(0xffffffffu, bi, o);
            if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        if ((tid & 31) == 0) { red_v[tid >> 5] = best; red_i[tid >> 5] = bi; }
        __syncthreads();
        if (tid == 0) {
            best = red_v[0];
            bi = red_i[0];
            for (int q = 1; q < nt / 32; ++q)
                if (red_v[q] > best || (red_v[q] == best && red_i[q] < bi)) { best = red_v[q]; bi = red_i[q]; }
            if (!(best > 0.0) || bi >= R) {
                s.flag[m] = 1;
                bi = c;
            }
            s_p = bi;
            piv[k0 + c] = k0 + bi;
        }
        __syncthreads();
        const int p = s_p;
        if (tid < nbe) {
            double t = Ws[tid * R + c];
            if (p != c) {
                const double o = Ws[tid * R + p];
                Ws[tid * R + c] = o;
                Ws[tid * R + p] = t;
                t = o;
            }
            s_row[tid] = t;
        }
        __syncthreads();
        const double d = s_row[c] != 0.0 ? s_row[c] : 1.0;
        for (int r = c + 1 + tid; r < R; r += nt) {
            const double l = Ws[c * R + r] / d;
            Ws[c * R + r] = l;
            for (int cc = c + 1; cc < nbe; ++cc) Ws[cc * R + r] -= l * s_row[cc];
        }
        __syncthreads();
    }
    for (int q = tid; q < nbe * nbe; q += nt) s_A[(q / nbe) * NB + (q % nbe)] = Ws[(q % nbe) * R + q / nbe];
    __syncthreads();
    a11_inverse(s_A, nbe, s.A11i + (long long)m * NB * NB);
}

// Large matrix: cooperative panel LU over G CTAs of 128 threads; thread owns one
// panel row in registers.  One grid sync per column: before it every CTA publishes
// its local argmax AND that candidate's whole row, and the owner of row k publishes
// row k; after it every CTA picks the global pivot and reads the pivot row straight
// from the winning CTA's slot.  All exchange buffers are double-buffered by column
// parity: a CTA can only overwrite parity c&1 again after passing column c+1's sync,
// which every CTA reaches only after finishing its reads of column c.
struct CoopScratch {
    double *cand_v;  // [2][G]
    int *cand_i;     // [2][G]
    double *crow;    // [2][G][NB] candidate rows
    double *kbuf;    // [2][NB] row k before the swap
    double *A;       // [NB][NB] LU'd pivot rows
};
// RPT rows per thread: fewer CTAs make the per-column grid barrier cheaper.
template <int RPT>
__global__ void __launch_bounds__(128, RPT == 1 ? 4 : 2) k_panel_coop(BDView v, BDScratch s, CoopScratch cs, int k0, int nbe) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double red_v[4];
    __shared__ int red_i[4];
    __shared__ int s_p, s_src, s_bi;
    __shared__ double s_pr[NB];  // the pivot row, staged once per CTA and column
    __shared__ double s_kb[NB];  // row k before the swap (what the pivot row's owner receives)
    const int n2 = v.n2;
    const double *M = v.mat;  // one matrix per class launch
    const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x;
    int rr[RPT];
    bool own[RPT];
    double w[RPT][NB];
#pragma unroll
    for (int t = 0; t < RPT; ++t) {
        rr[t] = k0 + g * 128 * RPT + t * 128 + tid;  // this thread's panel rows
        own[t] = rr[t] < n2;
#pragma unroll
        for (int c = 0; c < NB; ++c) w[t][c] = (own[t] && c < nbe) ? M[(long long)rr[t] * n2 + k0 + c] : 0.0;
    }
#pragma unroll 1
    for (int c = 0; c < nbe; ++c) {
        const int k = k0 + c, par = c & 1;
        double *cv_ = cs.cand_v + par * G;
        int *ci_ = cs.cand_i + par * G;
        double *crow = cs.crow + (long long)par * G * NB;
        double *kb = cs.kbuf + par * NB;
        double best = -1.0;
        int bi = n2;
#pragma unroll
        for (int t = 0; t < RPT; ++t) {
            double wc = 0.0;
#pragma unroll
            for (int q = 0; q < NB; ++q)
                if (q == c) wc = w[t][q];
            const double b = (own[t] && rr[t] >= k) ? fabs(wc) : -1.0;
            const int ix = (own[t] && rr[t] >= k) ? rr[t] : n2;
            if (b > best || (b == best && ix < bi)) { best = b; bi = ix; }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_down_sync(0xffffffffu, best, o);
            const int oi = __shfl_down_sync(0xffffffffu, bi, o);
            if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        if ((tid & 31) == 0) { red_v[tid >> 5] = best; red_i[tid >> 5] = bi; }
        __syncthreads();
        if (tid == 0) {
            best = red_v[0];
            bi = red_i[0];
            for (int q = 1; q < 4; ++q)
                if (red_v[q] > best || (red_v[q] == best && red_i[q] < bi)) { best = red_v[q]; bi = red_i[q]; }
            cv_[g] = best;
            ci_[g] = bi;
            s_bi = bi;
        }
        __syncthreads();
#pragma unroll
        for (int t = 0; t < RPT; ++t) {
            if (own[t] && rr[t] == s_bi) {
#pragma unroll
                for (int q = 0; q < NB; ++q) crow[(long long)g * NB + q] = w[t][q];
            }
            if (own[t] && rr[t] == k) {
#pragma unroll
                for (int q = 0; q < NB; ++q) kb[q] = w[t][q];
            }
        }
        grid.sync();
        int src = -1;
        if (tid < 32) {
            // warp 0 reduces the G candidates: lanes load in parallel (one L2
            // round trip instead of G serial ones), then a shuffle tree
            best = -1.0;
            bi = n2;
            for (int q = tid; q < G; q += 32) {
                const double cv = __ldcg(cv_ + q);
                const int ci = __ldcg(ci_ + q);
                if (cv > best || (cv == best && ci < bi)) { best = cv; bi = ci; src = q; }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_down_sync(0xffffffffu, best, o);
                const int oi = __shfl_down_sync(0xffffffffu, bi, o);
                const int os = __shfl_down_sync(0xffffffffu, src, o);
                if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; src = os; }
            }
        }
        if (tid == 0) {
            if (!(best > 0.0) || bi >= n2) {
                if (g == 0) s.flag[0] = 1;
                bi = k;
                src = -1;  // no usable pivot: keep row k (read back from kbuf)
            }
            s_p = bi;
            s_src = src;
            if (g == 0) s.piv[k] = bi;
        }
        __syncthreads();
        const int p = s_p;
        // the pivot row and row k (before the swap) staged once per CTA: both L2 reads in flight together
        if (tid < NB) s_pr[tid] = (s_src >= 0 ? crow + (long long)s_src * NB : kb)[tid];
        else if (tid < 2 * NB) s_kb[tid - NB] = kb[tid - NB];
        __syncthreads();
        const double *pr = s_pr;
        double dd = pr[c];
        if (dd == 0.0) dd = 1.0;
#pragma unroll
        for (int t = 0; t < RPT; ++t) {
            if (own[t] && rr[t] == k) {
#pragma unroll
                for (int q = 0; q < NB; ++q) w[t][q] = pr[q];
            } else if (own[t] && rr[t] == p) {
#pragma unroll
                for (int q = 0; q < NB; ++q) w[t][q] = s_kb[q];
            }
            if (own[t] && rr[t] > k) {
                // ONE division per row and column (round 2 had it inside the unrolled
                // select loop: 32 predicated divisions, ~800 DFMA and half the column's time)
                double wc = 0.0;
#pragma unroll
                for (int q = 0; q < NB; ++q)
                    if (q == c) wc = w[t][q];
                const double l = wc / dd;
#pragma unroll
                for (int q = 0; q < NB; ++q) {
                    if (q == c) w[t][q] = l;
                    if (q > c && q < nbe) w[t][q] -= l * pr[q];
                }
            }
        }
    }
#pragma unroll
    for (int t = 0; t < RPT; ++t) {
        if (own[t] && rr[t] < k0 + nbe) {
#pragma unroll
            for (int q = 0; q < NB; ++q) cs.A[(rr[t] - k0) * NB + q] = w[t][q];
        }
    }
    grid.sync();
    if (g == 0) a11_inverse(cs.A, nbe, s.A11i);
}

// Apply the panel's row swaps to all columns of M (sequential in k, parallel over columns).
__global__ void k_swap(BDView v, BDScratch s, int k0, int nbe, double *TS = nullptr, int tsw = 0) {
    const int m = blockIdx.y;
    const int col = blockIdx.x * blockDim.x + threadIdx.x;
    const int n2 = v.n2;
    if (col >= n2 + tsw) return;
    // columns >= n2: the first tsw columns of TS ([n2][kSB]), the T-hat columns of
    // the earlier sub-panels of the current super-panel, whose rows follow M's
    double *base = col < n2 ? v.mat + (long long)m * v.mstride + col : TS + (col - n2);
    const long long ld = col < n2 ? n2 : kSB;
    const int *piv = s.piv + (long long)m * n2;
    for (int c = 0; c < nbe; ++c) {
        int k = k0 + c, p = piv[k];
        if (p != k) {
            double t = base[(long long)k * ld];
            base[(long long)k * ld] = base[(long long)p * ld];
            base[(long long)p * ld] = t;
        }
    }
}

// k_swap over a column subset (the lookahead schedule of the delayed update):
// M columns [c0, c1) except [skip0, skip1), then the first tsw columns of TS.
// Swaps of different columns are independent, so a super-panel's nk swaps may
// reach the columns outside its slab later, in one launch, in the same order.
__global__ void k_swap_rng(BDView v, BDScratch s, int k0, int nk, int c0, int c1, int skip0, int skip1,
                           double *TS, int tsw) {
    const int n2 = v.n2;
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    double *base;
    long long ld;
    if (t < c1 - c0) {
        const int col = c0 + t;
        if (col >= skip0 && col < skip1) return;
        base = v.mat + col;
        ld = n2;
    } else {
        t -= c1 - c0;
        if (t >= tsw) return;
        base = TS + t;
        ld = kSB;
    }
    const int *piv = s.piv;
    for (int c = 0; c < nk; ++c) {
        const int k = k0 + c, p = piv[k];
        if (p != k) {
            const double x = base[(long long)k * ld];
            base[(long long)k * ld] = base[(long long)p * ld];
            base[(long long)p * ld] = x;
        }
    }
}

// T = M[:, K]; with TS: also T-hat = T - E_K (identity on the pivot rows K)
// into columns [tcol, tcol + NB) of TS -- the sub-panel's column of the
// aggregated update (k_update_agg).
__global__ void k_copy_T(BDView v, BDScratch s, int k0, int nbe, double *TS = nullptr, int tcol = 0) {
    const int m = blockIdx.y;
    const int n2 = v.n2;
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (long long)n2 * NB) return;
    const int r = (int)(q / NB), c = (int)(q % NB);
    const double *M = v.mat + (long long)m * v.mstride;
    const double t = c < nbe ? M[(long long)r * n2 + k0 + c] : 0.0;
    s.T[(long long)m * n2 * NB + q] = t;
    if (TS) TS[(long long)r * kSB + tcol + c] = (c < nbe && r == k0 + c) ? t - 1.0 : t;
}

// G[c][j] = sum_c' A11i[c][c'] M[k0+c'][j]  (j outside K);  G[c][K] = A11i.
__global__ void k_make_G(BDView v, BDScratch s, int k0, int nbe, int jlo = 0, int jhi = 1 << 30) {
    const int m = blockIdx.y;
    const int n2 = v.n2;
    const int j = jlo + blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= jhi) return;
    __shared__ double Ai[NB][NB];
    const double *A = s.A11i + (long long)m * NB * NB;
    for (int q = threadIdx.x; q < NB * NB; q += blockDim.x) Ai[q / NB][q % NB] = A[q];
    __syncthreads();
    if (j >= n2) return;
    const double *M = v.mat + (long long)m * v.mstride;
    double *G = s.G + (long long)m * NB * n2;
    if (j >= k0 && j < k0 + nbe) {
        for (int c = 0; c < NB; ++c) G[(long long)c * n2 + j] = c < nbe ? Ai[c][j - k0] : 0.0;
        return;
    }
    double col[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) col[c] = c < nbe ? M[(long long)(k0 + c) * n2 + j] : 0.0;
    for (int c = 0; c < NB; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < NB; ++q) acc = fma(Ai[c][q], col[q], acc);
        G[(long long)c * n2 + j] = c < nbe ? acc : 0.0;
    }
}

// The sweep, v2: 128x128 output tile per CTA, 256 threads, 8x8 outputs per
// thread (rows tr + 16a, columns 2tc + 32b + {0,1}); T staged transposed and G
// row-wise in shared memory (12 shared loads per 64 DFMA per panel column).
constexpr int UT2 = 128;
constexpr int UT2P = UT2 + 2;  // padding keeps double2 alignment and spreads banks
__global__ void __launch_bounds__(256) k_update2(BDView v, BDScratch s, int k0, int nbe) {
    extern __shared__ double sm2[];
    double *Ts = sm2;              // [NB][UT2P]  Ts[c][i] = T[i0 + i][c]
    double *Gs = sm2 + NB * UT2P;  // [NB][UT2P]  Gs[c][j] = G[c][j0 + j]
    const int m = blockIdx.z;
    const int n2 = v.n2;
    const int i0 = blockIdx.y * UT2, j0 = blockIdx.x * UT2;
    const double *T = s.T + (long long)m * n2 * NB;
    const double *G = s.G + (long long)m * NB * n2;
    double *M = v.mat + (long long)m * v.mstride;
    const int tid = threadIdx.x;
    for (int q = tid; q < UT2 * NB; q += 256) {
        const int i = q / NB, c = q % NB;
        Ts[c * UT2P + i] = (i0 + i < n2) ? T[(long long)(i0 + i) * NB + c] : 0.0;
    }
    for (int q = tid; q < NB * UT2; q += 256) {
        const int c = q / UT2, j = q % UT2;
        Gs[c * UT2P + j] = (j0 + j < n2) ? G[(long long)c * n2 + j0 + j] : 0.0;
    }
    __syncthreads();
    const int tr = tid >> 4, tc = tid & 15;
    double acc[8][8];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] = 0.0;
#pragma unroll 4
    for (int c = 0; c < NB; ++c) {
        double ta[8], gb[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) ta[a] = Ts[c * UT2P + tr + 16 * a];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const double2 g2 = *reinterpret_cast<const double2 *>(&Gs[c * UT2P + 2 * tc + 32 * b]);
            gb[2 * b] = g2.x;
            gb[2 * b + 1] = g2.y;
        }
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int b = 0; b < 8; ++b) acc[a][b] = fma(ta[a], gb[b], acc[a][b]);
    }
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        const int gi = i0 + tr + 16 * a;
        if (gi >= n2) continue;
        const bool rowK = gi >= k0 && gi < k0 + nbe;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int jj = 2 * tc + 32 * b;
            const int gj = j0 + jj;
            if (gj >= n2) continue;  // n2 even, gj even -> gj + 1 < n2 too
            double2 *dst = reinterpret_cast<double2 *>(M + (long long)gi * n2 + gj);
            double2 o;
            if (rowK) {
                o = *reinterpret_cast<const double2 *>(&Gs[(gi - k0) * UT2P + jj]);
            } else {
                double2 base = *dst;
                if (gj >= k0 && gj < k0 + nbe) base.x = 0.0;
                if (gj + 1 >= k0 && gj + 1 < k0 + nbe) base.y = 0.0;
                o = make_double2(base.x - acc[a][2 * b], base.y - acc[a][2 * b + 1]);
            }
            *dst = o;
        }
    }
}

// The sweep, v3, on the FP64 tensor cores: out = base - T G is a rank-32 dense
// update, i.e. a GEMM with K = 32, computed with mma.sync.m8n8k4.f64 (DMMA).
// CTA tile 64x64, 4 warps in 2x2, each warp 32x32 = 4x4 DMMA tiles; T (64x32)
// and G (32x64) staged in shared memory; fragments:
//   A (8x4, row): lane t holds A[t>>2][t&3];  B (4x8, col): lane t holds B[t&3][t>>2];
//   C (8x8): lane t holds C[t>>2][2(t&3)], C[t>>2][2(t&3)+1].
__device__ __forceinline__ void dmma_m8n8k4(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}
constexpr int UT3 = 64;
__global__ void __launch_bounds__(128, 4) k_update3(BDView v, BDScratch s, int k0, int nbe, int jlo = 0,
                                                   int jhi = 1 << 30) {
    // row strides = 4 (mod 16) doubles: the DMMA fragment reads (lane (gr, gq) reads
    // Ts[.. + gr][.. + gq] and Gs[.. + gq][.. + gr]) then touch 16 distinct 8-byte bank
    // pairs per half-warp; with the +1 padding of round 1 they were 4-way conflicts
    // (8 wavefronts per LDS.64, and the kernels were bound by shared-memory bandwidth)
    __shared__ double Ts[UT3][NB + 4];  // Ts[i][c] = T[i0 + i][c]
    __shared__ double Gs[NB][UT3 + 4];  // Gs[c][j] = G[c][j0 + j]
    const int m = blockIdx.z;
    const int n2 = v.n2;
    const int jend = min(n2, jhi);  // column bound of this launch
    const int i0 = blockIdx.y * UT3, j0 = jlo + blockIdx.x * UT3;
    const double *T = s.T + (long long)m * n2 * NB;
    const double *G = s.G + (long long)m * NB * n2;
    double *M = v.mat + (long long)m * v.mstride;
    const int tid = threadIdx.x;
    const int lane = tid & 31, wid = tid >> 5;
    const int wr = (wid >> 1) * 32, wc = (wid & 1) * 32;
    const int gr = lane >> 2, gq = lane & 3;
    // staging: all 32 loads of a thread are issued before any shared store
    // (latency-bound otherwise: ncu showed long-scoreboard stalls dominating)
    {
        constexpr int PER = UT3 * NB / 128;  // 16
        double tv[PER], gv[PER];
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const int q = tid + 128 * r;
            const int i = q / NB, c = q % NB;
            tv[r] = (i0 + i < n2) ? T[(long long)(i0 + i) * NB + c] : 0.0;
        }
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const int q = tid + 128 * r;
            const int c = q / UT3, j = q % UT3;
            gv[r] = (j0 + j < jend) ? G[(long long)c * n2 + j0 + j] : 0.0;
        }
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const int q = tid + 128 * r;
            Ts[q / NB][q % NB] = tv[r];
            Gs[q / UT3][q % UT3] = gv[r];
        }
    }
    __syncthreads();
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < NB / 4; ++kk) {
        double af[4], bf[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = Ts[wr + 8 * i + gr][kk * 4 + gq];
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = Gs[kk * 4 + gq][wc + 8 * j + gr];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma_m8n8k4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    // epilogue: the 16 double2 reads of M are issued together, then the writes
    double2 base[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int gi = i0 + wr + 8 * i + gr;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gj = j0 + wc + 8 * j + 2 * gq;
            base[i][j] = (gi < n2 && gj < jend) ? __ldcs(reinterpret_cast<const double2 *>(M + (long long)gi * n2 + gj))
                                              : make_double2(0.0, 0.0);
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int li = wr + 8 * i + gr;
        const int gi = i0 + li;
        if (gi >= n2) continue;
        const bool rowK = gi >= k0 && gi < k0 + nbe;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int lj = wc + 8 * j + 2 * gq;
            const int gj = j0 + lj;
            if (gj >= jend) continue;  // n2, jend even, gj even
            double2 *dst = reinterpret_cast<double2 *>(M + (long long)gi * n2 + gj);
            double2 o;
            if (rowK) {
                o = make_double2(Gs[gi - k0][lj], Gs[gi - k0][lj + 1]);
            } else {
                double2 b = base[i][j];
                if (gj >= k0 && gj < k0 + nbe) b.x = 0.0;
                if (gj + 1 >= k0 && gj + 1 < k0 + nbe) b.y = 0.0;
                o = make_double2(b.x - acc[i][j][0], b.y - acc[i][j][1]);
            }
            __stcs(dst, o);
        }
    }
}

// ---------------------------------------------------------------------------
// Delayed (aggregated) update of a large single block (the wall).
// The NB-column sub-panels p = 0..nsub-1 of a kSB-column super-panel S are
// factored and applied to the slab M[:, S] one by one (k_make_G / k_update3
// restricted to S).  Every other column j only receives the row swaps; its
// update, the product of the nsub elementary Gauss-Jordan steps
//   x <- x - T-hat_p A11i_p x[K_p]     (T-hat_p = T_p - E_{K_p}: rows K_p become G)
// is applied at once as x <- x - T-hat_S y with y = [y_0; ...; y_{nsub-1}],
//   y_p = A11i_p (x[K_p] - sum_{q<p} T-hat_q[K_p, :] y_q)       (k_make_Y),
// one rank-kSB DMMA pass over the block (k_update_agg) instead of nsub rank-NB
// passes: a quarter of the HBM traffic for the same flops.  T-hat_q's rows follow
// the later sub-panels' swaps (k_swap swaps TS with M), so the algebra is the
// sequential one; only the rounding order of the updates differs.

// y for every column j outside S, Y[kSB][n2] row-major.  A CTA takes 32 columns
// (lanes) x 4 row groups (warps; 8 of a sub-panel's NB pivot rows each): the
// round-2 one-thread-per-column form left under one warp per scheduler with 253
// registers and was latency-bound (0.215 ms per super-panel, on the lookahead's
// critical path).  Same sums in the same order, so Y is bitwise unchanged.
constexpr int kYCols = 32;
__global__ void __launch_bounds__(128) k_make_Y(BDView v, const double *__restrict__ TS,
                                                const double *__restrict__ A11S, double *Y, int s0, int sbe,
                                                int nsub) {
    __shared__ double s_acc[NB][kYCols + 1];
    __shared__ double s_A[NB][NB + 1];
    const int n2 = v.n2;
    const int lane = threadIdx.x & 31, rg = threadIdx.x >> 5;
    const int t = blockIdx.x * kYCols + lane;
    const bool ok = t < n2 - sbe;
    const int j = ok ? (t < s0 ? t : t + sbe) : 0;
    const double *M = v.mat;
    for (int p = 0; p < nsub; ++p) {
        const int k0 = s0 + p * NB, nbe = min(NB, n2 - k0);
        for (int q = threadIdx.x; q < NB * NB; q += 128) s_A[q / NB][q % NB] = A11S[(long long)p * NB * NB + q];
        double acc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int c = rg * 8 + i;
            acc[i] = (ok && c < nbe) ? M[(long long)(k0 + c) * n2 + j] : 0.0;
        }
        for (int q = 0; q < p; ++q) {
#pragma unroll 8
            for (int cc = 0; cc < NB; ++cc) {
                const double y = ok ? Y[(long long)(q * NB + cc) * n2 + j] : 0.0;
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    acc[i] = fma(-__ldg(TS + (long long)(k0 + rg * 8 + i) * kSB + q * NB + cc), y, acc[i]);
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) s_acc[rg * 8 + i][lane] = acc[i];
        __syncthreads();
        double y[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) y[i] = 0.0;
#pragma unroll 4
        for (int cc = 0; cc < NB; ++cc) {
            if (cc < nbe) {  // A11i is nbe x nbe
                const double a = s_acc[cc][lane];
#pragma unroll
                for (int i = 0; i < 8; ++i) y[i] = fma(s_A[rg * 8 + i][cc], a, y[i]);
            }
        }
        if (ok) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int c = rg * 8 + i;
                Y[(long long)(p * NB + c) * n2 + j] = c < nbe ? y[i] : 0.0;
            }
        }
        __syncthreads();  // Y of this sub-panel visible to the CTA's other warps; s_acc / s_A reusable
    }
}

// M[:, j] -= TS[:, 0:K] Y[0:K, j] for the column tiles outside S (K = nsub NB),
// on the FP64 tensor cores: k_update3's 64x64 DMMA tiles with the K dimension
// looped in NB chunks through the same shared-memory tiles.
__global__ void __launch_bounds__(128, 3) k_update_agg(BDView v, const double *__restrict__ TS,
                                                       const double *__restrict__ Y, int s0, int sbe, int nsub) {
    __shared__ double Ts[UT3][NB + 4];  // strides = 4 (mod 16): conflict-free fragment reads (k_update3)
    __shared__ double Gs[NB][UT3 + 4];
    const int n2 = v.n2;
    const int i0 = blockIdx.y * UT3, j0 = blockIdx.x * UT3;
    if (j0 >= s0 && j0 < s0 + sbe) return;  // the slab is final (s0, sbe multiples of UT3)
    double *M = v.mat;
    const int tid = threadIdx.x;
    const int lane = tid & 31, wid = tid >> 5;
    const int wr = (wid >> 1) * 32, wc = (wid & 1) * 32;
    const int gr = lane >> 2, gq = lane & 3;
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int p = 0; p < nsub; ++p) {
        constexpr int PER = UT3 * NB / 128;  // 16
        double tv[PER], gv[PER];
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const int q = tid + 128 * r;
            const int i = q / NB, c = q % NB;
            tv[r] = (i0 + i < n2) ? TS[(long long)(i0 + i) * kSB + p * NB + c] : 0.0;
        }
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const int q = tid + 128 * r;
            const int c = q / UT3, j = q % UT3;
            gv[r] = (j0 + j < n2) ? Y[(long long)(p * NB + c) * n2 + j0 + j] : 0.0;
        }
        __syncthreads();  // the previous chunk's fragments are read
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const int q = tid + 128 * r;
            Ts[q / NB][q % NB] = tv[r];
            Gs[q / UT3][q % UT3] = gv[r];
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < NB / 4; ++kk) {
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = Ts[wr + 8 * i + gr][kk * 4 + gq];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = Gs[kk * 4 + gq][wc + 8 * j + gr];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma_m8n8k4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
    }
    double2 base[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int gi = i0 + wr + 8 * i + gr;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gj = j0 + wc + 8 * j + 2 * gq;
            base[i][j] = (gi < n2 && gj < n2) ? __ldcs(reinterpret_cast<const double2 *>(M + (long long)gi * n2 + gj))
                                              : make_double2(0.0, 0.0);
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int gi = i0 + wr + 8 * i + gr;
        if (gi >= n2) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gj = j0 + wc + 8 * j + 2 * gq;
            if (gj >= n2) continue;
            __stcs(reinterpret_cast<double2 *>(M + (long long)gi * n2 + gj),
                   make_double2(base[i][j].x - acc[i][j][0], base[i][j].y - acc[i][j][1]));
        }
    }
}

// k_update_agg with the K chunks staged by cp.async into double-buffered shared
// memory (the default; the register-staged kernel above is the A/B alternative,
// BIE_BD_AGGK=0): chunk p + 1 streams in while chunk p feeds the DMMAs, so a CTA
// no longer idles through a global-load round trip per chunk.  n2 % UT3 == 0
// (checked by the caller), so there are no ragged tiles.
__device__ __forceinline__ void bd_cp_async16(void *smem, const void *gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem));
}
constexpr int kAggTsLd = NB + 4, kAggGsLd = UT3 + 4;  // doubles; = 4 (mod 16), rows 16-byte aligned
constexpr int kAggStage = UT3 * kAggTsLd + NB * kAggGsLd;  // doubles per stage
constexpr size_t kAggSmem = sizeof(double) * 2 * kAggStage;
__global__ void __launch_bounds__(128, 4) k_update_agg_async(BDView v, const double *__restrict__ TS,
                                                             const double *__restrict__ Y, int s0, int sbe,
                                                             int nsub, int jt0 = 0, int x0 = -1, int x1 = -1) {
    extern __shared__ __align__(16) double agg_smem[];
    const int n2 = v.n2;
    const int i0 = blockIdx.y * UT3, j0 = (jt0 + blockIdx.x) * UT3;
    if (j0 >= s0 && j0 < s0 + sbe) return;  // the slab is final (s0, sbe multiples of UT3)
    if (j0 >= x0 && j0 < x1) return;        // columns another launch of this update covers (lookahead)
    double *M = v.mat;
    const int tid = threadIdx.x;
    const int lane = tid & 31, wid = tid >> 5;
    const int wr = (wid >> 1) * 32, wc = (wid & 1) * 32;
    const int gr = lane >> 2, gq = lane & 3;
    auto stage = [&](int buf, int p) {
        double *Ts = agg_smem + buf * kAggStage, *Gs = Ts + UT3 * kAggTsLd;
        // Ts: 64 rows x 32 doubles = 64 x 16 pieces of 16 B; Gs: 32 rows x 64 doubles = 32 x 32 pieces
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int q = tid + 128 * r;
            const int i = q >> 4, c = (q & 15) * 2;
            bd_cp_async16(Ts + i * kAggTsLd + c, TS + (long long)(i0 + i) * kSB + p * NB + c);
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int q = tid + 128 * r;
            const int c = q >> 5, j = (q & 31) * 2;
            bd_cp_async16(Gs + c * kAggGsLd + j, Y + (long long)(p * NB + c) * n2 + j0 + j);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    stage(0, 0);
    for (int p = 0; p < nsub; ++p) {
        if (p + 1 < nsub) {
            stage((p + 1) & 1, p + 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const double *Ts = agg_smem + (p & 1) * kAggStage, *Gs = Ts + UT3 * kAggTsLd;
#pragma unroll
        for (int kk = 0; kk < NB / 4; ++kk) {
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = Ts[(wr + 8 * i + gr) * kAggTsLd + kk * 4 + gq];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = Gs[(kk * 4 + gq) * kAggGsLd + wc + 8 * j + gr];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma_m8n8k4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        __syncthreads();  // this stage is overwritten by the fetch of chunk p + 2
    }
    // epilogue in two halves of the warp tile's rows (8 double2 reads in flight per
    // thread): with the whole tile's base values live beside the accumulators the
    // kernel needs 160 registers; at <= 128 three of its CTAs leave room on the SM for
    // one CTA of the cooperative panel that the lookahead schedule runs beside it
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        double2 base[2][4];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int gi = i0 + wr + 8 * (2 * h + i) + gr;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int gj = j0 + wc + 8 * j + 2 * gq;
                base[i][j] = __ldcs(reinterpret_cast<const double2 *>(M + (long long)gi * n2 + gj));
            }
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int gi = i0 + wr + 8 * (2 * h + i) + gr;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int gj = j0 + wc + 8 * j + 2 * gq;
                __stcs(reinterpret_cast<double2 *>(M + (long long)gi * n2 + gj),
                       make_double2(base[i][j].x - acc[2 * h + i][j][0], base[i][j].y - acc[2 * h + i][j][1]));
            }
        }
    }
}

// Column unpermutation: A^{-1}[:, q[r]] = M[:, r], q = row order after all swaps.
__global__ void k_perm(BDView v, BDScratch s) {
    const int m = blockIdx.x;
    const int n2 = v.n2;
    int *q = s.piv + (long long)m * n2;  // in place: piv -> q (single thread, sequential)
    if (threadIdx.x != 0) return;
    // q built in W's int view is avoided: reuse T as int storage
    int *perm = reinterpret_cast<int *>(s.T + (long long)m * n2 * NB);
    for (int r = 0; r < n2; ++r) perm[r] = r;
    for (int k = 0; k < n2; ++k) {
        int p = q[k];
        int t = perm[k];
        perm[k] = perm[p];
        perm[p] = t;
    }
}

__global__ void k_unpermute(BDView v, BDScratch s) {
    extern __shared__ double row[];
    const int m = blockIdx.y, r = blockIdx.x;
    const int n2 = v.n2;
    double *M = v.mat + (long long)m * v.mstride + (long long)r * n2;
    const int *perm = reinterpret_cast<const int *>(s.T + (long long)m * n2 * NB);
    for (int j = threadIdx.x; j < n2; j += blockDim.x) row[j] = M[j];
    __syncthreads();
    for (int j = threadIdx.x; j < n2; j += blockDim.x) M[perm[j]] = row[j];
}

// Rows too long for shared memory (n2 > 27k: the config-5 wall, 32768 columns):
// rows [r0, r0 + NB) staged in the panel workspace W (NB x n2 per matrix).
__global__ void k_unpermute_g(BDView v, BDScratch s, int r0) {
    const int m = blockIdx.y, r = r0 + blockIdx.x;
    const int n2 = v.n2;
    if (r >= n2) return;
    double *M = v.mat + (long long)m * v.mstride + (long long)r * n2;
    double *row = s.W + (long long)m * n2 * NB + (long long)blockIdx.x * n2;
    const int *perm = reinterpret_cast<const int *>(s.T + (long long)m * n2 * NB);
    for (int j = threadIdx.x; j < n2; j += blockDim.x) row[j] = M[j];
    __syncthreads();
    for (int j = threadIdx.x; j < n2; j += blockDim.x) M[perm[j]] = row[j];
}

// ------------------------------------------------------------------ apply (A7)
// One warp per row of the explicit inverse; NVA vectors per pass.
// Vectors are local to the handle's body range: local row 0 is node row_lo.
template <int NVA>
__global__ void __launch_bounds__(256) k_bd_apply(const double *__restrict__ inv, const long long *__restrict__ off,
                                                  int wall_lo, int n_pore, int N, int b0, int row_lo, int rows_loc,
                                                  const double *in, double *out, long long stride, int v0) {
    pdl_wait();
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= 2 * rows_loc) return;
    const int node = row_lo + (warp >> 1);
    int b, lo, n;
    if (node < wall_lo) {
        b = node / n_pore;
        lo = b * n_pore;
        n = n_pore;
    } else {
        b = wall_lo / max(n_pore, 1);  // wall body index = M
        if (n_pore == 0) b = 0;
        lo = wall_lo;
        n = N - wall_lo;
    }
    const int n2 = 2 * n;
    const int lr = 2 * (node - lo) + (warp & 1);
    // the row lies inside body b's inverse: [off[b - b0], off[b - b0 + 1])
    BIE_DCHECK(b >= b0 && off[b - b0] + (long long)(lr + 1) * n2 <= off[b - b0 + 1]);
    const double2 *row = reinterpret_cast<const double2 *>(inv + off[b - b0] + (long long)lr * n2);
    const int lo_loc = lo - row_lo;
    double acc[NVA];
#pragma unroll
    for (int v = 0; v < NVA; ++v) acc[v] = 0.0;
    for (int c = lane; c < n; c += 32) {
        const double2 a = __ldcs(row + c);
#pragma unroll
        for (int v = 0; v < NVA; ++v) {
            const double2 x = reinterpret_cast<const double2 *>(in + (long long)(v0 + v) * stride + 2LL * lo_loc)[c];
            acc[v] = fma(a.x, x.x, fma(a.y, x.y, acc[v]));
        }
    }
#pragma unroll
    for (int v = 0; v < NVA; ++v) {
        double t = acc[v];
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) out[(long long)(v0 + v) * stride + warp] = t;
    }
}

static int factor_class(Geometry *g, BDView v, int lo0, int nodes, bool is_wall, cudaStream_t st,
                        int *d_flag, int op) {
    if (v.count == 0) return BIE_OK;
    const int n2 = v.n2;
    BDScratch s{};
    size_t wbytes = sizeof(double) * (size_t)v.count * n2 * NB;
    BIE_CUDA_TRY(cudaMallocAsync(&s.W, wbytes, st));
    BIE_CUDA_TRY(cudaMallocAsync(&s.T, wbytes, st));
    BIE_CUDA_TRY(cudaMallocAsync(&s.G, wbytes, st));
    BIE_CUDA_TRY(cudaMallocAsync(&s.A11i, sizeof(double) * (size_t)v.count * NB * NB, st));
    BIE_CUDA_TRY(cudaMallocAsync(&s.piv, sizeof(int) * (size_t)v.count * n2, st));
    s.flag = d_flag;
    {
        long long elems = (long long)nodes * nodes;
        dim3 grid((unsigned)((elems + 255) / 256), v.count);
        if (op) {
            KRWeights kr;
            for (int k = 0; k < 6; ++k) kr.g[k] = g->kr[k];
            k_bd_assemble_slp<<<grid, 256, 0, st>>>(v, lo0, nodes, g->pos, g->w, kr);
        } else {
            k_bd_assemble<<<grid, 256, 0, st>>>(v, lo0, nodes, is_wall ? 1 : 0, g->pos, g->nw, g->nrm, g->tan,
                                                g->w, g->selfc, g->pore, g->wall_len);
        }
        count_launch();
        BIE_CUDA_TRY(cudaGetLastError());
    }
    // panel strategy: shared-memory panel (one CTA per matrix) while the panel fits,
    // cooperative multi-CTA panel for the single large block (Gamma_0 of configs 2-5)
    const bool coop = n2 > kSmemPanelRows && v.count == 1;
    CoopScratch cs{};
    // rows per thread of the cooperative panel (tuning knob BIE_PANEL_RPT = 1 | 2;
    // measured config 4, round 1: 1 row 0.72-0.74 s factor, 2 rows 0.78-0.80 s; with the
    // round-2 lookahead schedule and one-division panel: 0.356 vs 0.354 s, 1 row kept)
    int rpt = 1;
    if (const char *e = getenv("BIE_PANEL_RPT")) rpt = std::max(1, std::min(2, atoi(e)));
    void *coop_kernel = rpt == 2 ? (void *)k_panel_coop<2> : (void *)k_panel_coop<1>;
    if (coop) {
        const int Gmax = (n2 + 127) / 128;
        int per_sm = 0, dev = 0, coop_ok = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&coop_ok, cudaDevAttrCooperativeLaunch, dev);
        BIE_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, coop_kernel, 128, 0));
        if (!coop_ok || (long long)per_sm * g->num_sms < Gmax) {
            set_error("bie_blockdiag_factor: cooperative launch unavailable for the panel factorisation");
            return BIE_ECUDA;
        }
        BIE_CUDA_TRY(cudaMallocAsync(&cs.cand_v, sizeof(double) * 2 * Gmax, st));
        BIE_CUDA_TRY(cudaMallocAsync(&cs.cand_i, sizeof(int) * 2 * Gmax, st));
        BIE_CUDA_TRY(cudaMallocAsync(&cs.crow, sizeof(double) * 2 * Gmax * NB, st));
        BIE_CUDA_TRY(cudaMallocAsync(&cs.kbuf, sizeof(double) * 2 * NB, st));
        BIE_CUDA_TRY(cudaMallocAsync(&cs.A, sizeof(double) * NB * NB, st));
    }
    const size_t upd_smem = sizeof(double) * 2 * NB * UT2P;
    // sweep kernel: 0 = DMMA tensor-core tiles (default), 1 = 128x128 DFMA tiles (A/B knob)
    int upd_variant = 0;
    if (const char *e = getenv("BIE_BD_UPDATE")) upd_variant = std::max(0, std::min(1, atoi(e)));
    BIE_CUDA_TRY(cudaFuncSetAttribute(k_update2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)upd_smem));
    BIE_CUDA_TRY(cudaFuncSetAttribute(k_panel_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(sizeof(double) * NB * kSmemPanelRows)));
    // large single block (the wall): super-panels of kSB columns with the delayed
    // rank-kSB update of the columns outside the slab (k_make_Y / k_update_agg)
    double *TS = nullptr, *Yb = nullptr, *A11S = nullptr;
    // BIE_BD_AGG: 0 never, 1 whenever the block is factored cooperatively (tests),
    // default: blocks of order >= 4096 (config 4: 0.83 -> 0.57 s in round 2's first form; with
    // the lookahead schedule order 4096 gains too, config 3 36.6 -> 31.3 ms; at order 1024 the
    // extra launches cost more than the saved traffic, 7.8 -> 8.6 ms)
    int agg_mode = 2;
    if (const char *e = getenv("BIE_BD_AGG")) agg_mode = std::max(0, std::min(1, atoi(e)));
    const bool agg = coop && n2 % UT3 == 0 && (agg_mode == 1 || (agg_mode == 2 && n2 >= 4096));
    // BIE_BD_AGGK: 1 (default) cp.async double-buffered sweep, 0 register-staged (A/B)
    bool agg_async = true;
    if (const char *e = getenv("BIE_BD_AGGK")) agg_async = atoi(e) != 0;
    if (agg) {
        BIE_CUDA_TRY(cudaFuncSetAttribute(k_update_agg_async, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)kAggSmem));
        // two parities: with the lookahead, super-panel S + 1 fills one set while the
        // sweep of S reads the other
        BIE_CUDA_TRY(cudaMallocAsync(&TS, sizeof(double) * 2 * (size_t)n2 * kSB, st));
        BIE_CUDA_TRY(cudaMallocAsync(&Yb, sizeof(double) * 2 * (size_t)n2 * kSB, st));
        BIE_CUDA_TRY(cudaMallocAsync(&A11S, sizeof(double) * 2 * 4 * NB * NB, st));
    }
    auto panel = [&](int k0, int nbe) -> int {
        if (coop) {
            int G = (n2 - k0 + 128 * rpt - 1) / (128 * rpt);
            void *args[] = {&v, &s, &cs, &k0, &nbe};
            BIE_CUDA_TRY(cudaLaunchCooperativeKernel(coop_kernel, G, 128, args, 0, st));
        } else if (n2 - k0 <= kSmemPanelRows) {
            k_panel_smem<<<v.count, 256, sizeof(double) * NB * (n2 - k0), st>>>(v, s, k0, nbe);
        } else {
            int panel_threads = n2 >= 1024 ? 1024 : 256;
            k_panel<<<v.count, panel_threads, 0, st>>>(v, s, k0, nbe);
        }
        return BIE_OK;
    };
    // Lookahead (BIE_BD_LOOKAHEAD, default on with the cp.async sweep): the sub-panels of
    // super-panel S + 1 are factored on a high-priority stream while the rank-kSB sweep of
    // S still runs over the columns outside both slabs.  Per super-panel:
    //   hp: A(S)  = sub-panel LUs, swaps / G / rank-NB updates restricted to the slab (+ T-hat);
    //       wait for the previous sweep; swaps of S on the columns outside the slab;
    //       Y(S); sweep of S on slab S + 1 only;
    //   st: sweep of S on every other column (reads TS/Y of parity S & 1).
    // The cooperative panel's CTAs take the SM slots the sweep's CTAs free as they retire.
    bool lookahead = agg_async;
    if (const char *e = getenv("BIE_BD_LOOKAHEAD")) lookahead = lookahead && atoi(e) != 0;
    if (agg && lookahead) {
        if (!g->bd_hp) {
            int pr_lo = 0, pr_hi = 0;
            BIE_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&pr_lo, &pr_hi));
            BIE_CUDA_TRY(cudaStreamCreateWithPriority(&g->bd_hp, cudaStreamNonBlocking, pr_hi));
            for (cudaEvent_t &e : g->bd_ev) BIE_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        cudaStream_t hp = g->bd_hp;
        cudaEvent_t ev_y = g->bd_ev[0], ev_b2 = g->bd_ev[1], ev_f = g->bd_ev[2];
        // hp is joined into st by the last event wait below; the host wait keeps the scratch
        // frees (stream-ordered on st) and a later factor on another stream safely behind it
        auto cleanup = [&]() { cudaStreamSynchronize(hp); };
        // BIE_BD_TRACE=1 (diagnostic): per super-panel, CUDA-event times of the slab
        // factorisation A(S) on hp and of the sweep B2(S) on st, printed to stderr
        const bool trace = getenv("BIE_BD_TRACE") && atoi(getenv("BIE_BD_TRACE")) != 0;
        std::vector<cudaEvent_t> tev, tsub;  // tsub: 3 per sub-panel (before / after the panel LU, after its slab update)
        auto mark = [&](cudaStream_t q, bool sub = false) {
            if (!trace) return;
            cudaEvent_t e;
            cudaEventCreate(&e);
            cudaEventRecord(e, q);
            (sub ? tsub : tev).push_back(e);
        };
        int rc = [&]() -> int {
            BIE_CUDA_TRY(cudaEventRecord(ev_f, st));
            BIE_CUDA_TRY(cudaStreamWaitEvent(hp, ev_f, 0));
            BIE_CUDA_TRY(cudaEventRecord(ev_b2, st));  // "previous sweep done" for the first super-panel
            const int nt = n2 / UT3;
            for (int s0 = 0, S = 0; s0 < n2; s0 += kSB, ++S) {
                const int sbe = std::min(kSB, n2 - s0), nsub = (sbe + NB - 1) / NB;
                double *TSb = TS + (size_t)(S & 1) * n2 * kSB, *Ybb = Yb + (size_t)(S & 1) * n2 * kSB;
                double *A11b = A11S + (size_t)(S & 1) * 4 * NB * NB;
                mark(hp);  // [4S]: A(S) begins
                for (int p = 0; p < nsub; ++p) {
                    int k0 = s0 + p * NB, nbe = std::min(NB, n2 - k0);
                    mark(hp, true);
                    {
                        int G = (n2 - k0 + 128 * rpt - 1) / (128 * rpt);
                        void *args[] = {&v, &s, &cs, &k0, &nbe};
                        BIE_CUDA_TRY(cudaLaunchCooperativeKernel(coop_kernel, G, 128, args, 0, hp));
                    }
                    mark(hp, true);
                    k_swap_rng<<<(sbe + p * NB + 127) / 128, 128, 0, hp>>>(v, s, k0, nbe, s0, s0 + sbe, -1, -1, TSb,
                                                                           p * NB);
                    k_copy_T<<<dim3((unsigned)(((long long)n2 * NB + 255) / 256), 1), 256, 0, hp>>>(v, s, k0, nbe,
                                                                                                  TSb, p * NB);
                    BIE_CUDA_TRY(cudaMemcpyAsync(A11b + p * NB * NB, s.A11i, sizeof(double) * NB * NB,
                                                 cudaMemcpyDeviceToDevice, hp));
                    k_make_G<<<dim3((sbe + 127) / 128, 1), 128, 0, hp>>>(v, s, k0, nbe, s0, s0 + sbe);
                    k_update3<<<dim3((sbe + UT3 - 1) / UT3, (n2 + UT3 - 1) / UT3, 1), 128, 0, hp>>>(v, s, k0, nbe,
                                                                                                 s0, s0 + sbe);
                    mark(hp, true);
                    count_launch(5);
                    BIE_CUDA_TRY(cudaGetLastError());
                }
                mark(hp);  // [4S + 1]: A(S) done
                if (n2 > sbe) {
                    const int s1 = s0 + sbe, s1e = std::min(n2, s1 + kSB);  // next slab [s1, s1e)
                    BIE_CUDA_TRY(cudaStreamWaitEvent(hp, ev_b2, 0));  // the previous sweep wrote these columns
                    k_swap_rng<<<(n2 + 127) / 128, 128, 0, hp>>>(v, s, s0, sbe, 0, n2, s0, s0 + sbe, nullptr, 0);
                    k_make_Y<<<(n2 - sbe + kYCols - 1) / kYCols, 128, 0, hp>>>(v, TSb, A11b, Ybb, s0, sbe, nsub);
                    count_launch(2);
                    if (s1 < n2) {
                        k_update_agg_async<<<dim3((s1e - s1) / UT3, nt), 128, kAggSmem, hp>>>(v, TSb, Ybb, s0, sbe,
                                                                                              nsub, s1 / UT3);
                        count_launch();
                    }
                    BIE_CUDA_TRY(cudaEventRecord(ev_y, hp));
                    BIE_CUDA_TRY(cudaStreamWaitEvent(st, ev_y, 0));
                    mark(st);  // [4S + 2]: B2(S) begins
                    k_update_agg_async<<<dim3(nt, nt), 128, kAggSmem, st>>>(v, TSb, Ybb, s0, sbe, nsub, 0, s1, s1e);
                    mark(st);  // [4S + 3]: B2(S) done
                    count_launch();
                    BIE_CUDA_TRY(cudaEventRecord(ev_b2, st));
                    BIE_CUDA_TRY(cudaGetLastError());
                }
            }
            BIE_CUDA_TRY(cudaEventRecord(ev_y, hp));
            BIE_CUDA_TRY(cudaStreamWaitEvent(st, ev_y, 0));
            return BIE_OK;
        }();
        cleanup();
        if (trace && rc == BIE_OK && tev.size() % 4 == 0 && !tev.empty()) {
            cudaStreamSynchronize(st);
            double sa = 0, sb = 0, gap = 0;
            const size_t ns = tev.size() / 4;
            float ms = 0;
            for (size_t i = 0; i < ns; ++i) {
                cudaEventElapsedTime(&ms, tev[4 * i], tev[4 * i + 1]);
                sa += ms;
                cudaEventElapsedTime(&ms, tev[4 * i + 2], tev[4 * i + 3]);
                sb += ms;
                if (i + 1 < ns) {
                    cudaEventElapsedTime(&ms, tev[4 * i + 3], tev[4 * i + 6]);
                    gap += ms;
                }
            }
            cudaEventElapsedTime(&ms, tev[0], tev[tev.size() - 1]);
            fprintf(stderr, "[bie bd trace] n2=%d super-panels=%zu  A(S) avg %.3f ms  B2(S) avg %.3f ms  "
                            "gap between sweeps avg %.3f ms  total %.1f ms\n",
                    n2, ns, sa / ns, sb / ns, gap / (ns - 1), ms);
        }
        if (trace && rc == BIE_OK && tsub.size() % 3 == 0 && !tsub.empty()) {
            double sp = 0, sr = 0;
            float ms = 0;
            for (size_t i = 0; i < tsub.size(); i += 3) {
                cudaEventElapsedTime(&ms, tsub[i], tsub[i + 1]);
                sp += ms;
                cudaEventElapsedTime(&ms, tsub[i + 1], tsub[i + 2]);
                sr += ms;
            }
            fprintf(stderr, "[bie bd trace] per sub-panel: panel LU avg %.3f ms, swap/T/G/slab update avg %.3f ms\n",
                    sp / (tsub.size() / 3), sr / (tsub.size() / 3));
        }
        for (cudaEvent_t e : tev) cudaEventDestroy(e);
        for (cudaEvent_t e : tsub) cudaEventDestroy(e);
        if (rc) return rc;
        cudaFreeAsync(TS, st);
        cudaFreeAsync(Yb, st);
        cudaFreeAsync(A11S, st);
    } else if (agg) {
        for (int s0 = 0; s0 < n2; s0 += kSB) {
            const int sbe = std::min(kSB, n2 - s0), nsub = (sbe + NB - 1) / NB;
            for (int p = 0; p < nsub; ++p) {
                const int k0 = s0 + p * NB, nbe = std::min(NB, n2 - k0);
                BIE_RC_TRY(panel(k0, nbe));
                k_swap<<<dim3((n2 + p * NB + 127) / 128, 1), 128, 0, st>>>(v, s, k0, nbe, TS, p * NB);
                k_copy_T<<<dim3((unsigned)(((long long)n2 * NB + 255) / 256), 1), 256, 0, st>>>(v, s, k0, nbe, TS,
                                                                                              p * NB);
                BIE_CUDA_TRY(cudaMemcpyAsync(A11S + p * NB * NB, s.A11i, sizeof(double) * NB * NB,
                                             cudaMemcpyDeviceToDevice, st));
                k_make_G<<<dim3((sbe + 127) / 128, 1), 128, 0, st>>>(v, s, k0, nbe, s0, s0 + sbe);
                k_update3<<<dim3((sbe + UT3 - 1) / UT3, (n2 + UT3 - 1) / UT3, 1), 128, 0, st>>>(v, s, k0, nbe, s0,
                                                                                             s0 + sbe);
                count_launch(5);
                BIE_CUDA_TRY(cudaGetLastError());
            }
            if (n2 > sbe) {
                k_make_Y<<<(n2 - sbe + kYCols - 1) / kYCols, 128, 0, st>>>(v, TS, A11S, Yb, s0, sbe, nsub);
                if (agg_async)
                    k_update_agg_async<<<dim3(n2 / UT3, n2 / UT3), 128, kAggSmem, st>>>(v, TS, Yb, s0, sbe, nsub);
                else
                    k_update_agg<<<dim3((n2 + UT3 - 1) / UT3, (n2 + UT3 - 1) / UT3), 128, 0, st>>>(v, TS, Yb, s0, sbe,
                                                                                                  nsub);
                count_launch(2);
                BIE_CUDA_TRY(cudaGetLastError());
            }
        }
        cudaFreeAsync(TS, st);
        cudaFreeAsync(Yb, st);
        cudaFreeAsync(A11S, st);
    }
    for (int k0 = 0; k0 < n2 && !agg; k0 += NB) {
        int nbe = std::min(NB, n2 - k0);
        BIE_RC_TRY(panel(k0, nbe));
        k_swap<<<dim3((n2 + 127) / 128, v.count), 128, 0, st>>>(v, s, k0, nbe);
        k_copy_T<<<dim3((unsigned)(((long long)n2 * NB + 255) / 256), v.count), 256, 0, st>>>(v, s, k0, nbe);
        k_make_G<<<dim3((n2 + 127) / 128, v.count), 128, 0, st>>>(v, s, k0, nbe);
        if (upd_variant == 1)
            k_update2<<<dim3((n2 + UT2 - 1) / UT2, (n2 + UT2 - 1) / UT2, v.count), 256, upd_smem, st>>>(v, s, k0,
                                                                                                       nbe);
        else
            k_update3<<<dim3((n2 + UT3 - 1) / UT3, (n2 + UT3 - 1) / UT3, v.count), 128, 0, st>>>(v, s, k0, nbe);
        count_launch(5);
        BIE_CUDA_TRY(cudaGetLastError());
    }
    if (coop) {
        cudaFreeAsync(cs.cand_v, st);
        cudaFreeAsync(cs.cand_i, st);
        cudaFreeAsync(cs.crow, st);
        cudaFreeAsync(cs.kbuf, st);
        cudaFreeAsync(cs.A, st);
    }
    k_perm<<<v.count, 32, 0, st>>>(v, s);
    size_t rowbytes = sizeof(double) * (size_t)n2;
    if (rowbytes <= 200 * 1024) {
        if (rowbytes > 48 * 1024)
            BIE_CUDA_TRY(cudaFuncSetAttribute(k_unpermute, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rowbytes));
        k_unpermute<<<dim3(n2, v.count), 256, rowbytes, st>>>(v, s);
    } else {
        for (int r0 = 0; r0 < n2; r0 += NB) {
            k_unpermute_g<<<dim3(NB, v.count), 256, 0, st>>>(v, s, r0);
            count_launch();
        }
    }
    count_launch(2);
    BIE_CUDA_TRY(cudaGetLastError());
    cudaFreeAsync(s.W, st);
    cudaFreeAsync(s.T, st);
    cudaFreeAsync(s.G, st);
    cudaFreeAsync(s.A11i, st);
    cudaFreeAsync(s.piv, st);
    return BIE_OK;
}

// ---------------------------------------------------------------------------
// Structured pore blocks (NEXT-4; pin V10 of DESIGN.md).  Equispaced circular
// pores with equal n_p have completed-DLP blocks
//   B_k = B_ref + c_k E,  E = 1 1^T (x) I_2 = U U^T,  c_k = (log r_ref - log r_k) / (4 pi n_p)
// (only the Stokeslet's -log r_k term of the completion depends on the radius),
// so by Woodbury  B_k^-1 = X - c_k W (I_2 + c_k G)^-1 Z  with X = B_ref^-1,
// W = X U, Z = U^T X, G = U^T X U.  Apply: Y = X [v_1 .. v_M] (one GEMM over
// all pores), s_k = U^T y_k, y_k -= W M_k s_k with M_k = c_k (I + c_k G)^-1.
// ---------------------------------------------------------------------------
__global__ void k_struct_WG(const double *__restrict__ X, int n2, double *W, double *G) {
    for (int i = threadIdx.x; i < n2; i += blockDim.x) {
        double w0 = 0.0, w1 = 0.0;
        for (int j = 0; j < n2; j += 2) {
            w0 += X[(long long)i * n2 + j];
            w1 += X[(long long)i * n2 + j + 1];
        }
        W[2 * i] = w0;
        W[2 * i + 1] = w1;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        const int a = threadIdx.x >> 1, c = threadIdx.x & 1;  // G[a][c] = sum_i W[2i + a][c]
        double g = 0.0;
        for (int i = 0; i < n2 / 2; ++i) g += W[2 * (2 * i + a) + c];
        G[threadIdx.x] = g;
    }
}

// Y[:, col] = X V[:, col] for col < ncols; column col is vector col / M,
// pore col % M, at base + (col / M) * stride + n2 * (col % M).  Tiles of 32
// columns x 8 RT rows (RT rows per thread); every output is one sequential FMA
// chain over k = 0 .. n2-1, so the tile shape does not change the result.
// RT = 4 when the 32-row grid fills the SMs (config 4: 30 us per apply; RT = 1
// there measured 63 us); RT = 1 otherwise (config 2: 8 -> 32 CTAs).
template <int RT>
__global__ void __launch_bounds__(256) k_struct_gemm(const double *__restrict__ X, int n2, int M, int ncols,
                                                     const double *__restrict__ in, double *out, long long stride) {
    pdl_wait();
    constexpr int TR = 8 * RT;  // tile rows
    __shared__ double Xs[TR][33];
    __shared__ double Vs[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // ty: 8 row groups of RT rows
    const int r0 = blockIdx.y * TR, c0 = blockIdx.x * 32;
    const int col = c0 + tx;
    const long long cbase = col < ncols ? (long long)(col / M) * stride + (long long)n2 * (col % M) : 0;
    double acc[RT];
#pragma unroll
    for (int q = 0; q < RT; ++q) acc[q] = 0.0;
    for (int k0 = 0; k0 < n2; k0 += 32) {
#pragma unroll
        for (int q = 0; q < RT; ++q) {
            const int rr = ty * RT + q;  // X tile row
            Xs[rr][tx] = (r0 + rr < n2 && k0 + tx < n2) ? X[(long long)(r0 + rr) * n2 + k0 + tx] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int kk = ty * 4 + q;  // V tile k
            Vs[kk][tx] = (col < ncols && k0 + kk < n2) ? in[cbase + k0 + kk] : 0.0;
        }
        __syncthreads();
#pragma unroll 8
        for (int kk = 0; kk < 32; ++kk) {
            const double v = Vs[kk][tx];
#pragma unroll
            for (int q = 0; q < RT; ++q) acc[q] = fma(Xs[ty * RT + q][kk], v, acc[q]);
        }
        __syncthreads();
    }
    if (col < ncols) {
#pragma unroll
        for (int q = 0; q < RT; ++q) {
            const int r = r0 + ty * RT + q;
            if (r < n2) out[cbase + r] = acc[q];
        }
    }
}

// ---------------------------------------------------------------------------
// SLP pore blocks through their rotating-frame circulant structure (NEXT-1 x
// NEXT-4; P:l.655-657 footnote: the pore blocks can be "accelerated using the
// FFT").  Pore k's nodes are x_j = c_k + r_k (cos, sin)(theta_j), theta_j =
// 2 pi j / n (reading C12), and its SLP block B[i][j] = W_ij G(x_i - x_j)
// (2x2 blocks; W periodic in j - i, C25) satisfies, with T_j = R(theta_j),
//   T_i^T B[i][j] T_j = b((j - i) mod n)       (G(R v) = R G(v) R^T),
// so B = D C D^T, D = diag(T_j), C block-circulant with first block row b(m).
// C^-1 is block-circulant with first block row
//   d(m) = (1/n) sum_f chat(f)^-1 w^{-fm},  chat(f) = sum_m b(m) w^{fm},  w = e^{2 pi i/n}
// (one 2x2 complex inverse per frequency).  Factor: one CTA per pore, direct
// O(n^2) DFTs in FP64 from the node table (the entries are those of
// k_bd_assemble_slp).  Apply: y_i = T_i sum_m d(m) T_{i+m}^T v_{(i+m) mod n}.
// Storage 4 n doubles per pore (config 5: 33 MB instead of 17 GB of dense
// inverses).
__global__ void __launch_bounds__(256) k_circ_factor(const double2 *__restrict__ pos, const double *__restrict__ w,
                                                     KRWeights kr, const double2 *__restrict__ tmpl, int n,
                                                     double *D, int *flag) {
    extern __shared__ double sh[];
    double *b = sh;                                          // [n][4]  b(m), row-major 2x2
    double *ci = sh + 4 * n;                                 // [n][8]  chat(f)^-1 (re, im per entry)
    double2 *tw = reinterpret_cast<double2 *>(sh + 12 * n);  // [n]     (cos, sin)(2 pi m / n)
    const int k = blockIdx.x, lo = k * n;
    for (int m = threadIdx.x; m < n; m += blockDim.x) {
        const double2 t = tmpl[m];
        tw[m] = t;
        double e00 = 0.0, e01 = 0.0, e11 = 0.0;
        if (m != 0) {
            const int kk = min(m, n - m);
            double W = w[lo + m];
            if (kk <= 6) W *= 1.0 + kr.g[kk - 1];
            const double2 xi = pos[lo], xj = pos[lo + m];
            const double rx = xi.x - xj.x, ry = xi.y - xj.y;
            const double rho2 = rx * rx + ry * ry;
            const double lg = 0.5 * log(rho2);
            const double f = W * (1.0 / (4.0 * kPi));
            e00 = f * (-lg + rx * rx / rho2);
            e01 = f * (rx * ry / rho2);
            e11 = f * (-lg + ry * ry / rho2);
        }
        // b(m) = B[0][m] T_m  (T_0 = I)
        b[4 * m + 0] = e00 * t.x + e01 * t.y;
        b[4 * m + 1] = -e00 * t.y + e01 * t.x;
        b[4 * m + 2] = e01 * t.x + e11 * t.y;
        b[4 * m + 3] = -e01 * t.y + e11 * t.x;
    }
    __syncthreads();
    for (int f = threadIdx.x; f < n; f += blockDim.x) {
        double re[4] = {0.0, 0.0, 0.0, 0.0}, im[4] = {0.0, 0.0, 0.0, 0.0};
        int idx = 0;  // f m mod n
        for (int m = 0; m < n; ++m) {
            const double2 c = tw[idx];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                re[q] = fma(b[4 * m + q], c.x, re[q]);
                im[q] = fma(b[4 * m + q], c.y, im[q]);
            }
            idx += f;
            if (idx >= n) idx -= n;
        }
        // inverse of [[a, bb], [c, d]] (complex): [[d, -bb], [-c, a]] / (a d - bb c)
        const double dr = (re[0] * re[3] - im[0] * im[3]) - (re[1] * re[2] - im[1] * im[2]);
        const double di = (re[0] * im[3] + im[0] * re[3]) - (re[1] * im[2] + im[1] * re[2]);
        const double den = dr * dr + di * di;
        if (!(den > 0.0) || !isfinite(den)) atomicExch(flag, 1);
        const double ir = dr / den, ii = -di / den;  // 1 / det
        const double er[4] = {re[3], -re[1], -re[2], re[0]}, ei[4] = {im[3], -im[1], -im[2], im[0]};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            ci[8 * f + 2 * q] = er[q] * ir - ei[q] * ii;
            ci[8 * f + 2 * q + 1] = er[q] * ii + ei[q] * ir;
        }
    }
    __syncthreads();
    const double inv_n = 1.0 / n;
    for (int m = threadIdx.x; m < n; m += blockDim.x) {
        double re[4] = {0.0, 0.0, 0.0, 0.0};
        int idx = 0;  // f m mod n;  Re(z conj(w^{fm})) = zr c + zi s
        for (int f = 0; f < n; ++f) {
            const double2 c = tw[idx];
#pragma unroll
            for (int q = 0; q < 4; ++q) re[q] = fma(ci[8 * f + 2 * q], c.x, fma(ci[8 * f + 2 * q + 1], c.y, re[q]));
            idx += m;
            if (idx >= n) idx -= n;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) D[((long long)k * n + m) * 4 + q] = re[q] * inv_n;
    }
}

// y_i = T_i sum_m d_k(m) T_{i+m}^T v_{(i+m) mod n}, one CTA per (vector, pore)
// column; v and d_k staged in shared memory.
__global__ void __launch_bounds__(128) k_circ_apply(const double *__restrict__ D, const double2 *__restrict__ tmpl,
                                                    int n, int M, const double *__restrict__ in, double *out,
                                                    long long stride) {
    pdl_wait();
    extern __shared__ double sh[];
    double2 *vt = reinterpret_cast<double2 *>(sh);  // [n] T_j^T v_j
    double *d = sh + 2 * n;                         // [n][4]
    const int col = blockIdx.x, k = col % M;
    const long long base = (long long)(col / M) * stride + 2LL * n * k;
    const double *Dk = D + (long long)k * n * 4;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const double2 t = tmpl[j];
        const double vx = in[base + 2 * j], vy = in[base + 2 * j + 1];
        vt[j] = make_double2(t.x * vx + t.y * vy, -t.y * vx + t.x * vy);
    }
    for (int q = threadIdx.x; q < 4 * n; q += blockDim.x) d[q] = Dk[q];
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double ax = 0.0, ay = 0.0;
        int j = i;
        for (int m = 0; m < n; ++m) {
            const double2 v = vt[j];
            ax = fma(d[4 * m], v.x, fma(d[4 * m + 1], v.y, ax));
            ay = fma(d[4 * m + 2], v.x, fma(d[4 * m + 3], v.y, ay));
            if (++j == n) j = 0;
        }
        const double2 t = tmpl[i];
        out[base + 2 * i] = t.x * ax - t.y * ay;
        out[base + 2 * i + 1] = t.y * ax + t.x * ay;
    }
}

// Rank-2 Woodbury correction, one warp per column (fixed-order sums).
__global__ void k_struct_corr(const double *__restrict__ W, const double *__restrict__ Mk, int n2, int M, int ncols,
                              double *out, long long stride) {
    pdl_wait();
    const int col = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (col >= ncols) return;
    const int k = col % M;
    double *y = out + (long long)(col / M) * stride + (long long)n2 * k;
    double s0 = 0.0, s1 = 0.0;
    for (int i = 2 * lane; i < n2; i += 64) {
        s0 += y[i];
        s1 += y[i + 1];
    }
    for (int o = 16; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    const double m0 = Mk[4 * k] * s0 + Mk[4 * k + 1] * s1;
    const double m1 = Mk[4 * k + 2] * s0 + Mk[4 * k + 3] * s1;
    for (int i = lane; i < n2; i += 32) y[i] -= W[2 * i] * m0 + W[2 * i + 1] * m1;
}

int blockdiag_apply_impl(BlockDiag *bd, const double *in, double *out, int nvec, cudaStream_t st) {
    Geometry *g = bd->g;
    const int rows_loc = bd->row_hi - bd->row_lo;
    const long long stride = 2LL * rows_loc;
    const int threads = 256;
    int blocks = (int)(((long long)2 * rows_loc * 32 + threads - 1) / threads);
    if (rows_loc == 0) return BIE_OK;
    int row_lo = bd->row_lo, rows_k = rows_loc, kb0 = bd->b0;
    if (bd->structured) {
        const int M = g->M, n2 = 2 * g->n_pore, ncols = nvec * M;
        if (M > 0 && bd->structured == 2) {  // SLP pores: rotating-frame circulant inverses
            BIE_LAUNCH(k_circ_apply, ncols, 128, sizeof(double) * 6 * g->n_pore, st, bd->sD, bd->sTmpl, g->n_pore, M,
                       in, out, stride);
            count_launch();
            BIE_CUDA_TRY(cudaGetLastError());
        } else if (M > 0) {
            const unsigned gx = (unsigned)((ncols + 31) / 32);
            if ((long long)gx * ((n2 + 31) / 32) >= g->num_sms)  // config 4: 256 CTAs of 32 rows
                BIE_LAUNCH(k_struct_gemm<4>, dim3(gx, (unsigned)((n2 + 31) / 32)), 256, 0, st, bd->sX, n2, M, ncols,
                           in, out, stride);
            else
                BIE_LAUNCH(k_struct_gemm<1>, dim3(gx, (unsigned)((n2 + 7) / 8)), 256, 0, st, bd->sX, n2, M, ncols,
                           in, out, stride);
            BIE_LAUNCH(k_struct_corr, (ncols * 32 + 255) / 256, 256, 0, st, bd->sW, bd->sM, n2, M, ncols, out,
                       stride);
            count_launch(2);
            BIE_CUDA_TRY(cudaGetLastError());
        }
        // the wall through the explicit-inverse kernel (rows [wall_lo, N), body M)
        row_lo = g->wall_lo;
        rows_k = g->N - g->wall_lo;
        kb0 = M;
        in += 2LL * g->wall_lo;
        out += 2LL * g->wall_lo;
        blocks = (int)(((long long)2 * rows_k * 32 + threads - 1) / threads);
        if (rows_k == 0) return BIE_OK;
    }
    int v = 0;
    while (v < nvec) {
        int rem = nvec - v;
        if (rem >= 4) {
            BIE_LAUNCH(k_bd_apply<4>, blocks, threads, 0, st, bd->inv, bd->d_off, g->wall_lo, g->n_pore, g->N,
                       kb0, row_lo, rows_k, in, out, stride, v);
            v += 4;
            count_launch();
        } else if (rem >= 2) {
            BIE_LAUNCH(k_bd_apply<2>, blocks, threads, 0, st, bd->inv, bd->d_off, g->wall_lo, g->n_pore, g->N,
                       kb0, row_lo, rows_k, in, out, stride, v);
            v += 2;
            count_launch();
        } else {
            BIE_LAUNCH(k_bd_apply<1>, blocks, threads, 0, st, bd->inv, bd->d_off, g->wall_lo, g->n_pore, g->N,
                       kb0, row_lo, rows_k, in, out, stride, v);
            v += 1;
            count_launch();
        }
        BIE_CUDA_TRY(cudaGetLastError());
    }
    return BIE_OK;
}

}  // namespace bie

using namespace bie;

extern "C" {

int bie_blockdiag_destroy(bie_blockdiag_t h) {
    BlockDiag *bd = as_bd(h);
    if (!bd) {
        set_error("bie_blockdiag_destroy: invalid blockdiag handle");
        return BIE_EINVAL;
    }
    cudaFree(bd->inv);
    cudaFree(bd->d_off);
    cudaFree(bd->sX);
    cudaFree(bd->sW);
    cudaFree(bd->sG);
    cudaFree(bd->sM);
    cudaFree(bd->sD);
    cudaFree(bd->sTmpl);
    bd->magic = 0;
    delete bd;
    return BIE_OK;
}

static int factor_range(Geometry *g, int b0, int b1, bie_blockdiag_t *out, cudaStream_t st, int op = 0) {
    *out = nullptr;
    BlockDiag *bd = new BlockDiag();
    bd->g = g;
    bd->op = op;
    bd->b0 = b0;
    bd->b1 = b1;
    bd->nb = b1 - b0;
    long long off = 0;
    for (int b = b0; b < b1; ++b) {
        int lo = b < g->M ? b * g->n_pore : g->wall_lo;
        int n = b < g->M ? g->n_pore : g->n_outer;
        bd->lo.push_back(lo);
        bd->n.push_back(n);
        bd->off.push_back(off);
        off += 4LL * n * n;
    }
    bd->off.push_back(off);
    bd->row_lo = bd->lo.front();
    bd->row_hi = bd->lo.back() + bd->n.back();
    int *d_flag = nullptr;
    auto fail = [&](int rc) {
        cudaFree(d_flag);
        bie_blockdiag_destroy(reinterpret_cast<bie_blockdiag_t>(bd));
        return rc;
    };
    cudaError_t e = cudaMalloc(&bd->inv, sizeof(double) * (size_t)off);
    if (e != cudaSuccess) return fail(cuda_fail(e, "cudaMalloc(blockdiag inverses)"));
    e = cudaMalloc(&bd->d_off, sizeof(long long) * bd->off.size());
    if (e != cudaSuccess) return fail(cuda_fail(e, "cudaMalloc(blockdiag offsets)"));
    e = cudaMemcpy(bd->d_off, bd->off.data(), sizeof(long long) * bd->off.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return fail(cuda_fail(e, "cudaMemcpy(blockdiag offsets)"));
    e = cudaMalloc(&d_flag, sizeof(int) * (size_t)bd->nb);
    if (e != cudaSuccess) return fail(cuda_fail(e, "cudaMalloc(flags)"));
    e = cudaMemsetAsync(d_flag, 0, sizeof(int) * (size_t)bd->nb, st);
    if (e != cudaSuccess) return fail(cuda_fail(e, "cudaMemsetAsync(flags)"));
    int rc;
    const int np_hi = std::min(b1, g->M);
    if (b0 < np_hi) {  // pores [b0, np_hi)
        BDView pv{bd->inv, 4LL * g->n_pore * g->n_pore, 2 * g->n_pore, np_hi - b0, b0};
        rc = factor_class(g, pv, b0 * g->n_pore, g->n_pore, false, st, d_flag, op);
        if (rc) return fail(rc);
    }
    if (b1 == g->M + 1) {  // the wall
        BDView wv{bd->inv + bd->off[g->M - b0], 0, 2 * g->n_outer, 1, g->M};
        rc = factor_class(g, wv, g->wall_lo, g->n_outer, true, st, d_flag + (g->M - b0), op);
        if (rc) return fail(rc);
    }
    std::vector<int> flags(bd->nb);
    e = cudaMemcpyAsync(flags.data(), d_flag, sizeof(int) * (size_t)bd->nb, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return fail(cuda_fail(e, "cudaMemcpyAsync(flags)"));
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(cuda_fail(e, "bie_blockdiag_factor (kernels)"));
    for (int q = 0; q < bd->nb; ++q) {
        if (flags[q]) {
            const int b = b0 + q;
            set_error("bie_blockdiag_factor: block of body " + std::to_string(b) +
                      (b < g->M ? " (pore)" : " (outer wall)") + " is singular (zero pivot)");
            return fail(BIE_ESINGULAR);
        }
    }
    cudaFree(d_flag);
    *out = reinterpret_cast<bie_blockdiag_t>(bd);
    return BIE_OK;
}

int bie_blockdiag_factor(bie_geometry_t gh, bie_blockdiag_t *out, void *stream) {
    Geometry *g = as_geom(gh);
    if (!g || !out) {
        set_error("bie_blockdiag_factor: invalid geometry handle or null output");
        return BIE_EINVAL;
    }
    return factor_range(g, 0, g->M + 1, out, (cudaStream_t)stream);
}

int bie_blockdiag_factor_slp(bie_geometry_t gh, bie_blockdiag_t *out, void *stream) {
    Geometry *g = as_geom(gh);
    if (!g || !out) {
        set_error("bie_blockdiag_factor_slp: invalid geometry handle or null output");
        return BIE_EINVAL;
    }
    return factor_range(g, 0, g->M + 1, out, (cudaStream_t)stream, 1);
}

int bie_blockdiag_factor_structured(bie_geometry_t gh, bie_blockdiag_t *out, void *stream) {
    Geometry *g = as_geom(gh);
    if (!g || !out) {
        set_error("bie_blockdiag_factor_structured: invalid geometry handle or null output");
        return BIE_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    *out = nullptr;
    BlockDiag *bd = new BlockDiag();
    bd->g = g;
    bd->b0 = 0;
    bd->b1 = g->M + 1;
    bd->nb = g->M + 1;
    bd->structured = 1;
    for (int b = 0; b <= g->M; ++b) {
        bd->lo.push_back(b < g->M ? b * g->n_pore : g->wall_lo);
        bd->n.push_back(b < g->M ? g->n_pore : g->n_outer);
    }
    const long long wsz = 4LL * g->n_outer * g->n_outer;
    bd->off = {0, wsz};  // explicit storage: the wall only
    bd->row_lo = 0;
    bd->row_hi = g->N;
    int *d_flag = nullptr;
    auto fail = [&](int rc) {
        cudaFree(d_flag);
        bie_blockdiag_destroy(reinterpret_cast<bie_blockdiag_t>(bd));
        return rc;
    };
    cudaError_t e = cudaMalloc(&bd->inv, sizeof(double) * (size_t)wsz);
    if (e != cudaSuccess) return fail(cuda_fail(e, "cudaMalloc(wall inverse)"));
    e = cudaMalloc(&bd->d_off, sizeof(long long) * 2);
    if (e != cudaSuccess) return fail(cuda_fail(e, "cudaMalloc(offsets)"));
    e = cudaMemcpy(bd->d_off, bd->off.data(), sizeof(long long) * 2, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return fail(cuda_fail(e, "cudaMemcpy(offsets)"));
    e = cudaMalloc(&d_flag, sizeof(int) * 2);
    if (e != cudaSuccess) return fail(cuda_fail(e, "cudaMalloc(flags)"));
    e = cudaMemsetAsync(d_flag, 0, sizeof(int) * 2, st);
    if (e != cudaSuccess) return fail(cuda_fail(e, "cudaMemsetAsync(flags)"));
    const int n2 = 2 * g->n_pore;
    if (g->M > 0) {  // the reference pore (pore 0): one exact inverse
        e = cudaMalloc(&bd->sX, sizeof(double) * (size_t)n2 * n2);
        if (e == cudaSuccess) e = cudaMalloc(&bd->sW, sizeof(double) * 2 * (size_t)n2);
        if (e == cudaSuccess) e = cudaMalloc(&bd->sG, sizeof(double) * 4);
        if (e == cudaSuccess) e = cudaMalloc(&bd->sM, sizeof(double) * 4 * (size_t)g->M);
        if (e != cudaSuccess) return fail(cuda_fail(e, "cudaMalloc(structured pore blocks)"));
        BDView pv{bd->sX, 0, n2, 1, 0};
        int rc = factor_class(g, pv, 0, g->n_pore, false, st, d_flag, 0);
        if (rc) return fail(rc);
        k_struct_WG<<<1, 256, 0, st>>>(bd->sX, n2, bd->sW, bd->sG);
        count_launch();
    }
    {
        BDView wv{bd->inv, 0, 2 * g->n_outer, 1, g->M};
        int rc = factor_class(g, wv, g->wall_lo, g->n_outer, true, st, d_flag + 1, 0);
        if (rc) return fail(rc);
    }
    int flags[2] = {0, 0};
    double G[4] = {0, 0, 0, 0};
    e = cudaMemcpyAsync(flags, d_flag, sizeof(int) * 2, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && g->M > 0) e = cudaMemcpyAsync(G, bd->sG, sizeof(double) * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(cuda_fail(e, "bie_blockdiag_factor_structured (kernels)"));
    if (flags[0] || flags[1]) {
        set_error(std::string("bie_blockdiag_factor_structured: block of body ") +
                  (flags[0] ? "0 (reference pore)" : std::to_string(g->M) + " (outer wall)") +
                  " is singular (zero pivot)");
        return fail(BIE_ESINGULAR);
    }
    if (g->M > 0) {
        bd->h_M.resize(4 * (size_t)g->M);
        const double r0 = g->h_pore_r[0];
        for (int k = 0; k < g->M; ++k) {
            const double c = (std::log(r0) - std::log(g->h_pore_r[k])) / (4.0 * kPi * g->n_pore);
            const double a00 = 1.0 + c * G[0], a01 = c * G[1], a10 = c * G[2], a11 = 1.0 + c * G[3];
            const double det = a00 * a11 - a01 * a10;
            if (!(std::fabs(det) > 1e-13 * (std::fabs(a00 * a11) + std::fabs(a01 * a10)))) {
                set_error("bie_blockdiag_factor_structured: block of body " + std::to_string(k) +
                          " (pore) is singular (Woodbury capacitance)");
                return fail(BIE_ESINGULAR);
            }
            bd->h_M[4 * k] = c * a11 / det;
            bd->h_M[4 * k + 1] = -c * a01 / det;
            bd->h_M[4 * k + 2] = -c * a10 / det;
            bd->h_M[4 * k + 3] = c * a00 / det;
        }
        e = cudaMemcpy(bd->sM, bd->h_M.data(), sizeof(double) * bd->h_M.size(), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return fail(cuda_fail(e, "cudaMemcpy(M_k)"));
    }
    cudaFree(d_flag);
    *out = reinterpret_cast<bie_blockdiag_t>(bd);
    return BIE_OK;
}

int bie_blockdiag_factor_structured_slp(bie_geometry_t gh, bie_blockdiag_t *out, void *stream) {
    Geometry *g = as_geom(gh);
    if (!g || !out) {
        set_error("bie_blockdiag_factor_structured_slp: invalid geometry handle or null output");
        return BIE_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    *out = nullptr;
    BlockDiag *bd = new BlockDiag();
    bd->g = g;
    bd->b0 = 0;
    bd->b1 = g->M + 1;
    bd->nb = g->M + 1;
    bd->op = 1;
    bd->structured = 2;
    for (int b = 0; b <= g->M; ++b) {
        bd->lo.push_back(b < g->M ? b * g->n_pore : g->wall_lo);
        bd->n.push_back(b < g->M ? g->n_pore : g->n_outer);
    }
    const long long wsz = 4LL * g->n_outer * g->n_outer;
    bd->off = {0, wsz};  // explicit storage: the wall only
    bd->row_lo = 0;
    bd->row_hi = g->N;
    int *d_flag = nullptr;
    auto fail = [&](int rc) {
        cudaFree(d_flag);
        bie_blockdiag_destroy(reinterpret_cast<bie_blockdiag_t>(bd));
        return rc;
    };
    cudaError_t e = cudaMalloc(&bd->inv, sizeof(double) * (size_t)wsz);
    if (e != cudaSuccess) return fail(cuda_fail(e, "cudaMalloc(wall inverse)"));
    e = cudaMalloc(&bd->d_off, sizeof(long long) * 2);
    if (e != cudaSuccess) return fail(cuda_fail(e, "cudaMalloc(offsets)"));
    e = cudaMemcpy(bd->d_off, bd->off.data(), sizeof(long long) * 2, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return fail(cuda_fail(e, "cudaMemcpy(offsets)"));
    e = cudaMalloc(&d_flag, sizeof(int) * 2);
    if (e != cudaSuccess) return fail(cuda_fail(e, "cudaMalloc(flags)"));
    e = cudaMemsetAsync(d_flag, 0, sizeof(int) * 2, st);
    if (e != cudaSuccess) return fail(cuda_fail(e, "cudaMemsetAsync(flags)"));
    const int n = g->n_pore;
    if (g->M > 0) {
        std::vector<double2> t;
        pore_template(n, t);
        e = cudaMalloc(&bd->sD, sizeof(double) * 4 * (size_t)n * g->M);
        if (e == cudaSuccess) e = cudaMalloc(&bd->sTmpl, sizeof(double2) * (size_t)n);
        if (e == cudaSuccess) e = cudaMemcpy(bd->sTmpl, t.data(), sizeof(double2) * (size_t)n, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return fail(cuda_fail(e, "cudaMalloc/cudaMemcpy(circulant pore blocks)"));
        KRWeights kr;
        for (int q = 0; q < 6; ++q) kr.g[q] = g->kr[q];
        k_circ_factor<<<g->M, 256, sizeof(double) * 14 * (size_t)n, st>>>(g->pos, g->w, kr, bd->sTmpl, n, bd->sD,
                                                                         d_flag);
        count_launch();
        e = cudaGetLastError();
        if (e != cudaSuccess) return fail(cuda_fail(e, "k_circ_factor"));
    }
    {
        BDView wv{bd->inv, 0, 2 * g->n_outer, 1, g->M};
        int rc = factor_class(g, wv, g->wall_lo, g->n_outer, true, st, d_flag + 1, 1);
        if (rc) return fail(rc);
    }
    int flags[2] = {0, 0};
    e = cudaMemcpyAsync(flags, d_flag, sizeof(int) * 2, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(cuda_fail(e, "bie_blockdiag_factor_structured_slp (kernels)"));
    if (flags[0] || flags[1]) {
        set_error(std::string("bie_blockdiag_factor_structured_slp: ") +
                  (flags[0] ? "a pore block has a singular Fourier block" : "the outer-wall block is singular") +
                  (flags[0] ? "" : " (zero pivot, body " + std::to_string(g->M) + ")"));
        return fail(BIE_ESINGULAR);
    }
    cudaFree(d_flag);
    *out = reinterpret_cast<bie_blockdiag_t>(bd);
    return BIE_OK;
}

int bie_blockdiag_factor_range(bie_geometry_t gh, int body_begin, int body_end, bie_blockdiag_t *out,
                               void *stream) {
    Geometry *g = as_geom(gh);
    if (!g || !out || body_begin < 0 || body_end > g->M + 1 || body_begin >= body_end) {
        set_error("bie_blockdiag_factor_range: invalid handle/output or body range not in [0, M+1]");
        return BIE_EINVAL;
    }
    return factor_range(g, body_begin, body_end, out, (cudaStream_t)stream);
}

int bie_blockdiag_factor_range_slp(bie_geometry_t gh, int body_begin, int body_end, bie_blockdiag_t *out,
                                   void *stream) {
    Geometry *g = as_geom(gh);
    if (!g || !out || body_begin < 0 || body_end > g->M + 1 || body_begin >= body_end) {
        set_error("bie_blockdiag_factor_range_slp: invalid handle/output or body range not in [0, M+1]");
        return BIE_EINVAL;
    }
    return factor_range(g, body_begin, body_end, out, (cudaStream_t)stream, 1);
}

int bie_blockdiag_rows(bie_blockdiag_t h, int *row_begin, int *row_end) {
    BlockDiag *bd = as_bd(h);
    if (!bd || !row_begin || !row_end) {
        set_error("bie_blockdiag_rows: invalid handle or null output");
        return BIE_EINVAL;
    }
    *row_begin = bd->row_lo;
    *row_end = bd->row_hi;
    return BIE_OK;
}

int bie_blockdiag_apply(bie_blockdiag_t h, const double *in, double *out, int nvec, void *stream) {
    BlockDiag *bd = as_bd(h);
    if (!bd || !in || !out || nvec < 1 || nvec > BIE_MAX_NVEC || in == out) {
        set_error("bie_blockdiag_apply: invalid handle/pointers, nvec out of [1,16], or in == out");
        return BIE_EINVAL;
    }
    return blockdiag_apply_impl(bd, in, out, nvec, (cudaStream_t)stream);
}

int bie_blockdiag_block_inverse(bie_blockdiag_t h, int body, double *host, long long host_len) {
    BlockDiag *bd = as_bd(h);
    if (!bd || !host || body < bd->b0 || body >= bd->b1) {
        set_error("bie_blockdiag_block_inverse: invalid handle, body not in the handle's range, or buffer");
        return BIE_EINVAL;
    }
    if (bd->structured) {
        Geometry *g = bd->g;
        if (body == g->M) {
            const long long n = bd->off[1];
            if (host_len < n) {
                set_error("bie_blockdiag_block_inverse: host buffer too small");
                return BIE_EINVAL;
            }
            BIE_CUDA_TRY(cudaMemcpy(host, bd->inv, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost));
            return BIE_OK;
        }
        const int n2 = 2 * g->n_pore;
        if (bd->structured == 2) {  // B_k^-1 [i][j] = T_i d_k((j - i) mod n) T_j^T
            const int n = g->n_pore;
            if (host_len < (long long)n2 * n2) {
                set_error("bie_blockdiag_block_inverse: host buffer too small");
                return BIE_EINVAL;
            }
            std::vector<double> d(4 * (size_t)n);
            std::vector<double2> t;
            pore_template(n, t);
            BIE_CUDA_TRY(cudaMemcpy(d.data(), bd->sD + 4LL * n * body, sizeof(double) * d.size(),
                                    cudaMemcpyDeviceToHost));
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j) {
                    const double *e = d.data() + 4 * (size_t)((j - i + n) % n);
                    const double ci = t[i].x, si = t[i].y, cj = t[j].x, sj = t[j].y;
                    // P = e T_j^T, then T_i P
                    const double p00 = e[0] * cj - e[1] * sj, p01 = e[0] * sj + e[1] * cj;
                    const double p10 = e[2] * cj - e[3] * sj, p11 = e[2] * sj + e[3] * cj;
                    host[(size_t)(2 * i) * n2 + 2 * j] = ci * p00 - si * p10;
                    host[(size_t)(2 * i) * n2 + 2 * j + 1] = ci * p01 - si * p11;
                    host[(size_t)(2 * i + 1) * n2 + 2 * j] = si * p00 + ci * p10;
                    host[(size_t)(2 * i + 1) * n2 + 2 * j + 1] = si * p01 + ci * p11;
                }
            return BIE_OK;
        }
        // B_k^-1 = X - W M_k Z, Z = U^T X (materialised on the host for inspection)
        if (host_len < (long long)n2 * n2) {
            set_error("bie_blockdiag_block_inverse: host buffer too small");
            return BIE_EINVAL;
        }
        std::vector<double> W(2 * (size_t)n2), Z(2 * (size_t)n2, 0.0);
        BIE_CUDA_TRY(cudaMemcpy(host, bd->sX, sizeof(double) * (size_t)n2 * n2, cudaMemcpyDeviceToHost));
        BIE_CUDA_TRY(cudaMemcpy(W.data(), bd->sW, sizeof(double) * W.size(), cudaMemcpyDeviceToHost));
        for (int i = 0; i < n2; ++i)
            for (int c = 0; c < n2; ++c) Z[(size_t)(i & 1) * n2 + c] += host[(size_t)i * n2 + c];
        const double *Mk = bd->h_M.data() + 4 * (size_t)body;
        for (int i = 0; i < n2; ++i) {
            const double p0 = W[2 * i] * Mk[0] + W[2 * i + 1] * Mk[2];
            const double p1 = W[2 * i] * Mk[1] + W[2 * i + 1] * Mk[3];
            for (int c = 0; c < n2; ++c) host[(size_t)i * n2 + c] -= p0 * Z[c] + p1 * Z[(size_t)n2 + c];
        }
        return BIE_OK;
    }
    body -= bd->b0;
    long long n = bd->off[body + 1] - bd->off[body];
    if (host_len < n) {
        set_error("bie_blockdiag_block_inverse: host buffer too small");
        return BIE_EINVAL;
    }
    BIE_CUDA_TRY(cudaMemcpy(host, bd->inv + bd->off[body], sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost));
    return BIE_OK;
}

}  // extern "C"

BIE_DCHECK_TU(blockdiag)
