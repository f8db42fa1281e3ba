// geometry.cu -- bie_geometry_* and error plumbing (A1 of SURVEY.md s8(a)).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "internal.cuh"

namespace bie {

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
static std::atomic<unsigned long long> g_bd_serial{0};
unsigned long long next_bd_serial() { return ++g_bd_serial; }
int ensure_side_stream(Geometry *g) {
    if (g->side) return BIE_OK;
    BIE_CUDA_TRY(cudaStreamCreateWithFlags(&g->side, cudaStreamNonBlocking));
    BIE_CUDA_TRY(cudaEventCreateWithFlags(&g->ev_fork, cudaEventDisableTiming));
    BIE_CUDA_TRY(cudaEventCreateWithFlags(&g->ev_join, cudaEventDisableTiming));
    return BIE_OK;
}

bool pdl_enabled() {
    static const bool on = [] {
        const char *e = getenv("BIE_PDL");
        return !(e && atoi(e) == 0);
    }();
    return on;
}

void set_error(const std::string &msg) { g_last_error = msg; }

int cuda_fail(cudaError_t e, const char *what) {
    set_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
    if (e == cudaErrorMemoryAllocation) return BIE_ENOMEM;
    return BIE_ECUDA;
}

Geometry *as_geom(bie_geometry_t g) {
    Geometry *p = reinterpret_cast<Geometry *>(g);
    if (!p || p->magic != kGeomMagic) return nullptr;
    return p;
}

BlockDiag *as_bd(bie_blockdiag_t b) {
    BlockDiag *p = reinterpret_cast<BlockDiag *>(b);
    if (!p || p->magic != kBlockMagic) return nullptr;
    return p;
}

// Pore-node template (reading C27 of DESIGN.md): (C_j, S_j) = cos / sin of
// theta_j = 2 pi j / n, CORRECTLY ROUNDED to double.  A 1-ulp difference in a
// pore node position is amplified ~1e4 by the near-tangent cancellation in r.n
// between neighbouring nodes of a small pore far from the origin (measured:
// 2e-12 max-norm at config 4), so the node table must be uniquely defined, not
// "within an ulp".  Exact octant reduction of the integer j, then Taylor
// series in double-double arithmetic (|error| ~ 1e-32) and one final rounding.
namespace {
struct DD {
    double hi, lo;
};
DD two_sum(double a, double b) {
    const double s = a + b, bb = s - a;
    return {s, (a - (s - bb)) + (b - bb)};
}
DD quick_two_sum(double a, double b) {
    const double s = a + b;
    return {s, b - (s - a)};
}
DD dd_add(DD a, DD b) {
    DD s = two_sum(a.hi, b.hi);
    const DD t = two_sum(a.lo, b.lo);
    s.lo += t.hi;
    s = quick_two_sum(s.hi, s.lo);
    s.lo += t.lo;
    return quick_two_sum(s.hi, s.lo);
}
DD dd_mul(DD a, DD b) {
    const double p = a.hi * b.hi;
    const double e = std::fma(a.hi, b.hi, -p) + (a.hi * b.lo + a.lo * b.hi);
    return quick_two_sum(p, e);
}
DD dd_div_d(DD a, double b) {  // a / b, b a small integer
    const double q1 = a.hi / b;
    const double p = q1 * b, pe = std::fma(q1, b, -p);
    const DD r = dd_add(a, DD{-p, -pe});
    const double q2 = r.hi / b;
    return quick_two_sum(q1, q2);
}
// sin and cos of phi in [0, pi/4] (double-double Taylor series)
void dd_sincos(DD phi, DD &sn, DD &cs) {
    const DD z2 = dd_mul(phi, phi);
    DD term = phi, s = phi;
    for (int k = 1; k < 40; ++k) {  // term_k = phi^(2k+1) / (2k+1)!
        term = dd_div_d(dd_mul(term, z2), (double)(2 * k) * (double)(2 * k + 1));
        s = dd_add(s, (k & 1) ? DD{-term.hi, -term.lo} : term);
        if (std::fabs(term.hi) < 1e-36) break;
    }
    DD c = {1.0, 0.0};
    term = {1.0, 0.0};
    for (int k = 1; k < 40; ++k) {  // term_k = phi^(2k) / (2k)!
        term = dd_div_d(dd_mul(term, z2), (double)(2 * k - 1) * (double)(2 * k));
        c = dd_add(c, (k & 1) ? DD{-term.hi, -term.lo} : term);
        if (std::fabs(term.hi) < 1e-36) break;
    }
    sn = s;
    cs = c;
}
}  // namespace

void pore_template(int n, std::vector<double2> &out) {
    const DD pi4 = {0.78539816339744827900, 3.0616169978683830179e-17};  // pi / 4
    out.resize(n);
    for (int j = 0; j < n; ++j) {
        const long long a = 8LL * j;
        const int o = (int)(a / n);
        const long long r = a - (long long)o * n;
        const bool odd = o & 1;
        const DD phi = dd_div_d(dd_mul(pi4, DD{(double)(odd ? n - r : r), 0.0}), (double)n);
        DD sd, cd;
        dd_sincos(phi, sd, cd);
        const double S = sd.hi + sd.lo, C = cd.hi + cd.lo;
        double c, s;  // theta_j = o pi/4 + phi (even o) or (o + 1) pi/4 - phi (odd o)
        switch (o) {
            case 0: c = C; s = S; break;
            case 1: c = S; s = C; break;
            case 2: c = -S; s = C; break;
            case 3: c = -C; s = S; break;
            case 4: c = -C; s = -S; break;
            case 5: c = -S; s = -C; break;
            case 6: c = S; s = -C; break;
            default: c = C; s = -S; break;
        }
        out[j] = make_double2(c, s);
    }
}

// A1 node kernel.  P:l.296-309, P:l.318-319, P:l.354; readings C2, C7, C12, C27.
// Pores (node i = k*n_pore + j), e = template (C_j, S_j):
//   x = c + r e, x' = r(-S, C), x'' = -r e, n = -e, t = x'/|x'|,
//   w = 2 pi r / n_pore, kappa_n = x''.n / |x'|^2.
// Gamma_0 (node i = wall_lo + j): w = |x'| T/n_outer, t = x'/|x'|,
// n = (t_y, -t_x), kappa_n = x''.n / |x'|^2.
// Every node quantity is one fixed sequence of correctly rounded operations
// (explicit _rn intrinsics: no contraction into FMA), so the node table is
// uniquely defined by the inputs (bit-identical to any implementation of the
// same formulas, e.g. the oracle's).
__global__ void k_nodes(int N, int M, int n_pore, int n_outer, double T, const double2 *__restrict__ oxy,
                        const double2 *__restrict__ odxy, const double2 *__restrict__ oddxy,
                        const double4 *__restrict__ pore, const double2 *__restrict__ unit, double2 *pos, double2 *nw,
                        double2 *nrm, double2 *tan, double *w, double *selfc, double *kappa) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    int wall_lo = M * n_pore;
    double2 x, n, t, d1, d2;
    double wi;
    if (i < wall_lo) {
        int k = i / n_pore, j = i - k * n_pore;
        const double4 p = pore[k];
        const double2 e = unit[j];
        d1 = make_double2(-__dmul_rn(p.z, e.y), __dmul_rn(p.z, e.x));
        d2 = make_double2(-__dmul_rn(p.z, e.x), -__dmul_rn(p.z, e.y));
        x = make_double2(__dadd_rn(p.x, __dmul_rn(p.z, e.x)), __dadd_rn(p.y, __dmul_rn(p.z, e.y)));
        n = make_double2(-e.x, -e.y);
        wi = __ddiv_rn(__dmul_rn(2.0 * kPi, p.z), (double)n_pore);
    } else {
        int j = i - wall_lo;
        d1 = odxy[j];
        d2 = oddxy[j];
        x = oxy[j];
    }
    const double sp2 = __dadd_rn(__dmul_rn(d1.x, d1.x), __dmul_rn(d1.y, d1.y));
    const double sp = __dsqrt_rn(sp2);
    t = make_double2(__ddiv_rn(d1.x, sp), __ddiv_rn(d1.y, sp));
    if (i >= wall_lo) {
        n = make_double2(t.y, -t.x);
        wi = __ddiv_rn(__dmul_rn(sp, T), (double)n_outer);
    }
    const double kn = __ddiv_rn(__dadd_rn(__dmul_rn(d2.x, n.x), __dmul_rn(d2.y, n.y)), __dmul_rn(sp, sp));
    pos[i] = x;
    nrm[i] = n;
    tan[i] = t;
    w[i] = wi;
    nw[i] = make_double2(wi * n.x / kPi, wi * n.y / kPi);
    selfc[i] = wi * kn / (2.0 * kPi);
    kappa[i] = kn;
}

// Kapur-Rokhlin sixth-order log-correction weights (P:l.321-330; reading C24
// of DESIGN.md).  gamma_1..gamma_6 solve, for l = 0, 1, 2,
//   2 sum_k gamma_k k^(2l)          = [l == 0]
//   2 sum_k gamma_k k^(2l) log k    = 2 zeta'(-2l),
//   zeta'(0) = -log(2 pi)/2,  zeta'(-2l) = (-1)^l (2l)! zeta(2l+1) / (2 (2 pi)^(2l)),
// computed here in long double: zeta(3), zeta(5) by direct summation to
// n = 10^5 with the integral tail plus its first two Euler-Maclaurin terms,
// then Gaussian elimination with partial pivoting.
static long double zeta_ld(int s) {
    const long n0 = 100000;
    long double acc = 0.0L;
    for (long n = n0 - 1; n >= 1; --n) acc += powl((long double)n, (long double)-s);  // small terms first
    const long double N = (long double)n0;
    acc += powl(N, (long double)(1 - s)) / (long double)(s - 1) + 0.5L * powl(N, (long double)-s) +
           (long double)s / 12.0L * powl(N, (long double)(-s - 1));
    return acc;
}

void kr_weights(double gamma[6]) {
    const long double two_pi = 2.0L * acosl(-1.0L);
    const long double zp[3] = {-0.5L * logl(two_pi), -2.0L * zeta_ld(3) / (2.0L * two_pi * two_pi),
                               24.0L * zeta_ld(5) / (2.0L * powl(two_pi, 4))};
    long double A[6][7];
    for (int l = 0; l < 3; ++l)
        for (int k = 1; k <= 6; ++k) {
            const long double k2l = powl((long double)k, (long double)(2 * l));
            A[l][k - 1] = 2.0L * k2l;
            A[3 + l][k - 1] = 2.0L * k2l * logl((long double)k);
        }
    for (int l = 0; l < 3; ++l) {
        A[l][6] = l == 0 ? 1.0L : 0.0L;
        A[3 + l][6] = 2.0L * zp[l];
    }
    for (int c = 0; c < 6; ++c) {
        int p = c;
        for (int r = c + 1; r < 6; ++r)
            if (fabsl(A[r][c]) > fabsl(A[p][c])) p = r;
        for (int q = 0; q < 7; ++q) std::swap(A[c][q], A[p][q]);
        for (int r = c + 1; r < 6; ++r) {
            const long double f = A[r][c] / A[c][c];
            for (int q = c; q < 7; ++q) A[r][q] -= f * A[c][q];
        }
    }
    long double x[6];
    for (int c = 5; c >= 0; --c) {
        long double t = A[c][6];
        for (int q = c + 1; q < 6; ++q) t -= A[c][q] * x[q];
        x[c] = t / A[c][c];
    }
    for (int k = 0; k < 6; ++k) gamma[k] = (double)x[k];
}

}  // namespace bie

using namespace bie;

extern "C" {

const char *bie_last_error(void) { return g_last_error.c_str(); }

int bie_geometry_destroy(bie_geometry_t gh) {
    Geometry *g = as_geom(gh);
    if (!g) {
        set_error("bie_geometry_destroy: invalid geometry handle");
        return BIE_EINVAL;
    }
    cudaFree(g->pos);
    cudaFree(g->nw);
    cudaFree(g->nrm);
    cudaFree(g->tan);
    cudaFree(g->w);
    cudaFree(g->selfc);
    cudaFree(g->kappa);
    cudaFree(g->pore);
    cudaFree(g->partial);
    cudaFree(g->moments);
    cudaFree(g->stage_in);
    cudaFree(g->stage_out);
    for (cudaEvent_t e : g->prof_ev) cudaEventDestroy(e);
    if (g->sym_trace) {  // BIE_SYM_TRACE=<file>: dump the last symmetric launch's CTA start/end times
        std::vector<unsigned long long> tr(2 * (size_t)g->sym_P);
        if (cudaMemcpy(tr.data(), g->sym_trace, sizeof(unsigned long long) * tr.size(), cudaMemcpyDeviceToHost) ==
            cudaSuccess) {
            if (FILE *f = fopen(getenv("BIE_SYM_TRACE"), "w")) {
                for (size_t q = 0; q < tr.size(); q += 2) fprintf(f, "%llu %llu\n", tr[q], tr[q + 1]);
                fclose(f);
            }
        }
        cudaFree(g->sym_trace);
    }
    cudaFree(g->slp_s);
    cudaFree(g->sym_counter);
    cudaFree(g->pair_counter);
    cudaFree(g->gm.V);
    cudaFree(g->gm.w);
    cudaFree(g->gm.t);
    cudaFree(g->gm.H);
    cudaFree(g->gm.small);
    cudaFree(g->gm.partial);
    if (g->gm.pinned) cudaFreeHost(g->gm.pinned);
    for (auto &ev : g->gm.evs)
        if (ev) cudaEventDestroy(ev);
    if (g->side) cudaStreamDestroy(g->side);
    if (g->bd_hp) cudaStreamDestroy(g->bd_hp);
    for (cudaEvent_t e : g->bd_ev)
        if (e) cudaEventDestroy(e);
    if (g->ev_fork) cudaEventDestroy(g->ev_fork);
    if (g->ev_join) cudaEventDestroy(g->ev_join);
    if (g->gm.gexec) cudaGraphExecDestroy(g->gm.gexec);
    if (g->gm.graph) cudaGraphDestroy(g->gm.graph);
    if (g->gm.cap) cudaStreamDestroy(g->gm.cap);
    cudaFree(g->gmb.V);
    cudaFree(g->gmb.w);
    cudaFree(g->gmb.H);
    cudaFree(g->gmb.small);
    cudaFree(g->gmb.partial);
    if (g->gmb.pinned) cudaFreeHost(g->gmb.pinned);
    cudaFree(g->sym_Q);
    cudaFree(g->sym_off);
    cudaFree(g->sym_acc);
    cudaFree(g->sym_diag);
    g->magic = 0;
    delete g;
    return BIE_OK;
}

int bie_geometry_create(const double *outer_xy, const double *outer_dxy, const double *outer_ddxy, int n_outer,
                        double outer_period, const double *pore_c, const double *pore_r, int n_pores,
                        int nodes_per_pore, bie_geometry_t *out) {
    if (!out || !outer_xy || !outer_dxy || !outer_ddxy || (n_pores > 0 && (!pore_c || !pore_r))) {
        set_error("bie_geometry_create: null pointer argument");
        return BIE_EINVAL;
    }
    *out = nullptr;
    if (n_outer < 16 || (n_outer & 1) || n_pores < 0 ||
        (n_pores > 0 && (nodes_per_pore < 16 || (nodes_per_pore & 1))) || !(outer_period > 0.0)) {
        set_error("bie_geometry_create: n_outer and nodes_per_pore must be even and >= 16, n_pores >= 0, "
                  "outer_period > 0");
        return BIE_EINVAL;
    }
    long long Nll = (long long)n_pores * (n_pores > 0 ? nodes_per_pore : 0) + n_outer;
    if (Nll > (1LL << 28)) {
        set_error("bie_geometry_create: too many nodes");
        return BIE_EINVAL;
    }
    for (int k = 0; k < n_pores; ++k) {
        if (!(pore_r[k] > 0.0) || !std::isfinite(pore_r[k]) || !std::isfinite(pore_c[2 * k]) ||
            !std::isfinite(pore_c[2 * k + 1])) {
            set_error("bie_geometry_create: pore " + std::to_string(k) + " has a non-positive or non-finite radius/centre");
            return BIE_EGEOM;
        }
    }
    for (int j = 0; j < 2 * n_outer; ++j) {
        if (!std::isfinite(outer_xy[j]) || !std::isfinite(outer_dxy[j]) || !std::isfinite(outer_ddxy[j])) {
            set_error("bie_geometry_create: non-finite outer-curve sample");
            return BIE_EGEOM;
        }
    }
    for (int j = 0; j < n_outer; ++j) {
        if (outer_dxy[2 * j] == 0.0 && outer_dxy[2 * j + 1] == 0.0) {
            set_error("bie_geometry_create: outer curve has a zero derivative sample");
            return BIE_EGEOM;
        }
    }
    // Pores must be disjoint and inside Gamma_0 (S:l.36): no two discs overlap, every
    // centre lies inside the outer polygon (winding number) and no outer node lies
    // in a disc.  O(M^2 + M n_outer) on the host.
    for (int a = 0; a < n_pores; ++a) {
        for (int b = a + 1; b < n_pores; ++b) {
            const double dx = pore_c[2 * a] - pore_c[2 * b], dy = pore_c[2 * a + 1] - pore_c[2 * b + 1];
            const double rr = pore_r[a] + pore_r[b];
            if (dx * dx + dy * dy <= rr * rr) {
                set_error("bie_geometry_create: pores " + std::to_string(a) + " and " + std::to_string(b) +
                          " overlap");
                return BIE_EGEOM;
            }
        }
        const double cx = pore_c[2 * a], cy = pore_c[2 * a + 1], r2 = pore_r[a] * pore_r[a];
        int wind = 0;
        for (int j = 0; j < n_outer; ++j) {
            const double x0 = outer_xy[2 * j], y0 = outer_xy[2 * j + 1];
            const int jn = (j + 1) % n_outer;
            const double x1 = outer_xy[2 * jn], y1 = outer_xy[2 * jn + 1];
            if ((x0 - cx) * (x0 - cx) + (y0 - cy) * (y0 - cy) <= r2) {
                set_error("bie_geometry_create: pore " + std::to_string(a) + " crosses the outer wall");
                return BIE_EGEOM;
            }
            const double cross = (x1 - x0) * (cy - y0) - (cx - x0) * (y1 - y0);
            if (y0 <= cy) {
                if (y1 > cy && cross > 0) ++wind;
            } else if (y1 <= cy && cross < 0) {
                --wind;
            }
        }
        if (wind == 0) {
            set_error("bie_geometry_create: pore " + std::to_string(a) + " lies outside the outer wall");
            return BIE_EGEOM;
        }
    }
    Geometry *g = new Geometry();
    g->N = (int)Nll;
    g->M = n_pores;
    g->n_pore = n_pores > 0 ? nodes_per_pore : 0;
    g->n_outer = n_outer;
    g->wall_lo = g->M * g->n_pore;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, dev);
    int N = g->N;
    int rc = BIE_OK;
    double2 *d_oxy = nullptr, *d_odxy = nullptr, *d_oddxy = nullptr, *d_unit = nullptr;
    std::vector<double4> hp(n_pores > 0 ? n_pores : 1);
    double wall_len = 0.0;
    auto fail = [&](int code) {
        cudaFree(d_oxy);
        cudaFree(d_odxy);
        cudaFree(d_oddxy);
        cudaFree(d_unit);
        bie_geometry_destroy(reinterpret_cast<bie_geometry_t>(g));
        return code;
    };
#define TRY(expr)                                             \
    do {                                                      \
        cudaError_t _e = (expr);                              \
        if (_e != cudaSuccess) return fail(cuda_fail(_e, #expr)); \
    } while (0)
    TRY(cudaMalloc(&g->pos, sizeof(double2) * N));
    TRY(cudaMalloc(&g->nw, sizeof(double2) * N));
    TRY(cudaMalloc(&g->nrm, sizeof(double2) * N));
    TRY(cudaMalloc(&g->tan, sizeof(double2) * N));
    TRY(cudaMalloc(&g->w, sizeof(double) * N));
    TRY(cudaMalloc(&g->selfc, sizeof(double) * N));
    TRY(cudaMalloc(&g->kappa, sizeof(double) * N));
    TRY(cudaMalloc(&g->pore, sizeof(double4) * (n_pores > 0 ? n_pores : 1)));
    TRY(cudaMalloc(&d_oxy, sizeof(double2) * n_outer));
    TRY(cudaMalloc(&d_odxy, sizeof(double2) * n_outer));
    TRY(cudaMalloc(&d_oddxy, sizeof(double2) * n_outer));
    TRY(cudaMemcpy(d_oxy, outer_xy, sizeof(double2) * n_outer, cudaMemcpyHostToDevice));
    TRY(cudaMemcpy(d_odxy, outer_dxy, sizeof(double2) * n_outer, cudaMemcpyHostToDevice));
    TRY(cudaMemcpy(d_oddxy, outer_ddxy, sizeof(double2) * n_outer, cudaMemcpyHostToDevice));
    {
        std::vector<double2> unit;
        pore_template(std::max(g->n_pore, 1), unit);
        TRY(cudaMalloc(&d_unit, sizeof(double2) * unit.size()));
        TRY(cudaMemcpy(d_unit, unit.data(), sizeof(double2) * unit.size(), cudaMemcpyHostToDevice));
    }
    // |Gamma_k| = sum_j w_j over the pore's nodes (reading C5); on an equispaced
    // circle every w_j = 2 pi r / n, so the sum is n * w (computed the same way
    // as the kernel's w to keep the ratio w_j/|Gamma_k| exact).
    for (int k = 0; k < n_pores; ++k) {
        double wk = 2.0 * kPi * pore_r[k] / (double)nodes_per_pore;
        double len = 0.0;
        for (int j = 0; j < nodes_per_pore; ++j) len += wk;
        hp[k] = make_double4(pore_c[2 * k], pore_c[2 * k + 1], pore_r[k], len);
        g->h_pore_r.push_back(pore_r[k]);
    }
    TRY(cudaMemcpy(g->pore, hp.data(), sizeof(double4) * (n_pores > 0 ? n_pores : 1), cudaMemcpyHostToDevice));
    k_nodes<<<(N + 255) / 256, 256>>>(N, g->M, g->n_pore, n_outer, outer_period, d_oxy, d_odxy, d_oddxy, g->pore,
                                      d_unit, g->pos, g->nw, g->nrm, g->tan, g->w, g->selfc, g->kappa);
    count_launch();
    TRY(cudaGetLastError());
    {
        std::vector<double> hw(n_outer);
        TRY(cudaMemcpy(hw.data(), g->w + g->wall_lo, sizeof(double) * n_outer, cudaMemcpyDeviceToHost));
        for (int j = 0; j < n_outer; ++j) wall_len += hw[j];
        g->wall_len = wall_len;
    }
    TRY(cudaMalloc(&g->moments, sizeof(double) * (size_t)BIE_MAX_NVEC * (3 * (size_t)(n_pores > 0 ? n_pores : 1) + 1)));
    TRY(cudaMalloc(&g->stage_in, sizeof(double) * (size_t)BIE_MAX_NVEC * 2 * N));
    TRY(cudaMalloc(&g->stage_out, sizeof(double) * (size_t)BIE_MAX_NVEC * 2 * N));
    rc = build_schedules(g);
    if (rc != BIE_OK) return fail(rc);
    kr_weights(g->kr);
    TRY(cudaDeviceSynchronize());
#undef TRY
    cudaFree(d_oxy);
    cudaFree(d_odxy);
    cudaFree(d_oddxy);
    cudaFree(d_unit);
    *out = reinterpret_cast<bie_geometry_t>(g);
    return BIE_OK;
}

int bie_geometry_info(bie_geometry_t gh, int *N, int *M) {
    Geometry *g = as_geom(gh);
    if (!g || !N || !M) {
        set_error("bie_geometry_info: invalid handle or null output");
        return BIE_EINVAL;
    }
    *N = g->N;
    *M = g->M;
    return BIE_OK;
}

int bie_geometry_nodes(bie_geometry_t gh, double *pos_host) {
    Geometry *g = as_geom(gh);
    if (!g || !pos_host) {
        set_error("bie_geometry_nodes: invalid handle or null output");
        return BIE_EINVAL;
    }
    BIE_CUDA_TRY(cudaMemcpy(pos_host, g->pos, sizeof(double2) * g->N, cudaMemcpyDeviceToHost));
    return BIE_OK;
}

int bie_geometry_node_table(bie_geometry_t gh, double *pos, double *nrm, double *tan, double *w, double *kappa) {
    Geometry *g = as_geom(gh);
    if (!g || !pos || !nrm || !tan || !w || !kappa) {
        set_error("bie_geometry_node_table: invalid handle or null output");
        return BIE_EINVAL;
    }
    const size_t N = (size_t)g->N;
    BIE_CUDA_TRY(cudaMemcpy(pos, g->pos, sizeof(double2) * N, cudaMemcpyDeviceToHost));
    BIE_CUDA_TRY(cudaMemcpy(nrm, g->nrm, sizeof(double2) * N, cudaMemcpyDeviceToHost));
    BIE_CUDA_TRY(cudaMemcpy(tan, g->tan, sizeof(double2) * N, cudaMemcpyDeviceToHost));
    BIE_CUDA_TRY(cudaMemcpy(w, g->w, sizeof(double) * N, cudaMemcpyDeviceToHost));
    BIE_CUDA_TRY(cudaMemcpy(kappa, g->kappa, sizeof(double) * N, cudaMemcpyDeviceToHost));
    return BIE_OK;
}

int bie_pore_template(int n, double *unit) {
    if (!unit || n < 1) {
        set_error("bie_pore_template: null output or n < 1");
        return BIE_EINVAL;
    }
    std::vector<double2> u;
    pore_template(n, u);
    std::memcpy(unit, u.data(), sizeof(double2) * (size_t)n);
    return BIE_OK;
}

long long bie_launch_count(void) { return g_launches.load(); }

int bie_profile_begin(bie_geometry_t gh) {
    Geometry *g = as_geom(gh);
    if (!g) {
        set_error("bie_profile_begin: invalid geometry handle");
        return BIE_EINVAL;
    }
    g->prof = true;
    g->prof_used = 0;
    return BIE_OK;
}

int bie_profile_end(bie_geometry_t gh, double *ms_moments, double *ms_pairs, double *ms_epilogue, int *applies) {
    Geometry *g = as_geom(gh);
    if (!g || !ms_moments || !ms_pairs || !ms_epilogue || !applies) {
        set_error("bie_profile_end: invalid handle or null output");
        return BIE_EINVAL;
    }
    double m = 0, p = 0, e = 0;
    for (size_t q = 0; q + 4 <= g->prof_used; q += 4) {
        BIE_CUDA_TRY(cudaEventSynchronize(g->prof_ev[q + 3]));
        float a = 0, b = 0, c = 0;
        BIE_CUDA_TRY(cudaEventElapsedTime(&a, g->prof_ev[q], g->prof_ev[q + 1]));
        BIE_CUDA_TRY(cudaEventElapsedTime(&b, g->prof_ev[q + 1], g->prof_ev[q + 2]));
        BIE_CUDA_TRY(cudaEventElapsedTime(&c, g->prof_ev[q + 2], g->prof_ev[q + 3]));
        m += a;
        p += b;
        e += c;
    }
    *ms_moments = m;
    *ms_pairs = p;
    *ms_epilogue = e;
    *applies = (int)(g->prof_used / 4);
    g->prof = false;
    g->prof_used = 0;
    return BIE_OK;
}

int bie_kr_weights(double *gamma) {
    if (!gamma) {
        set_error("bie_kr_weights: null output");
        return BIE_EINVAL;
    }
    kr_weights(gamma);
    return BIE_OK;
}

}  // extern "C"

BIE_DCHECK_TU(geometry)
