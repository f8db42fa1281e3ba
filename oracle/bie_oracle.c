/*
 * bie_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for the hot path of
 * arxiv 1609.04484 as scoped in SURVEY.md s8: the completed Stokes
 * double-layer (DLP) boundary operator, its per-body block-diagonal (BD)
 * preconditioner (dense LU with partial pivoting + explicit inverse), and
 * left-preconditioned full GMRES.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA library under
 * paper_1609_04484_b200/csrc, and must never be on the product path.
 *
 * Build: gcc -O3 -fno-fast-math -ffp-contract=off -fopenmp -shared -fPIC
 * (no FMA contraction, sequential in-row sums; OpenMP only over target rows,
 * blocks, or independent columns).
 *
 * Citations: P:l.N = /root/reference/PAPER.md line N; readings C1..C19 are
 * listed in DESIGN.md s3 (taken from SURVEY.md s8(c)).
 *
 * It also holds the paper's own single-layer operator with the Kapur-Rokhlin
 * correction (NEXT-1; readings C24-C26), pinned by tests/test_oracle_slp.py
 * (periodic log integral, sixth-order convergence against Bessel closed
 * forms, circle closed forms, the normal null space, an exact Stokes flow).
 *
 * Parity pins (tests/test_oracle_*.py): Gauss identities (V1), Bessel circle
 * integral (V2), null space of the bare operator (V3), completion closed forms
 * (V4), Couette flow (V5), the paper's Stokeslet/rotlet exact solution (V6),
 * brute force / long-double / symmetry checks (V7), GMRES and BD special
 * cases (V8), shear-flow density structure (V9), pore-block universality
 * (V10).  No function here is "parity unpinned".
 */
#include <math.h>
#include <quadmath.h>
#include <stdlib.h>
#include <string.h>

#define ORA_PI 3.14159265358979323846

#define ORA_D_ONLY 1u /* PV sum + self term only (no -1/2 I, no N0, no completion) */

/* ---------------------------------------------------------------------------
 * A1: node table.  P:l.296-309 (collocation points), P:l.318-319 and P:l.354
 * (w_j = arclength x quadrature weight), reading C7 (periodic trapezoid),
 * C2 (normal points out of the fluid domain), C12 (node start/direction).
 *
 * Outer wall Gamma_0: samples x(t_j), x'(t_j), x''(t_j), t_j = j T/n_outer, CCW.
 *   w_j  = |x'(t_j)| T / n_outer
 *   t_j  = x'/|x'|,  n_j = (t_y, -t_x)       (outward of Omega_0 = out of fluid)
 *   kn_j = (x'' . n_j) / |x'|^2              (= x_ss . n, x_ss = d2x/ds2)
 * Pore k (circle c_k, r_k), theta_j = 2 pi j / n_pore:
 *   x = c + r (cos, sin), x' = r(-sin, cos), x'' = -r(cos, sin)
 *   n = -(cos, sin)                          (into the pore = out of fluid)
 *   w = 2 pi r / n_pore, t = (-sin, cos), kn = (x''.n)/|x'|^2 = 1/r
 * Dof order: pores 1..M (node k*n_pore + j), then Gamma_0 (P:l.734-736).
 * ------------------------------------------------------------------------- */
/* Pore template (reading C27): (cos, sin)(2 pi j / n) correctly rounded to
 * double -- exact octant reduction of the integer j, quad-precision
 * (libquadmath, 113-bit) cos/sin of the reduced angle in [0, pi/4], one
 * rounding.  Node positions are ill-conditioned for the operator (1 ulp moves
 * the matvec by ~1e-12 at config 4), so the table must be uniquely defined. */
void ora_pore_template(int n, double *unit)
{
    for (int j = 0; j < n; ++j) {
        long long a = 8LL * j;
        int o = (int)(a / n);
        long long r = a - (long long)o * n;
        long long k = (o & 1) ? n - r : r;
        __float128 phi = (M_PIq / 4) * (__float128)k / (__float128)n;
        double C = (double)cosq(phi), S = (double)sinq(phi), c, s;
        switch (o) { /* theta = o pi/4 + phi (o even) or (o + 1) pi/4 - phi (o odd) */
        case 0: c = C; s = S; break;
        case 1: c = S; s = C; break;
        case 2: c = -S; s = C; break;
        case 3: c = -C; s = S; break;
        case 4: c = -C; s = -S; break;
        case 5: c = -S; s = -C; break;
        case 6: c = S; s = -C; break;
        default: c = C; s = -S; break;
        }
        unit[2 * j] = c;
        unit[2 * j + 1] = s;
    }
}

int ora_nodes(const double *oxy, const double *odxy, const double *oddxy, int n_outer, double T,
              const double *pc, const double *pr, int M, int n_pore,
              double *x, double *nrm, double *w, double *tan, double *kn)
{
    int i = 0;
    double *unit = (double *)malloc(2 * (size_t)(n_pore > 0 ? n_pore : 1) * sizeof(double));
    ora_pore_template(n_pore, unit);
    for (int k = 0; k < M; ++k) {
        for (int j = 0; j < n_pore; ++j, ++i) {
            double c = unit[2 * j], s = unit[2 * j + 1];
            double r = pr[k];
            double dx = -r * s, dy = r * c;       /* x'  */
            double ddx = -r * c, ddy = -r * s;    /* x'' */
            double sp = sqrt(dx * dx + dy * dy);
            x[2 * i] = pc[2 * k] + r * c;
            x[2 * i + 1] = pc[2 * k + 1] + r * s;
            tan[2 * i] = dx / sp;
            tan[2 * i + 1] = dy / sp;
            nrm[2 * i] = -c;
            nrm[2 * i + 1] = -s;
            w[i] = 2.0 * ORA_PI * r / (double)n_pore;
            kn[i] = (ddx * nrm[2 * i] + ddy * nrm[2 * i + 1]) / (sp * sp);
        }
    }
    free(unit);
    for (int j = 0; j < n_outer; ++j, ++i) {
        double dx = odxy[2 * j], dy = odxy[2 * j + 1];
        double sp = sqrt(dx * dx + dy * dy);
        double tx = dx / sp, ty = dy / sp;
        x[2 * i] = oxy[2 * j];
        x[2 * i + 1] = oxy[2 * j + 1];
        tan[2 * i] = tx;
        tan[2 * i + 1] = ty;
        nrm[2 * i] = ty;
        nrm[2 * i + 1] = -tx;
        w[i] = sp * T / (double)n_outer;
        kn[i] = (oddxy[2 * j] * nrm[2 * i] + oddxy[2 * j + 1] * nrm[2 * i + 1]) / (sp * sp);
    }
    return i;
}

/* Node table passed around by the oracle. */
typedef struct {
    int N, M, n_pore;
    const double *x, *nrm, *w, *tan, *kn; /* from ora_nodes */
    const double *pc, *pr;                /* pore centres (2M), radii (M) */
    int op;                               /* 0: completed DLP; 1: SLP + Kapur-Rokhlin (NEXT-1) */
    const double *gam;                    /* op 1: KR corrections gamma_1..gamma_6 */
} ora_geom;

#define ORA_OP_SLP 1
static void ora_slp_row(const ora_geom *g, const double *sig, int i, double *yo);

/* ---------------------------------------------------------------------------
 * A2: moments of the completion (reading C5), per density vector.
 *   |Gamma_k| = sum_{j in Gamma_k} w_j
 *   lambda_k  = (1/|Gamma_k|) sum_{j in Gamma_k} w_j sigma_j
 *   mu_k      = (1/(|Gamma_k| r_k)) sum_{j in Gamma_k} w_j sigma_j . (x_j - c_k)^perp,
 *               (a,b)^perp = (b,-a)   (P:l.956)
 *   nu        = (1/|Gamma_0|) sum_{j in Gamma_0} w_j n_j . sigma_j
 * ------------------------------------------------------------------------- */
static void ora_moments(const ora_geom *g, const double *sig, double *lam, double *mu, double *nu)
{
    int np = g->n_pore;
    for (int k = 0; k < g->M; ++k) {
        double len = 0.0, lx = 0.0, ly = 0.0, m = 0.0;
        for (int j = k * np; j < (k + 1) * np; ++j) {
            double px = g->x[2 * j + 1] - g->pc[2 * k + 1];     /* (x - c)^perp, first comp = y */
            double py = -(g->x[2 * j] - g->pc[2 * k]);          /* second comp = -x */
            len += g->w[j];
            lx += g->w[j] * sig[2 * j];
            ly += g->w[j] * sig[2 * j + 1];
            m += g->w[j] * (sig[2 * j] * px + sig[2 * j + 1] * py);
        }
        lam[2 * k] = lx / len;
        lam[2 * k + 1] = ly / len;
        mu[k] = m / (len * g->pr[k]);
    }
    double len0 = 0.0, s0 = 0.0;
    for (int j = g->M * np; j < g->N; ++j) {
        len0 += g->w[j];
        s0 += g->w[j] * (g->nrm[2 * j] * sig[2 * j] + g->nrm[2 * j + 1] * sig[2 * j + 1]);
    }
    *nu = s0 / len0;
}

/* ---------------------------------------------------------------------------
 * The completed operator applied to one density, row i (2 outputs).
 *
 *   y_i = -1/2 sigma_i                                                  [jump, C3]
 *       + sum_{j != i, ascending} (w_j/pi)(r.n_j)(r.sigma_j) r / rho^4   [P:l.243-248 with
 *                                                          trapezoid weights P:l.310-319]
 *       + (w_i/(2 pi)) kn_i (t_i.sigma_i) t_i                          [diagonal limit, C4]
 *       + [i in Gamma_0] nu n_i                                         [N0, C5]
 *       + sum_k (1/4pi)(-log rho_ik I + r r^T/rho_ik^2) lambda_k
 *               + r_k (r^perp/rho_ik^2) mu_k,   r = x_i - c_k           [completion, C5;
 *                                           Stokeslet/rotlet forms of P:l.944-948]
 * with r = x_i - x_j, rho = |r|.  D_ONLY keeps only the DLP sum and the self term.
 * ------------------------------------------------------------------------- */
static void ora_row(const ora_geom *g, const double *sig, const double *lam, const double *mu,
                    double nu, unsigned flags, int i, double *yo)
{
    double xi = g->x[2 * i], yi = g->x[2 * i + 1];
    double ux = 0.0, uy = 0.0;
    for (int j = 0; j < g->N; ++j) {
        if (j == i)
            continue;
        double rx = xi - g->x[2 * j];
        double ry = yi - g->x[2 * j + 1];
        double rho2 = rx * rx + ry * ry;
        double rn = rx * g->nrm[2 * j] + ry * g->nrm[2 * j + 1];
        double rs = rx * sig[2 * j] + ry * sig[2 * j + 1];
        double coef = (g->w[j] / ORA_PI) * rn * rs / (rho2 * rho2);
        ux += coef * rx;
        uy += coef * ry;
    }
    /* self term (diagonal limit of the kernel times the trapezoid weight) */
    {
        double tx = g->tan[2 * i], ty = g->tan[2 * i + 1];
        double ts = tx * sig[2 * i] + ty * sig[2 * i + 1];
        double a = (g->w[i] / (2.0 * ORA_PI)) * g->kn[i] * ts;
        ux += a * tx;
        uy += a * ty;
    }
    if (!(flags & ORA_D_ONLY)) {
        ux += -0.5 * sig[2 * i];
        uy += -0.5 * sig[2 * i + 1];
        if (i >= g->M * g->n_pore) {
            ux += nu * g->nrm[2 * i];
            uy += nu * g->nrm[2 * i + 1];
        }
        for (int k = 0; k < g->M; ++k) {
            double rx = xi - g->pc[2 * k];
            double ry = yi - g->pc[2 * k + 1];
            double rho2 = rx * rx + ry * ry;
            double lg = 0.5 * log(rho2); /* log rho */
            double rl = rx * lam[2 * k] + ry * lam[2 * k + 1];
            ux += (1.0 / (4.0 * ORA_PI)) * (-lg * lam[2 * k] + rx * rl / rho2);
            uy += (1.0 / (4.0 * ORA_PI)) * (-lg * lam[2 * k + 1] + ry * rl / rho2);
            ux += g->pr[k] * (ry / rho2) * mu[k];
            uy += g->pr[k] * (-rx / rho2) * mu[k];
        }
    }
    yo[0] = ux;
    yo[1] = uy;
}

static void ora_apply_g(const ora_geom *g, const double *sig, double *out, unsigned flags,
                        const int *rows, int nrows)
{
    double *lam = (double *)calloc(2 * (size_t)(g->M > 0 ? g->M : 1), sizeof(double));
    double *mu = (double *)calloc((size_t)(g->M > 0 ? g->M : 1), sizeof(double));
    double nu = 0.0;
    if (!(flags & ORA_D_ONLY) && g->op != ORA_OP_SLP)
        ora_moments(g, sig, lam, mu, &nu);
    int n = rows ? nrows : g->N;
#pragma omp parallel for schedule(dynamic, 16)
    for (int q = 0; q < n; ++q) {
        int i = rows ? rows[q] : q;
        if (g->op == ORA_OP_SLP)
            ora_slp_row(g, sig, i, out + 2 * (size_t)q);
        else
            ora_row(g, sig, lam, mu, nu, flags, i, out + 2 * (size_t)q);
    }
    free(lam);
    free(mu);
}

/* Public: out = A sigma for nvec densities ([nvec][2N] -> [nvec][2*nrows]). */
void ora_apply(int N, int M, int n_pore, const double *x, const double *nrm, const double *w,
               const double *tan, const double *kn, const double *pc, const double *pr,
               const double *sigma, double *out, int nvec, unsigned flags, const int *rows, int nrows)
{
    ora_geom g = {N, M, n_pore, x, nrm, w, tan, kn, pc, pr, 0, NULL};
    int n = rows ? nrows : N;
    for (int v = 0; v < nvec; ++v)
        ora_apply_g(&g, sigma + (size_t)v * 2 * N, out + (size_t)v * 2 * n, flags, rows, nrows);
}

/* ---------------------------------------------------------------------------
 * Off-surface velocity u(x) = D[sigma](x) + completion fields (no jump, no
 * self term, no N0 -- those belong to the boundary operator only).
 * Trapezoid evaluation as in P:l.346-354 (eq. stokesSLP_discretized, with the
 * DLP kernel of P:l.243-246 in place of G).
 * ------------------------------------------------------------------------- */
void ora_field(int N, int M, int n_pore, const double *x, const double *nrm, const double *w,
               const double *pc, const double *pr, const double *sig,
               const double *tgt, int ntgt, double *u)
{
    ora_geom g = {N, M, n_pore, x, nrm, w, NULL, NULL, pc, pr, 0, NULL};
    double *lam = (double *)calloc(2 * (size_t)(M > 0 ? M : 1), sizeof(double));
    double *mu = (double *)calloc((size_t)(M > 0 ? M : 1), sizeof(double));
    double nu = 0.0;
    ora_moments(&g, sig, lam, mu, &nu);
#pragma omp parallel for schedule(dynamic, 16)
    for (int q = 0; q < ntgt; ++q) {
        double xi = tgt[2 * q], yi = tgt[2 * q + 1];
        double ux = 0.0, uy = 0.0;
        for (int j = 0; j < N; ++j) {
            double rx = xi - x[2 * j];
            double ry = yi - x[2 * j + 1];
            double rho2 = rx * rx + ry * ry;
            double rn = rx * nrm[2 * j] + ry * nrm[2 * j + 1];
            double rs = rx * sig[2 * j] + ry * sig[2 * j + 1];
            double coef = (w[j] / ORA_PI) * rn * rs / (rho2 * rho2);
            ux += coef * rx;
            uy += coef * ry;
        }
        for (int k = 0; k < M; ++k) {
            double rx = xi - pc[2 * k];
            double ry = yi - pc[2 * k + 1];
            double rho2 = rx * rx + ry * ry;
            double lg = 0.5 * log(rho2);
            double rl = rx * lam[2 * k] + ry * lam[2 * k + 1];
            ux += (1.0 / (4.0 * ORA_PI)) * (-lg * lam[2 * k] + rx * rl / rho2);
            uy += (1.0 / (4.0 * ORA_PI)) * (-lg * lam[2 * k + 1] + ry * rl / rho2);
            ux += pr[k] * (ry / rho2) * mu[k];
            uy += pr[k] * (-rx / rho2) * mu[k];
        }
        u[2 * q] = ux;
        u[2 * q + 1] = uy;
    }
    free(lam);
    free(mu);
}


/* ---------------------------------------------------------------------------
 * NEXT-1: the paper's own operator -- the Stokes single-layer
 * potential with the Kapur-Rokhlin sixth-order correction.
 *   P:l.270-276 (eq. stokesSLP):  G(x, y) = (1/4pi)(-log rho I + r r^T/rho^2),
 *   P:l.310-319 (eq. dense):      f_i = sum_j w_j G(x_i, x_j) sigma_j,
 *   P:l.321-330: "identical to the trapezoid rule, except that the weights are
 *   modified at the six nodes to the left and right of the singularity".
 * Weights (readings C24-C25): for target i on closed curve Gamma
 * (a pore or Gamma_0, n nodes, periodic local index),
 *   W_ii = 0;  W_ij = w_j (1 + gamma_k) if j is on Gamma at periodic offset
 *   +-k, 1 <= k <= 6;  W_ij = w_j otherwise (other offsets, other curves).
 * gamma_1..gamma_6 are passed in (oracle/__init__.py: kr_weights()).
 * ------------------------------------------------------------------------- */
static void ora_curve(const ora_geom *g, int i, int *lo, int *n)
{
    if (i < g->M * g->n_pore) {
        *lo = (i / g->n_pore) * g->n_pore;
        *n = g->n_pore;
    } else {
        *lo = g->M * g->n_pore;
        *n = g->N - *lo;
    }
}

static double ora_slp_weight(const ora_geom *g, int i, int j)
{
    if (j == i)
        return 0.0;
    int lo_i, n_i, lo_j, n_j;
    ora_curve(g, i, &lo_i, &n_i);
    ora_curve(g, j, &lo_j, &n_j);
    if (lo_i != lo_j)
        return g->w[j];
    int d = ((j - i) % n_i + n_i) % n_i; /* periodic offset on the curve */
    int k = d < n_i - d ? d : n_i - d;
    if (k <= 6)
        return g->w[j] * (1.0 + g->gam[k - 1]);
    return g->w[j];
}

/* G(x, y) sigma with the 1/4pi factor; r = x - y. */
static void ora_slp_kernel(double rx, double ry, double sx, double sy, double *gx, double *gy)
{
    double rho2 = rx * rx + ry * ry;
    double lg = 0.5 * log(rho2); /* log rho */
    double rs = rx * sx + ry * sy;
    *gx = (1.0 / (4.0 * ORA_PI)) * (-lg * sx + rx * rs / rho2);
    *gy = (1.0 / (4.0 * ORA_PI)) * (-lg * sy + ry * rs / rho2);
}

static void ora_slp_row(const ora_geom *g, const double *sig, int i, double *yo)
{
    double xi = g->x[2 * i], yi = g->x[2 * i + 1];
    double ux = 0.0, uy = 0.0;
    for (int j = 0; j < g->N; ++j) {
        if (j == i)
            continue;
        double W = ora_slp_weight(g, i, j);
        double gx, gy;
        ora_slp_kernel(xi - g->x[2 * j], yi - g->x[2 * j + 1], sig[2 * j], sig[2 * j + 1], &gx, &gy);
        ux += W * gx;
        uy += W * gy;
    }
    yo[0] = ux;
    yo[1] = uy;
}

/* out = A_SLP sigma for nvec densities ([nvec][2N] -> [nvec][2*nrows]). */
void ora_slp_apply(int N, int M, int n_pore, const double *x, const double *w, const double *gam,
                   const double *sigma, double *out, int nvec, const int *rows, int nrows)
{
    ora_geom g = {N, M, n_pore, x, NULL, w, NULL, NULL, NULL, NULL, ORA_OP_SLP, gam};
    int n = rows ? nrows : N;
    for (int v = 0; v < nvec; ++v)
        ora_apply_g(&g, sigma + (size_t)v * 2 * N, out + (size_t)v * 2 * n, 0u, rows, nrows);
}

/* Off-surface velocity u(x) = sum_j w_j G(x, x_j) sigma_j: the trapezoid rule
 * of P:l.346-354 (eq. stokesSLP_discretized), no correction. */
void ora_slp_field(int N, const double *x, const double *w, const double *sig, const double *tgt, int ntgt,
                   double *u)
{
#pragma omp parallel for schedule(dynamic, 16)
    for (int q = 0; q < ntgt; ++q) {
        double ux = 0.0, uy = 0.0;
        for (int j = 0; j < N; ++j) {
            double gx, gy;
            ora_slp_kernel(tgt[2 * q] - x[2 * j], tgt[2 * q + 1] - x[2 * j + 1], sig[2 * j], sig[2 * j + 1],
                           &gx, &gy);
            ux += w[j] * gx;
            uy += w[j] * gy;
        }
        u[2 * q] = ux;
        u[2 * q + 1] = uy;
    }
}

/* BD block of the SLP operator for body b: entries W_ij G(x_i, x_j) for i, j
 * on body b (2x2 node blocks, zero for i == j). */
static void ora_slp_block_g(const ora_geom *g, int b, double *B)
{
    int lo, hi;
    if (b < g->M) {
        lo = b * g->n_pore;
        hi = lo + g->n_pore;
    } else {
        lo = g->M * g->n_pore;
        hi = g->N;
    }
    int n2 = 2 * (hi - lo);
    for (int i = lo; i < hi; ++i) {
        for (int j = lo; j < hi; ++j) {
            double e00 = 0.0, e01 = 0.0, e10 = 0.0, e11 = 0.0;
            if (j != i) {
                double W = ora_slp_weight(g, i, j);
                double gx, gy;
                double rx = g->x[2 * i] - g->x[2 * j], ry = g->x[2 * i + 1] - g->x[2 * j + 1];
                ora_slp_kernel(rx, ry, W, 0.0, &gx, &gy); /* column for sigma = (1, 0) */
                e00 = gx;
                e10 = gy;
                ora_slp_kernel(rx, ry, 0.0, W, &gx, &gy); /* column for sigma = (0, 1) */
                e01 = gx;
                e11 = gy;
            }
            size_t r0 = (size_t)(2 * (i - lo)), c0 = (size_t)(2 * (j - lo));
            B[r0 * n2 + c0] = e00;
            B[r0 * n2 + c0 + 1] = e01;
            B[(r0 + 1) * n2 + c0] = e10;
            B[(r0 + 1) * n2 + c0 + 1] = e11;
        }
    }
}

void ora_slp_block(int N, int M, int n_pore, const double *x, const double *w, const double *gam, int b,
                   double *B)
{
    ora_geom g = {N, M, n_pore, x, NULL, w, NULL, NULL, NULL, NULL, ORA_OP_SLP, gam};
    ora_slp_block_g(&g, b, B);
}

/* ---------------------------------------------------------------------------
 * A6: BD blocks.  P:l.651-657: "diagonal blocks corresponding to the
 * self-interactions of the individual pores and the outer boundary ...
 * assembled, factorized, and inverted exactly".  Block b = rows and columns
 * of the completed operator restricted to body b (b < M: pore b, b == M:
 * Gamma_0).  Entry (2x2) for nodes i, j of body b, from the formula above
 * written per column:
 *   i != j : (w_j/pi)(r.n_j) r r^T / rho^4
 *   i == j : (w_i/2pi) kn_i t_i t_i^T - 1/2 I
 *   pore k : + (w_j/|Gamma_k|) [ S(x_i - c_k) + R(x_i - c_k) ((x_j - c_k)^perp)^T ]
 *            S(r) = (1/4pi)(-log rho I + r r^T/rho^2),  R(r) = r^perp / rho^2
 *   wall   : + n_i n_j^T w_j / |Gamma_0|
 * Row-major, unknown index 2*local_node + component.
 * ------------------------------------------------------------------------- */
static void ora_body_range(const ora_geom *g, int b, int *lo, int *hi)
{
    if (b < g->M) {
        *lo = b * g->n_pore;
        *hi = (b + 1) * g->n_pore;
    } else {
        *lo = g->M * g->n_pore;
        *hi = g->N;
    }
}

static void ora_bd_block_g(const ora_geom *g, int b, double *B)
{
    if (g->op == ORA_OP_SLP) {
        ora_slp_block_g(g, b, B);
        return;
    }
    int lo, hi;
    ora_body_range(g, b, &lo, &hi);
    int n = hi - lo, n2 = 2 * n;
    double len = 0.0;
    for (int j = lo; j < hi; ++j)
        len += g->w[j];
    for (int i = lo; i < hi; ++i) {
        for (int j = lo; j < hi; ++j) {
            double e00, e01, e10, e11;
            if (i != j) {
                double rx = g->x[2 * i] - g->x[2 * j];
                double ry = g->x[2 * i + 1] - g->x[2 * j + 1];
                double rho2 = rx * rx + ry * ry;
                double rn = rx * g->nrm[2 * j] + ry * g->nrm[2 * j + 1];
                double c = (g->w[j] / ORA_PI) * rn / (rho2 * rho2);
                e00 = c * rx * rx;
                e01 = c * rx * ry;
                e10 = c * ry * rx;
                e11 = c * ry * ry;
            } else {
                double tx = g->tan[2 * i], ty = g->tan[2 * i + 1];
                double a = (g->w[i] / (2.0 * ORA_PI)) * g->kn[i];
                e00 = a * tx * tx - 0.5;
                e01 = a * tx * ty;
                e10 = a * ty * tx;
                e11 = a * ty * ty - 0.5;
            }
            if (b < g->M) {
                double rx = g->x[2 * i] - g->pc[2 * b];
                double ry = g->x[2 * i + 1] - g->pc[2 * b + 1];
                double rho2 = rx * rx + ry * ry;
                double lg = 0.5 * log(rho2);
                double f = g->w[j] / len;
                double s00 = (1.0 / (4.0 * ORA_PI)) * (-lg + rx * rx / rho2);
                double s01 = (1.0 / (4.0 * ORA_PI)) * (rx * ry / rho2);
                double s11 = (1.0 / (4.0 * ORA_PI)) * (-lg + ry * ry / rho2);
                double Rx = ry / rho2, Ry = -rx / rho2;           /* R(x_i - c) */
                double qx = g->x[2 * j + 1] - g->pc[2 * b + 1];   /* (x_j - c)^perp */
                double qy = -(g->x[2 * j] - g->pc[2 * b]);
                e00 += f * (s00 + Rx * qx);
                e01 += f * (s01 + Rx * qy);
                e10 += f * (s01 + Ry * qx);
                e11 += f * (s11 + Ry * qy);
            } else {
                double f = g->w[j] / len;
                e00 += f * g->nrm[2 * i] * g->nrm[2 * j];
                e01 += f * g->nrm[2 * i] * g->nrm[2 * j + 1];
                e10 += f * g->nrm[2 * i + 1] * g->nrm[2 * j];
                e11 += f * g->nrm[2 * i + 1] * g->nrm[2 * j + 1];
            }
            int li = i - lo, lj = j - lo;
            B[(size_t)(2 * li) * n2 + 2 * lj] = e00;
            B[(size_t)(2 * li) * n2 + 2 * lj + 1] = e01;
            B[(size_t)(2 * li + 1) * n2 + 2 * lj] = e10;
            B[(size_t)(2 * li + 1) * n2 + 2 * lj + 1] = e11;
        }
    }
}

void ora_bd_block(int N, int M, int n_pore, const double *x, const double *nrm, const double *w,
                  const double *tan, const double *kn, const double *pc, const double *pr, int b, double *B)
{
    ora_geom g = {N, M, n_pore, x, nrm, w, tan, kn, pc, pr, 0, NULL};
    ora_bd_block_g(&g, b, B);
}

/* Doolittle LU with partial pivoting, in place, row-major n x n.
 * Pivot = row of max |a_ik| over i >= k, lowest index on ties.
 * piv[k] = row swapped with k.  Returns 0, or k+1 if a zero pivot is met. */
int ora_lu(int n, double *A, int *piv)
{
    for (int k = 0; k < n; ++k) {
        int p = k;
        double best = fabs(A[(size_t)k * n + k]);
        for (int i = k + 1; i < n; ++i) {
            double v = fabs(A[(size_t)i * n + k]);
            if (v > best) {
                best = v;
                p = i;
            }
        }
        piv[k] = p;
        if (best == 0.0)
            return k + 1;
        if (p != k) {
            for (int c = 0; c < n; ++c) {
                double t = A[(size_t)k * n + c];
                A[(size_t)k * n + c] = A[(size_t)p * n + c];
                A[(size_t)p * n + c] = t;
            }
        }
        double d = A[(size_t)k * n + k];
#pragma omp parallel for schedule(static) if (n - k > 1536)
        for (int i = k + 1; i < n; ++i) {
            double l = A[(size_t)i * n + k] / d;
            A[(size_t)i * n + k] = l;
            for (int c = k + 1; c < n; ++c)
                A[(size_t)i * n + c] -= l * A[(size_t)k * n + c];
        }
    }
    return 0;
}

/* Explicit inverse from the LU factors by n solves A x = e_c. */
void ora_lu_inverse(int n, const double *LU, const int *piv, double *Ainv)
{
#pragma omp parallel for schedule(dynamic, 4) if (n > 128)
    for (int c = 0; c < n; ++c) {
        double *z = (double *)malloc((size_t)n * sizeof(double));
        for (int i = 0; i < n; ++i)
            z[i] = (i == c) ? 1.0 : 0.0;
        for (int k = 0; k < n; ++k) { /* apply P */
            int p = piv[k];
            if (p != k) {
                double t = z[k];
                z[k] = z[p];
                z[p] = t;
            }
        }
        for (int i = 0; i < n; ++i) { /* L z = Pb, unit lower */
            double s = z[i];
            for (int q = 0; q < i; ++q)
                s -= LU[(size_t)i * n + q] * z[q];
            z[i] = s;
        }
        for (int i = n - 1; i >= 0; --i) { /* U x = z */
            double s = z[i];
            for (int q = i + 1; q < n; ++q)
                s -= LU[(size_t)i * n + q] * z[q];
            z[i] = s / LU[(size_t)i * n + i];
        }
        for (int i = 0; i < n; ++i)
            Ainv[(size_t)i * n + c] = z[i];
        free(z);
    }
}

/* ---------------------------------------------------------------------------
 * BD preconditioner object: explicit inverse per body.
 * ------------------------------------------------------------------------- */
typedef struct {
    int N, M, n_pore, nb;
    size_t *off; /* offset of block b in inv */
    int *lo, *n; /* node range per body */
    double *inv;
} ora_bd;

/* Returns NULL on allocation failure; *bad = body index + 1 if singular. */
static void *ora_bd_factor_g(const ora_geom *gp, int *bad)
{
    const ora_geom g = *gp;
    int N = g.N, M = g.M, n_pore = g.n_pore;
    ora_bd *bd = (ora_bd *)calloc(1, sizeof(ora_bd));
    int nb = M + (N > M * n_pore ? 1 : 0);
    bd->N = N;
    bd->M = M;
    bd->n_pore = n_pore;
    bd->nb = nb;
    bd->off = (size_t *)calloc((size_t)nb + 1, sizeof(size_t));
    bd->lo = (int *)calloc((size_t)nb, sizeof(int));
    bd->n = (int *)calloc((size_t)nb, sizeof(int));
    for (int b = 0; b < nb; ++b) {
        int lo, hi;
        ora_body_range(&g, b, &lo, &hi);
        bd->lo[b] = lo;
        bd->n[b] = hi - lo;
        bd->off[b + 1] = bd->off[b] + (size_t)(2 * (hi - lo)) * (size_t)(2 * (hi - lo));
    }
    bd->inv = (double *)malloc(bd->off[nb] * sizeof(double));
    *bad = 0;
    if (!bd->inv)
        return NULL;
    int nsmall = M; /* pores: parallel over blocks; wall: parallel inside */
#pragma omp parallel for schedule(dynamic, 1)
    for (int b = 0; b < nsmall; ++b) {
        int n2 = 2 * bd->n[b];
        double *B = (double *)malloc((size_t)n2 * n2 * sizeof(double));
        int *piv = (int *)malloc((size_t)n2 * sizeof(int));
        ora_bd_block_g(&g, b, B);
        int rc = ora_lu(n2, B, piv);
        if (rc) {
#pragma omp critical
            *bad = b + 1;
        } else {
            ora_lu_inverse(n2, B, piv, bd->inv + bd->off[b]);
        }
        free(B);
        free(piv);
    }
    for (int b = nsmall; b < nb; ++b) {
        int n2 = 2 * bd->n[b];
        double *B = (double *)malloc((size_t)n2 * n2 * sizeof(double));
        int *piv = (int *)malloc((size_t)n2 * sizeof(int));
        ora_bd_block_g(&g, b, B);
        int rc = ora_lu(n2, B, piv);
        if (rc)
            *bad = b + 1;
        else
            ora_lu_inverse(n2, B, piv, bd->inv + bd->off[b]);
        free(B);
        free(piv);
    }
    return bd;
}

void *ora_bd_factor(int N, int M, int n_pore, const double *x, const double *nrm, const double *w,
                    const double *tan, const double *kn, const double *pc, const double *pr, int *bad)
{
    ora_geom g = {N, M, n_pore, x, nrm, w, tan, kn, pc, pr, 0, NULL};
    return ora_bd_factor_g(&g, bad);
}

/* BD of the SLP operator (NEXT-1): the same exact per-body inverses of the
 * SLP blocks (P:l.651-657 footnote). */
void *ora_slp_bd_factor(int N, int M, int n_pore, const double *x, const double *w, const double *gam, int *bad)
{
    ora_geom g = {N, M, n_pore, x, NULL, w, NULL, NULL, NULL, NULL, ORA_OP_SLP, gam};
    return ora_bd_factor_g(&g, bad);
}

/* Solve with stored LU factors (Doolittle, partial pivoting): z = A^{-1} v. */
static void ora_lu_solve(int n, const double *LU, const int *piv, const double *v, double *z)
{
    for (int i = 0; i < n; ++i)
        z[i] = v[i];
    for (int k = 0; k < n; ++k) {
        int p = piv[k];
        if (p != k) {
            double t = z[k];
            z[k] = z[p];
            z[p] = t;
        }
    }
    for (int i = 0; i < n; ++i) {
        double s = z[i];
        for (int q = 0; q < i; ++q)
            s -= LU[(size_t)i * n + q] * z[q];
        z[i] = s;
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = z[i];
        for (int q = i + 1; q < n; ++q)
            s -= LU[(size_t)i * n + q] * z[q];
        z[i] = s / LU[(size_t)i * n + i];
    }
}

/* BD in "LU" form: the same preconditioner P^{-1} = B_b^{-1} per body, applied
 * by forward/back substitution with the stored factors instead of an explicit
 * inverse (used where forming the inverse in plain loops is too slow: the
 * 16384^2 wall block of config 4).  Same operator, different rounding only. */
typedef struct {
    int N, M, n_pore, nb;
    size_t *off;
    int *lo, *n;
    double *lu;
    int *piv; /* piv of block b at 2*lo[b] */
} ora_bdlu;

static void *ora_bdlu_factor_g(const ora_geom *gp, int *bad)
{
    const ora_geom g = *gp;
    int N = g.N, M = g.M, n_pore = g.n_pore;
    ora_bdlu *bd = (ora_bdlu *)calloc(1, sizeof(ora_bdlu));
    int nb = M + (N > M * n_pore ? 1 : 0);
    bd->N = N;
    bd->M = M;
    bd->n_pore = n_pore;
    bd->nb = nb;
    bd->off = (size_t *)calloc((size_t)nb + 1, sizeof(size_t));
    bd->lo = (int *)calloc((size_t)nb, sizeof(int));
    bd->n = (int *)calloc((size_t)nb, sizeof(int));
    for (int b = 0; b < nb; ++b) {
        int lo, hi;
        ora_body_range(&g, b, &lo, &hi);
        bd->lo[b] = lo;
        bd->n[b] = hi - lo;
        bd->off[b + 1] = bd->off[b] + (size_t)(2 * (hi - lo)) * (size_t)(2 * (hi - lo));
    }
    bd->lu = (double *)malloc(bd->off[nb] * sizeof(double));
    bd->piv = (int *)malloc((size_t)2 * N * sizeof(int));
    *bad = 0;
    if (!bd->lu || !bd->piv)
        return NULL;
#pragma omp parallel for schedule(dynamic, 1)
    for (int b = 0; b < M; ++b) {
        ora_bd_block_g(&g, b, bd->lu + bd->off[b]);
        if (ora_lu(2 * bd->n[b], bd->lu + bd->off[b], bd->piv + 2 * bd->lo[b])) {
#pragma omp critical
            *bad = b + 1;
        }
    }
    for (int b = M; b < nb; ++b) {
        ora_bd_block_g(&g, b, bd->lu + bd->off[b]);
        if (ora_lu(2 * bd->n[b], bd->lu + bd->off[b], bd->piv + 2 * bd->lo[b]))
            *bad = b + 1;
    }
    return bd;
}

void *ora_bdlu_factor(int N, int M, int n_pore, const double *x, const double *nrm, const double *w,
                      const double *tan, const double *kn, const double *pc, const double *pr, int *bad)
{
    ora_geom g = {N, M, n_pore, x, nrm, w, tan, kn, pc, pr, 0, NULL};
    return ora_bdlu_factor_g(&g, bad);
}

void *ora_slp_bdlu_factor(int N, int M, int n_pore, const double *x, const double *w, const double *gam, int *bad)
{
    ora_geom g = {N, M, n_pore, x, NULL, w, NULL, NULL, NULL, NULL, ORA_OP_SLP, gam};
    return ora_bdlu_factor_g(&g, bad);
}

void ora_bdlu_apply(void *h, const double *in, double *out)
{
    ora_bdlu *bd = (ora_bdlu *)h;
#pragma omp parallel for schedule(dynamic, 1)
    for (int b = 0; b < bd->nb; ++b)
        ora_lu_solve(2 * bd->n[b], bd->lu + bd->off[b], bd->piv + 2 * bd->lo[b], in + 2 * (size_t)bd->lo[b],
                     out + 2 * (size_t)bd->lo[b]);
}

void ora_bdlu_free(void *h)
{
    ora_bdlu *bd = (ora_bdlu *)h;
    if (!bd)
        return;
    free(bd->lu);
    free(bd->piv);
    free(bd->off);
    free(bd->lo);
    free(bd->n);
    free(bd);
}

/* z_b = B_b^{-1} v_b for each body (A7). */
void ora_bd_apply(void *h, const double *in, double *out)
{
    ora_bd *bd = (ora_bd *)h;
    for (int b = 0; b < bd->nb; ++b) {
        int n2 = 2 * bd->n[b];
        const double *Bi = bd->inv + bd->off[b];
        const double *v = in + 2 * (size_t)bd->lo[b];
        double *z = out + 2 * (size_t)bd->lo[b];
#pragma omp parallel for schedule(static) if (n2 > 512)
        for (int i = 0; i < n2; ++i) {
            double s = 0.0;
            for (int c = 0; c < n2; ++c)
                s += Bi[(size_t)i * n2 + c] * v[c];
            z[i] = s;
        }
    }
}

/* Copy out the explicit inverse of block b (for parity tests). */
int ora_bd_block_inverse(void *h, int b, double *dst)
{
    ora_bd *bd = (ora_bd *)h;
    if (b < 0 || b >= bd->nb)
        return -1;
    memcpy(dst, bd->inv + bd->off[b], (bd->off[b + 1] - bd->off[b]) * sizeof(double));
    return 0;
}

void ora_bd_free(void *h)
{
    ora_bd *bd = (ora_bd *)h;
    if (!bd)
        return;
    free(bd->inv);
    free(bd->off);
    free(bd->lo);
    free(bd->n);
    free(bd);
}

/* ---------------------------------------------------------------------------
 * A8/A9: left-preconditioned full GMRES (P:l.596-601 tol, P:l.661-663 left
 * PC, P:l.678-686 residual pair), x0 = 0, CGS2, Givens rotations (reading
 * C13 of DESIGN.md):
 *   r0 = P^{-1} f, beta = ||r0||, v0 = r0/beta, g = beta e_0, hist[0] = 1
 *   for k = 0..: w = P^{-1}(A v_k); w0 = ||w||
 *     h = V^T w; w -= V h; h' = V^T w; w -= V h'; H[:,k] = h + h'
 *     H[k+1,k] = ||w||; apply old rotations to column k;
 *     d = hypot(H[k,k], H[k+1,k]); c = H[k,k]/d; s = H[k+1,k]/d; H[k,k] = d
 *     g[k+1] = -s g[k]; g[k] = c g[k]; hist[k+1] = |g[k+1]|/beta
 *     stop if hist[k+1] < tol, or H[k+1,k] <= 1e-14 w0 (happy breakdown,
 *     counted as converged), or k+1 == max_iter
 *     v_{k+1} = w / H[k+1,k]
 *   y = H^{-1} g (upper triangular), x = V y.
 * Operators are callbacks so the same routine serves the completed DLP
 * operator and the dense special cases of the pins (V8).
 * ------------------------------------------------------------------------- */
typedef void (*ora_op)(void *ctx, const double *in, double *out);

/* Sensitivity runs (reading C23; tools/make_golden.py).  Test
 * infrastructure for the GMRES parity envelope, not part of the method: every
 * primitive of the iteration gets seeded Gaussian noise at the measured
 * GPU-vs-oracle disagreement of that primitive (profiles/round2/
 * disagreement.json), so the envelope is the oracle's own sensitivity to
 * exactly the rounding differences the GPU path introduces:
 *   eps[0] A v        out_i += eps max|out| z_i
 *   eps[1] P^-1 v     out_i += eps max|out| z_i
 *   eps[2] V_j . w    h_j   += eps ||w|| z       (||V_j|| = 1)
 *   eps[3] ||w||      nrm   *= 1 + eps z
 *   eps[4] w -= V h   w_i   += eps max|w| z_i    (each CGS pass)
 * z ~ N(0, 1) from a counter-based generator (splitmix64 of (seed, event, i),
 * Box-Muller).  All eps = 0 (the default) leaves every result bit-identical
 * to the unperturbed oracle. */
static double ora_pert_eps[5] = {0, 0, 0, 0, 0};
static unsigned long long ora_pert_seed = 0, ora_pert_calls = 0;

void ora_gmres_set_perturbation(const double *eps5, unsigned long long seed)
{
    for (int q = 0; q < 5; ++q)
        ora_pert_eps[q] = eps5 ? eps5[q] : 0.0;
    ora_pert_seed = seed;
    ora_pert_calls = 0;
}

static unsigned long long ora_splitmix(unsigned long long x)
{
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

static double ora_gauss(unsigned long long call, unsigned long long i)
{
    unsigned long long h = ora_splitmix(ora_splitmix(ora_pert_seed ^ (call << 32)) + i);
    double u1 = ((h >> 11) + 1.0) * (1.0 / 9007199254740993.0); /* (0, 1] */
    double u2 = (ora_splitmix(h) >> 11) * (1.0 / 9007199254740992.0);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * ORA_PI * u2);
}

/* vector primitive: v_i += eps max|v| z_i */
static void ora_perturb(int n, double *v, double eps)
{
    if (eps == 0.0)
        return;
    const unsigned long long call = ora_pert_calls++;
    double m = 0.0;
    for (int i = 0; i < n; ++i)
        m = fabs(v[i]) > m ? fabs(v[i]) : m;
    for (int i = 0; i < n; ++i)
        v[i] += eps * m * ora_gauss(call, (unsigned long long)i);
}

/* scalar primitive: x + eps scale z */
static double ora_perturb_s(double x, double eps, double scale)
{
    if (eps == 0.0)
        return x;
    return x + eps * scale * ora_gauss(ora_pert_calls++, 0);
}

static double ora_dot(int n, const double *a, const double *b)
{
    double s = 0.0;
    for (int i = 0; i < n; ++i)
        s += a[i] * b[i];
    return s;
}

static int ora_gmres_core(int n, ora_op A, void *actx, ora_op P, void *pctx, const double *f, double *x,
                          double tol, int max_iter, double *hist, double *res_pc, double *res_true,
                          int *converged)
{
    double *r = (double *)malloc((size_t)n * sizeof(double));
    double *t = (double *)malloc((size_t)n * sizeof(double));
    double *wv = (double *)malloc((size_t)n * sizeof(double));
    double **V = (double **)calloc((size_t)max_iter + 1, sizeof(double *));
    double *H = (double *)calloc((size_t)(max_iter + 1) * (size_t)max_iter, sizeof(double)); /* H[row*max_iter+col] */
    double *cs = (double *)calloc((size_t)max_iter, sizeof(double));
    double *sn = (double *)calloc((size_t)max_iter, sizeof(double));
    double *gv = (double *)calloc((size_t)max_iter + 1, sizeof(double));
    double *h = (double *)calloc((size_t)max_iter + 1, sizeof(double));
    double *h2 = (double *)calloc((size_t)max_iter + 1, sizeof(double));
    int iters = 0;
    *converged = 0;

    if (P) {
        P(pctx, f, r);
        ora_perturb(n, r, ora_pert_eps[1]);
    } else {
        memcpy(r, f, (size_t)n * sizeof(double));
    }
    double beta = sqrt(ora_dot(n, r, r));
    beta = ora_perturb_s(beta, ora_pert_eps[3], beta);
    for (int i = 0; i < n; ++i)
        x[i] = 0.0;
    hist[0] = 1.0;
    if (beta == 0.0) {
        *converged = 1;
        *res_pc = 0.0;
        *res_true = 0.0;
        goto done;
    }
    V[0] = (double *)malloc((size_t)n * sizeof(double));
    for (int i = 0; i < n; ++i)
        V[0][i] = r[i] / beta;
    gv[0] = beta;
    for (int k = 0; k < max_iter; ++k) {
        A(actx, V[k], t);
        ora_perturb(n, t, ora_pert_eps[0]);
        if (P) {
            P(pctx, t, wv);
            ora_perturb(n, wv, ora_pert_eps[1]);
        } else {
            memcpy(wv, t, (size_t)n * sizeof(double));
        }
        double w0 = sqrt(ora_dot(n, wv, wv));
        w0 = ora_perturb_s(w0, ora_pert_eps[3], w0);
        for (int pass = 0; pass < 2; ++pass) {
            double *hh = pass ? h2 : h;
#pragma omp parallel for schedule(static) if (n > 4096)
            for (int j = 0; j <= k; ++j)
                hh[j] = ora_dot(n, V[j], wv);
            if (ora_pert_eps[2] != 0.0) {
                double nw = sqrt(ora_dot(n, wv, wv));
                for (int j = 0; j <= k; ++j)
                    hh[j] = ora_perturb_s(hh[j], ora_pert_eps[2], nw);
            }
#pragma omp parallel for schedule(static) if (n > 4096)
            for (int i = 0; i < n; ++i) {
                double s = wv[i];
                for (int j = 0; j <= k; ++j)
                    s -= V[j][i] * hh[j];
                wv[i] = s;
            }
            ora_perturb(n, wv, ora_pert_eps[4]);
        }
        for (int j = 0; j <= k; ++j)
            H[(size_t)j * max_iter + k] = h[j] + h2[j];
        double hk1 = sqrt(ora_dot(n, wv, wv));
        hk1 = ora_perturb_s(hk1, ora_pert_eps[3], hk1);
        H[(size_t)(k + 1) * max_iter + k] = hk1;
        for (int j = 0; j < k; ++j) {
            double a = H[(size_t)j * max_iter + k], b = H[(size_t)(j + 1) * max_iter + k];
            H[(size_t)j * max_iter + k] = cs[j] * a + sn[j] * b;
            H[(size_t)(j + 1) * max_iter + k] = -sn[j] * a + cs[j] * b;
        }
        {
            double a = H[(size_t)k * max_iter + k], b = H[(size_t)(k + 1) * max_iter + k];
            /* sqrt(a^2 + b^2) correctly rounded (reading C28: library hypot()s
             * differ by an ulp; quad-precision evaluation, one rounding) */
            double d = (double)sqrtq((__float128)a * a + (__float128)b * b);
            cs[k] = a / d;
            sn[k] = b / d;
            H[(size_t)k * max_iter + k] = d;
            H[(size_t)(k + 1) * max_iter + k] = 0.0;
            gv[k + 1] = -sn[k] * gv[k];
            gv[k] = cs[k] * gv[k];
        }
        double est = fabs(gv[k + 1]) / beta;
        hist[k + 1] = est;
        iters = k + 1;
        if (est < tol || hk1 <= 1e-14 * w0) {
            *converged = 1;
            break;
        }
        if (k + 1 == max_iter)
            break;
        V[k + 1] = (double *)malloc((size_t)n * sizeof(double));
        for (int i = 0; i < n; ++i)
            V[k + 1][i] = wv[i] / hk1;
    }
    {
        double *y = (double *)calloc((size_t)iters + 1, sizeof(double));
        for (int i = iters - 1; i >= 0; --i) {
            double s = gv[i];
            for (int j = i + 1; j < iters; ++j)
                s -= H[(size_t)i * max_iter + j] * y[j];
            y[i] = s / H[(size_t)i * max_iter + i];
        }
        for (int i = 0; i < n; ++i) {
            double s = 0.0;
            for (int j = 0; j < iters; ++j)
                s += V[j][i] * y[j];
            x[i] = s;
        }
        free(y);
    }
    /* residual pair (P:l.678-686) */
    A(actx, x, t);
    for (int i = 0; i < n; ++i)
        t[i] = f[i] - t[i];
    *res_true = sqrt(ora_dot(n, t, t)) / sqrt(ora_dot(n, f, f));
    if (P) {
        P(pctx, t, wv);
        *res_pc = sqrt(ora_dot(n, wv, wv)) / beta;
    } else {
        *res_pc = *res_true;
    }
done:
    for (int j = 0; j <= max_iter; ++j)
        free(V[j]);
    free(V);
    free(H);
    free(cs);
    free(sn);
    free(gv);
    free(h);
    free(h2);
    free(r);
    free(t);
    free(wv);
    return iters;
}

/* The iteration's own primitives, exported so the GPU-vs-oracle disagreement
 * of each can be measured (tools/measure_disagreement.py): out[j] = V_j . w
 * (sequential ascending sums, as in CGS) and w_i -= sum_j V_j,i h_j. */
void ora_cgs_dots(int n, int nv, const double *V, const double *w, double *out)
{
#pragma omp parallel for schedule(static) if (n > 4096)
    for (int j = 0; j < nv; ++j)
        out[j] = ora_dot(n, V + (size_t)j * n, w);
}

void ora_cgs_sub(int n, int nv, const double *V, const double *h, double *w)
{
#pragma omp parallel for schedule(static) if (n > 4096)
    for (int i = 0; i < n; ++i) {
        double s = w[i];
        for (int j = 0; j < nv; ++j)
            s -= V[(size_t)j * n + i] * h[j];
        w[i] = s;
    }
}

/* --- dense special cases (V8) --- */
typedef struct {
    int n;
    const double *A;
} ora_dense;

static void ora_dense_apply(void *ctx, const double *in, double *out)
{
    ora_dense *d = (ora_dense *)ctx;
    for (int i = 0; i < d->n; ++i) {
        double s = 0.0;
        for (int c = 0; c < d->n; ++c)
            s += d->A[(size_t)i * d->n + c] * in[c];
        out[i] = s;
    }
}

int ora_gmres_dense(int n, const double *A, const double *Pinv, const double *f, double *x, double tol,
                    int max_iter, double *hist, double *res_pc, double *res_true, int *converged)
{
    ora_dense a = {n, A}, p = {n, Pinv};
    return ora_gmres_core(n, ora_dense_apply, &a, Pinv ? ora_dense_apply : NULL, &p, f, x, tol, max_iter,
                          hist, res_pc, res_true, converged);
}

/* --- the completed DLP operator, BD preconditioned or not --- */
typedef struct {
    ora_geom g;
} ora_opctx;

static void ora_op_apply(void *ctx, const double *in, double *out)
{
    ora_opctx *c = (ora_opctx *)ctx;
    ora_apply_g(&c->g, in, out, 0u, NULL, 0); /* op 0: completed DLP, op 1: SLP */
}

static void ora_op_bd(void *ctx, const double *in, double *out)
{
    ora_bd_apply(ctx, in, out);
}

static void ora_op_bdlu(void *ctx, const double *in, double *out)
{
    ora_bdlu_apply(ctx, in, out);
}

/* Same GMRES with the BD preconditioner applied through LU solves (ora_bdlu). */
int ora_gmres_bdlu(int N, int M, int n_pore, const double *x, const double *nrm, const double *w, const double *tan,
                   const double *kn, const double *pc, const double *pr, void *bdlu, const double *f, double *sol,
                   double tol, int max_iter, double *hist, double *res_pc, double *res_true, int *converged)
{
    ora_opctx c = {{N, M, n_pore, x, nrm, w, tan, kn, pc, pr, 0, NULL}};
    return ora_gmres_core(2 * N, ora_op_apply, &c, ora_op_bdlu, bdlu, f, sol, tol, max_iter, hist, res_pc,
                          res_true, converged);
}

int ora_gmres(int N, int M, int n_pore, const double *x, const double *nrm, const double *w, const double *tan,
              const double *kn, const double *pc, const double *pr, void *bd, const double *f, double *sol,
              double tol, int max_iter, double *hist, double *res_pc, double *res_true, int *converged)
{
    ora_opctx c = {{N, M, n_pore, x, nrm, w, tan, kn, pc, pr, 0, NULL}};
    return ora_gmres_core(2 * N, ora_op_apply, &c, bd ? ora_op_bd : NULL, bd, f, sol, tol, max_iter, hist,
                          res_pc, res_true, converged);
}

/* GMRES on the SLP operator (NEXT-1); pc_kind 0: none, 1: explicit-inverse BD
 * (ora_slp_bd_factor), 2: LU-form BD (ora_slp_bdlu_factor). */
int ora_slp_gmres(int N, int M, int n_pore, const double *x, const double *w, const double *gam, void *pc,
                  int pc_kind, const double *f, double *sol, double tol, int max_iter, double *hist, double *res_pc,
                  double *res_true, int *converged)
{
    ora_opctx c = {{N, M, n_pore, x, NULL, w, NULL, NULL, NULL, NULL, ORA_OP_SLP, gam}};
    ora_op P = pc_kind == 1 ? ora_op_bd : pc_kind == 2 ? ora_op_bdlu : NULL;
    return ora_gmres_core(2 * N, ora_op_apply, &c, P, pc, f, sol, tol, max_iter, hist, res_pc, res_true,
                          converged);
}
