"""Pins of the CPU oracle against values the paper and the mathematics fix
(SURVEY.md s8(c) V1-V10).  None of these compares the oracle with itself.

Tolerances are those DESIGN.md s3 derives (trapezoid near-field error for the
Gauss identities, rounding for the algebraic identities)."""
import numpy as np
import pytest
from scipy.special import iv

import oracle
from bie_inputs import (
    density,
    make_problem,
    rhs_pipe,
    rhs_rotation_outer,
    rhs_shear_all,
    stokeslet_rotlet_field,
    stokeslet_rotlet_params,
)
from bie_inputs.geometry import Problem, make_circle_problem, make_pipe


@pytest.fixture(scope="module")
def g1():
    return oracle.OracleGeometry(make_problem(1))


@pytest.fixture(scope="module")
def g2():
    return oracle.OracleGeometry(make_problem(2))


@pytest.fixture(scope="module")
def bd2(g2):
    return oracle.OracleBD(g2)


# ---------------------------------------------------------------- V1 Gauss
@pytest.mark.parametrize("cid,tol", [(1, 1e-14), (2, 1e-12)])
def test_V1_gauss_identity_whole_geometry(cid, tol):
    """Constant density e: PV D[e] = -1/2 e at every node of the multiply
    connected geometry (n out of the fluid: wall -1/2 e, own pore +1/2 e,
    plus -e from Gamma_0 on pore nodes) -- jump relations, C2/C3/C4."""
    g = oracle.OracleGeometry(make_problem(cid))
    for e in ([1.0, 0.0], [0.0, 1.0], [0.3, -0.7]):
        s = np.tile(e, g.N)
        d = g.apply(s, flags=oracle.D_ONLY)
        assert np.abs(d + 0.5 * s).max() < tol


def test_V1_gauss_config4_worst_rows():
    """Config 4 (C16 geometry): the Gauss identity holds to the trapezoid
    near-field error (C18): ~2e-10 at the pore nodes nearest the wall, ~9e-9
    at the closest pore pair (gap 0.02).  Rows chosen by distance to the
    nearest node of another body."""
    from scipy.spatial import cKDTree

    p = make_problem(4)
    g = oracle.OracleGeometry(p)
    x = g.x.reshape(-1, 2)
    body = np.concatenate([np.repeat(np.arange(p.M), p.n_pore), np.full(p.N - p.M * p.n_pore, p.M)])
    dd, ii = cKDTree(x).query(x, k=40)
    mind = np.full(p.N, np.inf)
    for c in range(40):
        other = body[ii[:, c]] != body
        mind = np.where(other & (dd[:, c] < mind), dd[:, c], mind)
    rows = np.argsort(mind)[:96].astype(np.int32)
    e = np.array([0.3, -0.7])
    y = g.apply(np.tile(e, p.N), flags=oracle.D_ONLY, rows=rows).reshape(-1, 2)
    err = np.abs(y + 0.5 * e).max()
    assert 1e-10 < err < 2e-8
    far = np.argsort(mind)[-64:].astype(np.int32)
    y = g.apply(np.tile(e, p.N), flags=oracle.D_ONLY, rows=far).reshape(-1, 2)
    assert np.abs(y + 0.5 * e).max() < 1e-11


def test_V1_gauss_off_surface_single_circle():
    """Circle with n away from its centre: D[e] = -e inside, 0 outside."""
    p = make_circle_problem(64, 0.7, (), 64)
    g = oracle.OracleGeometry(p)
    e = np.tile([0.4, -1.1], g.N)
    inside = np.array([[0.0, 0.0], [0.2, -0.1], [-0.3, 0.25]])
    outside = np.array([[2.0, 0.0], [0.0, -3.0], [1.5, 1.5]])
    assert np.abs(g.field(e, inside) + np.array([0.4, -1.1])).max() < 1e-14
    assert np.abs(g.field(e, outside)).max() < 1e-14


# ---------------------------------------------------------------- V2 Bessel
def test_V2_spectral_convergence_bessel():
    """sigma = (e^{cos th}, 0) on a circle (n outward): PV D[sigma](th) =
    -1/2 (I0(1) - I1(1) cos th, -I1(1) sin th); trapezoid converges spectrally."""
    errs = {}
    for n in (4, 8, 12, 16, 32):
        p = make_circle_problem(n, 0.7, (), 64)
        g = oracle.OracleGeometry(p)
        th = 2 * np.pi * np.arange(n) / n
        s = np.stack([np.exp(np.cos(th)), 0 * th], 1).reshape(-1)
        d = g.apply(s, flags=oracle.D_ONLY).reshape(-1, 2)
        ex = -0.5 * np.stack([iv(0, 1) - iv(1, 1) * np.cos(th), -iv(1, 1) * np.sin(th)], 1)
        errs[n] = np.abs(d - ex).max()
    assert 1e-3 < errs[4] < 5e-2
    assert errs[8] < 5e-6 and errs[8] > 1e-8
    assert errs[12] < 5e-11
    assert errs[16] < 2e-15 and errs[32] < 2e-15


# ---------------------------------------------------------------- V3 null space
def test_V3_nullspace_bare_and_completed(g1):
    """Bare -1/2 I + D has nullity 3M+1 (rank-3 per pore: 2 translations +
    rotation, P:l.260-264; 1 on Gamma_0); the completed operator is nonsingular."""
    n2 = 2 * g1.N
    I = np.eye(n2)
    D = g1.apply(I, flags=oracle.D_ONLY).T
    sb = np.linalg.svd(-0.5 * I + D, compute_uv=False)
    sf = np.linalg.svd(g1.apply(I).T, compute_uv=False)
    assert np.all(sb[-4:] < 1e-14) and sb[-5] > 1e-2
    assert sf[-1] > 1e-2 and sf[0] / sf[-1] < 200


def test_V3_rotation_in_bare_nullspace(g2):
    p = g2.problem
    k = 2
    lo, hi = g2.body_range(k)
    q = g2.x.reshape(-1, 2)[lo:hi] - p.pore_c[k]
    s = np.zeros(2 * g2.N)
    s[2 * lo:2 * hi:2], s[2 * lo + 1:2 * hi:2] = q[:, 1], -q[:, 0]
    bare = -0.5 * s + g2.apply(s, flags=oracle.D_ONLY)
    assert np.abs(bare).max() < 1e-13


# ---------------------------------------------------------------- V11 N0 term (nu)
def _wall_normal_density(p, R):
    """sigma = n on Gamma_0 (outward of Omega_0, reading C2: n = x / R on a
    circle centred at 0), zero on the pores -- built from the raw input curve."""
    s = np.zeros(2 * p.N)
    lo = p.M * p.n_pore
    s[2 * lo:] = (p.outer_xy / R).reshape(-1)
    return s, lo


@pytest.mark.parametrize("R,n_outer,pores", [(1.0, 64, ((0.0, 0.0, 0.3),)),
                                             (2.5, 96, ((0.4, -0.3, 0.5), (-1.1, 0.6, 0.35)))])
def test_V11_nu_closed_form_circle(R, n_outer, pores):
    """Closed form that fixes the null-space term N0 (reading C5, P:l.260-264).
    On a circle of radius R, r.n_y = -rho^2 / (2R) for x, y on the curve, so the
    DLP kernel applied to sigma = n is (1/pi) r / (4 R^2) and, the trapezoid
    rule being exact for the degree-1 trigonometric integrand,
    D[n] = n / 2 at every wall node: (-1/2 I + D)[n] = 0.  The self term
    vanishes (t.n = 0) and lambda_k = mu_k = 0 (sigma = 0 on the pores), so the
    completed operator gives A sigma = nu n on the wall rows with
    nu = (1/|Gamma_0|) sum_j w_j n_j.n_j = 1, i.e. A sigma = n there.  Inside
    Gamma_0 the same density is the zero Stokes flow (Dirichlet uniqueness):
    A sigma = 0 on the pore rows up to the trapezoid error at the pores'
    distance.  A sign or scale slip in nu fails the wall rows."""
    p = make_circle_problem(n_outer, R, pores, 64)
    g = oracle.OracleGeometry(p)
    s, lo = _wall_normal_density(p, R)
    y = g.apply(s)
    assert np.abs(y[2 * lo:] - s[2 * lo:]).max() < 1e-14
    assert np.abs(y[:2 * lo]).max() < 1e-13
    # the D-only part alone vanishes on the wall rows (no N0 there)
    d = -0.5 * s + g.apply(s, flags=oracle.D_ONLY)
    assert np.abs(d[2 * lo:]).max() < 1e-14


# ---------------------------------------------------------------- V4 completion
def test_V4_completion_closed_forms(g2):
    p = g2.problem
    pts = g2.x.reshape(-1, 2)
    for k in (0, 3, 9):
        lo, hi = g2.body_range(k)
        r = pts - p.pore_c[k]
        rho2 = (r * r).sum(1)
        for e in ([1.0, 0.0], [0.0, 1.0]):
            s = np.zeros(2 * g2.N)
            s[2 * lo:2 * hi] = np.tile(e, hi - lo)
            y = g2.apply(s).reshape(-1, 2)
            rl = r @ np.array(e)
            ex = (1 / (4 * np.pi)) * (-0.5 * np.log(rho2)[:, None] * np.array(e)[None, :] + (rl / rho2)[:, None] * r)
            assert np.abs(y - ex).max() < 1e-13
        q = pts[lo:hi] - p.pore_c[k]
        s = np.zeros(2 * g2.N)
        s[2 * lo:2 * hi:2], s[2 * lo + 1:2 * hi:2] = q[:, 1], -q[:, 0]
        y = g2.apply(s).reshape(-1, 2)
        ex = p.pore_r[k] ** 2 * np.stack([r[:, 1], -r[:, 0]], 1) / rho2[:, None]
        assert np.abs(y - ex).max() < 1e-13


# ---------------------------------------------------------------- V5 Couette
def test_V5_couette_closed_form(g1):
    """Rotating unit circle, still pore r=0.3 (C11): u_theta = A r + B/r,
    A = 1/0.91, B = -0.09/0.91 -- whole pipeline including BD-GMRES."""
    bd = oracle.OracleBD(g1)
    res = oracle.gmres(g1, rhs_rotation_outer(g1.problem), bd, tol=1e-13, max_iter=100)
    assert res["converged"]
    A, B = 1 / 0.91, -0.09 / 0.91
    th = np.linspace(0, 2 * np.pi, 7, endpoint=False)
    for rad, tol in ((0.5, 1e-12), (0.65, 1e-9)):
        pts = rad * np.stack([np.cos(th), np.sin(th)], 1)
        u = g1.field(res["x"], pts)
        ex = (A * rad + B / rad) * np.stack([-np.sin(th), np.cos(th)], 1)
        assert np.abs(u - ex).max() < tol


# ---------------------------------------------------------------- V6 paper exact solution
def test_V6_stokeslet_rotlet_exact_solution(g2, bd2):
    """P:l.943-958: f from Stokeslets/rotlets outside Omega is an exact Stokes
    solution; after the solve, u = D[sigma] + completion reproduces it inside."""
    p = g2.problem
    cs, lam, mu = stokeslet_rotlet_params(p)
    f = stokeslet_rotlet_field(g2.x.reshape(-1, 2), cs, lam, mu).reshape(-1)
    res = oracle.gmres(g2, f, bd2, tol=1e-13, max_iter=400)
    assert res["converged"]
    rng = np.random.default_rng(5)
    L, H = p.meta["L"], p.meta["H"]
    pts = []
    while len(pts) < 60:
        q = np.array([rng.uniform(0.5, L - 0.5), rng.uniform(-H + 0.3, H - 0.3)])
        if np.all(np.linalg.norm(p.pore_c - q, axis=1) - p.pore_r >= 0.3):
            pts.append(q)
    pts = np.array(pts)
    u = g2.field(res["x"], pts)
    ex = stokeslet_rotlet_field(pts, cs, lam, mu)
    assert np.abs(u - ex).max() / np.abs(ex).max() < 1e-11


# ---------------------------------------------------------------- V7 brute force / symmetries
def _dense_from_definition(g):
    """Independent dense assembly of the completed operator in numpy from the
    per-column form of the moments (linear functionals), tiny inputs only."""
    p = g.problem
    N = g.N
    x = g.x.reshape(-1, 2)
    n = g.nrm.reshape(-1, 2)
    t = g.tan.reshape(-1, 2)
    A = np.zeros((2 * N, 2 * N))
    r = x[:, None, :] - x[None, :, :]
    rho2 = (r ** 2).sum(-1)
    np.fill_diagonal(rho2, 1.0)
    rn = (r * n[None, :, :]).sum(-1)
    c = (g.w[None, :] / np.pi) * rn / rho2 ** 2
    np.fill_diagonal(c, 0.0)
    for a in range(2):
        for b in range(2):
            A[a::2, b::2] = c * r[:, :, a] * r[:, :, b]
    for i in range(N):
        A[2 * i:2 * i + 2, 2 * i:2 * i + 2] += (g.w[i] / (2 * np.pi)) * g.kn[i] * np.outer(t[i], t[i]) - 0.5 * np.eye(2)
    wall = slice(p.M * p.n_pore, N)
    L0 = g.w[wall].sum()
    for i in range(p.M * p.n_pore, N):
        for j in range(p.M * p.n_pore, N):
            A[2 * i:2 * i + 2, 2 * j:2 * j + 2] += np.outer(n[i], n[j]) * g.w[j] / L0
    for k in range(p.M):
        lo, hi = g.body_range(k)
        Lk = g.w[lo:hi].sum()
        for i in range(N):
            rr = x[i] - p.pore_c[k]
            q2 = rr @ rr
            S = (1 / (4 * np.pi)) * (-0.5 * np.log(q2) * np.eye(2) + np.outer(rr, rr) / q2)
            R = np.array([rr[1], -rr[0]]) / q2
            for j in range(lo, hi):
                qq = x[j] - p.pore_c[k]
                A[2 * i:2 * i + 2, 2 * j:2 * j + 2] += (g.w[j] / Lk) * (S + np.outer(R, [qq[1], -qq[0]]))
    return A


def test_V7_brute_force_dense(g1):
    A = _dense_from_definition(g1)
    s = density(g1.problem, nvec=3)
    y = g1.apply(s)
    ref = s @ A.T
    assert np.abs(y - ref).max() / np.abs(ref).max() < 1e-14


@pytest.mark.parametrize("cid", [1, 2])
def test_V7_long_double_summation(cid):
    """Oracle within 1e-14 (max-norm relative) of an 80-bit accumulation of
    the same DLP sum (summation-error bound)."""
    g = oracle.OracleGeometry(make_problem(cid))
    s = density(g.problem)[0]
    y = g.apply(s, flags=oracle.D_ONLY).reshape(-1, 2)
    ld = np.longdouble
    x = g.x.reshape(-1, 2).astype(ld)
    n = g.nrm.reshape(-1, 2).astype(ld)
    sg = s.reshape(-1, 2).astype(ld)
    w = g.w.astype(ld)
    rows = np.arange(0, g.N, max(1, g.N // 200))
    pi = ld(np.pi)
    for i in rows:
        r = x[i][None, :] - x
        rho2 = (r * r).sum(1)
        rho2[i] = 1
        coef = (w / pi) * (r * n).sum(1) * (r * sg).sum(1) / rho2 ** 2
        coef[i] = 0
        u = (coef[:, None] * r).sum(0)
        t = g.tan.reshape(-1, 2)[i].astype(ld)
        u += (w[i] / (2 * pi)) * ld(g.kn[i]) * (t @ sg[i]) * t
        assert np.abs(y[i] - u.astype(np.float64)).max() < 1e-14 * np.abs(y).max()


def _shifted(p: Problem, shift=None, rot90=False):
    R = np.array([[0.0, -1.0], [1.0, 0.0]])
    f = (lambda a: a @ R.T) if rot90 else (lambda a: a)
    sh = np.zeros(2) if shift is None else np.asarray(shift)
    return Problem(p.name + "_t", f(p.outer_xy) + sh, f(p.outer_dxy), f(p.outer_ddxy), p.period,
                   f(p.pore_c) + sh, p.pore_r.copy(), p.n_pore, p.config_id, dict(p.meta))


def test_V7_translation_invariance(g2):
    p = g2.problem
    gt = oracle.OracleGeometry(_shifted(p, shift=(3.7, -1.2)))
    s = density(p)[0]
    y, yt = g2.apply(s), gt.apply(s)
    assert np.abs(y - yt).max() / np.abs(y).max() < 1e-12


def test_V7_rotation_equivariance(g2):
    p = g2.problem
    gr = oracle.OracleGeometry(_shifted(p, rot90=True))
    R = np.array([[0.0, -1.0], [1.0, 0.0]])
    s = density(p)[0].reshape(-1, 2)
    # rotated pore node (j + n/4) is old node j; wall nodes keep their index
    perm = np.arange(p.N)
    q = p.n_pore // 4
    for k in range(p.M):
        base = k * p.n_pore
        perm[base:base + p.n_pore] = base + (np.arange(p.n_pore) - q) % p.n_pore
    s_new = (s @ R.T)[perm]
    y_old = g2.apply(s.reshape(-1)).reshape(-1, 2)
    y_new = gr.apply(s_new.reshape(-1)).reshape(-1, 2)
    assert np.abs(y_new - (y_old @ R.T)[perm]).max() / np.abs(y_old).max() < 1e-12


def test_V7_linearity(g2):
    s = density(g2.problem, nvec=2)
    a, b = 0.7, -1.3
    y = g2.apply(a * s[0] + b * s[1])
    y2 = a * g2.apply(s[0]) + b * g2.apply(s[1])
    assert np.abs(y - y2).max() / np.abs(y).max() < 1e-13


def test_row_subset_matches_full(g2):
    s = density(g2.problem)[0]
    rows = np.array([0, 5, 1279, 1280, 1791], dtype=np.int32)
    full = g2.apply(s).reshape(-1, 2)
    sub = g2.apply(s, rows=rows).reshape(-1, 2)
    assert np.array_equal(full[rows], sub)


# ---------------------------------------------------------------- V8 GMRES / BD special cases
def test_V8_gmres_dense_special_cases():
    f = np.array([1.0, -2.0, 0.5, 3.0])
    r = oracle.gmres_dense(np.eye(4), f)
    assert r["iters"] == 1 and r["converged"] and np.allclose(r["x"], f)
    D = np.diag([1.0, 2.0, 1.0, 2.0])
    r = oracle.gmres_dense(D, f)
    assert r["iters"] == 2 and np.allclose(r["x"], f / np.diag(D), atol=1e-14)
    rng = np.random.default_rng(0)
    A = rng.standard_normal((30, 30)) + 30 * np.eye(30)
    r = oracle.gmres_dense(A, rng.standard_normal(30), Pinv=np.linalg.inv(A))
    assert r["iters"] == 1
    b = rng.standard_normal(30)
    r = oracle.gmres_dense(A, b, tol=1e-12)
    assert np.all(np.diff(r["hist"]) <= 1e-15)  # monotone history
    # P = I: final estimate equals the true residual (to rounding)
    assert abs(r["hist"][-1] - r["res_true"]) < 1e-13
    assert np.abs(A @ r["x"] - b).max() < 1e-10


def test_V8_lu_inverse_identity():
    rng = np.random.default_rng(1)
    A = rng.standard_normal((64, 64))
    LU, piv, rc = oracle.lu(A)
    assert rc == 0
    Ai = oracle.lu_inverse(LU, piv)
    assert np.abs(Ai @ A - np.eye(64)).max() < 1e-12
    LU, piv, rc = oracle.lu(np.zeros((4, 4)))
    assert rc == 1


def test_V8_single_body_one_iteration():
    """M = 0: BD = A, so BD-GMRES converges in 1 iteration (S:l.388)."""
    p = make_pipe(0, 10.0, 256, 0, (0.1, 0.2), 0.05, 16)
    g = oracle.OracleGeometry(p)
    bd = oracle.OracleBD(g)
    res = oracle.gmres(g, rhs_pipe(p), bd, tol=1e-8, max_iter=20)
    assert res["iters"] == 1 and res["converged"]


def test_V8_bd_blocks_inverse_and_locality(g2, bd2):
    for b in (0, 7, g2.M):
        B = g2.bd_block(b)
        Bi = bd2.block_inverse(b)
        assert np.abs(Bi @ B - np.eye(B.shape[0])).max() < 1e-12
    v = np.zeros(2 * g2.N)
    lo, hi = g2.body_range(4)
    v[2 * lo:2 * hi] = density(g2.problem)[0][2 * lo:2 * hi]
    z = bd2.apply(v)
    assert np.count_nonzero(z[:2 * lo]) == 0 and np.count_nonzero(z[2 * hi:]) == 0
    # the BD block is the diagonal block of the full operator
    s = np.zeros(2 * g2.N)
    s[2 * lo] = 1.0
    col = g2.apply(s)
    assert np.abs(col[2 * lo:2 * hi] - g2.bd_block(4)[:, 0]).max() < 1e-14


def test_V8_bd_vs_nopc_iterations(g2, bd2):
    """Qualitative paper claim (P:l.669-677): BD needs fewer iterations."""
    f = rhs_pipe(g2.problem)
    r_bd = oracle.gmres(g2, f, bd2, tol=1e-8, max_iter=1000)
    r_no = oracle.gmres(g2, f, None, tol=1e-8, max_iter=1000)
    assert r_bd["converged"] and r_no["converged"]
    assert r_bd["iters"] < r_no["iters"]
    assert np.all(np.diff(r_bd["hist"]) <= 1e-15)


# ---------------------------------------------------------------- V9 shear structure
def test_V9_shear_density_zero_on_pores(g2, bd2):
    """P:l.636-638 / P:l.733-736: shear (y,0) on all curves -> sigma = 0 on pores."""
    res = oracle.gmres(g2, rhs_shear_all(g2.problem), bd2, tol=1e-13, max_iter=400)
    s = res["x"].reshape(-1, 2)
    npn = g2.M * g2.n_pore
    assert np.abs(s[:npn]).max() / np.abs(s[npn:]).max() < 1e-10


# ---------------------------------------------------------------- V10 pore-block universality
def test_V10_pore_block_universality(g2, bd2):
    """Equispaced circle blocks differ only by the Stokeslet log term:
    B_a - B_b = ((log r_b - log r_a)/(4 pi n_p)) (11^T kron I2); then
    Sherman-Morrison-Woodbury gives B_b^{-1} from B_a^{-1}."""
    p = g2.problem
    a, b = 0, 5
    Ba, Bb = g2.bd_block(a), g2.bd_block(b)
    n = p.n_pore
    E = np.kron(np.ones((n, 1)), np.eye(2))
    alpha = (np.log(p.pore_r[b]) - np.log(p.pore_r[a])) / (4 * np.pi * n)
    assert np.abs(Ba - Bb - alpha * E @ E.T).max() < 1e-13
    Ai = bd2.block_inverse(a)
    # Bb = Ba - alpha E E^T -> Bb^{-1} = Ai + alpha Ai E (I - alpha E^T Ai E)^{-1} E^T Ai
    C = np.linalg.inv(np.eye(2) - alpha * E.T @ Ai @ E)
    Bbi = Ai + alpha * Ai @ E @ C @ E.T @ Ai
    assert np.abs(Bbi - bd2.block_inverse(b)).max() < 1e-12


def test_bd_lu_form_equals_explicit_inverse(g2, bd2):
    """The LU-solve form of the BD preconditioner (used for config 4's golden
    history) is the same operator as the explicit inverses."""
    bdlu = oracle.OracleBDLU(g2)
    v = density(g2.problem, vec_id=7)[0]
    a, b = bd2.apply(v), bdlu.apply(v)
    assert np.abs(a - b).max() / np.abs(a).max() < 1e-13
    f = rhs_pipe(g2.problem)
    r1 = oracle.gmres(g2, f, bd2, tol=1e-8, max_iter=200)
    r2 = oracle.gmres_bdlu(g2, f, bdlu, tol=1e-8, max_iter=200)
    assert r1["iters"] == r2["iters"]
    assert (np.abs(r1["hist"] - r2["hist"]) / r1["hist"]).max() < 1e-10
