"""Pins of the oracle's single-layer operator with Kapur-Rokhlin corrections
(NEXT-1 of SURVEY.md s8(f); P:l.270-330) against closed forms and convergence
properties -- none of these compares the oracle with itself except S6/S7, which
tie the BD block builder and the SLP GMRES driver to the pinned apply.

Readings C24-C26:
  C24 the KR weights are the sixth-order log-correction of the punctured
      trapezoid rule, derived from Navot's generalised Euler-Maclaurin expansion;
  C25 corrections act on the whole 2x2 kernel with the same scalar weight, on
      the target's own curve only, periodic offsets +-1..+-6, W_ii = 0;
  C26 S n_k = 0 for every closed curve (continuous null space), so S_h n_k is
      O(h^6); Stokes data have zero flux through each curve (consistent system).
"""
import numpy as np
import pytest
from scipy.special import iv

import oracle
from bie_inputs import make_problem
from bie_inputs.geometry import make_circle_problem


def _kr_rule(N, f_of_t, ti_idx):
    """Corrected punctured trapezoid on [0, 2pi) for a target at node ti_idx."""
    gam = oracle.kr_weights()
    h = 2 * np.pi / N
    t = np.arange(N) * h
    w = np.full(N, h)
    w[ti_idx] = 0.0
    for k in range(1, 7):
        w[(ti_idx + k) % N] += h * gam[k - 1]
        w[(ti_idx - k) % N] += h * gam[k - 1]
    m = np.arange(N) != ti_idx
    return np.sum(w[m] * f_of_t(t[m], t[ti_idx]))


def test_S1_periodic_log_integral_is_zero():
    """SPEC example: int_0^2pi log(2 sin(t/2)) dt = 0; corrected rule at N = 256."""
    val = _kr_rule(256, lambda t, ti: np.log(np.abs(2 * np.sin((t - ti) / 2))), 0)
    assert abs(val) < 1e-12


def _bessel_exact(a, ti):
    # exp(a cos t) = I0(a) + 2 sum_m I_m(a) cos(m t);
    # int_0^2pi log|2 sin((t - ti)/2)| cos(m t) dt = -(pi/m) cos(m ti)
    m = np.arange(1, 60)
    return -2 * np.pi * np.sum(iv(m, a) * np.cos(m * ti) / m)


@pytest.mark.parametrize("a", [1.0, 1.5])
def test_S2_sixth_order_convergence_on_log_singular_integrand(a):
    """Observed order >= 5.5 over N in {64, 128, 256, 512} (SPEC invariant)."""
    Ns = [64, 128, 256, 512]
    errs = []
    for N in Ns:
        e = 0.0
        for frac in (0.0, 0.2, 0.45, 0.7):
            ti_idx = int(frac * N)
            ti = 2 * np.pi * ti_idx / N
            val = _kr_rule(N, lambda t, tt: np.log(np.abs(2 * np.sin((t - tt) / 2))) * np.exp(a * np.cos(t)), ti_idx)
            e = max(e, abs(val - _bessel_exact(a, ti)))
        errs.append(e)
    slope = -np.polyfit(np.log(Ns), np.log(errs), 1)[0]
    assert slope >= 5.5, (errs, slope)
    assert errs[-1] < 1e-9


def _circle_exact(R, N, coef):
    """SLP of a trigonometric density on the circle |x| = R (nodes at 2 pi j/N).

    log part: int log|2R sin((t - ti)/2)| e^{imt} R dt = R e^{im ti} (2 pi log R [m=0] - (pi/|m|) [m!=0]);
    r r^T/rho^2 on a circle = (1/2)[[1 - cos(t+ti), -sin(t+ti)], [-sin(t+ti), 1 + cos(t+ti)]]
    (chord direction), a trigonometric polynomial, integrated exactly by a fine
    un-punctured trapezoid."""
    th = 2 * np.pi * np.arange(N) / N
    out = np.zeros((N, 2))
    k4 = 1 / (4 * np.pi)
    for (c, m), (a, b) in coef.items():
        if m == 0:
            out[:, c] += k4 * (-R * 2 * np.pi * np.log(R)) * a
        else:
            out[:, c] += k4 * (R * np.pi / m) * (a * np.cos(m * th) + b * np.sin(m * th))
    K = 2048
    t = 2 * np.pi * np.arange(K) / K
    sig = np.zeros((K, 2))
    for (c, m), (a, b) in coef.items():
        sig[:, c] += a * np.cos(m * t) + b * np.sin(m * t)
    for i in range(N):
        ph = t + th[i]
        exx, exy, eyy = 0.5 * (1 - np.cos(ph)), -0.5 * np.sin(ph), 0.5 * (1 + np.cos(ph))
        out[i, 0] += k4 * np.sum(exx * sig[:, 0] + exy * sig[:, 1]) * R * 2 * np.pi / K
        out[i, 1] += k4 * np.sum(exy * sig[:, 0] + eyy * sig[:, 1]) * R * 2 * np.pi / K
    return out


_COEF = {(0, 0): (0.5, 0.0), (0, 3): (1.0, 0.2), (1, 2): (0.3, -0.7), (1, 1): (-0.3, 0.4), (0, 5): (0.1, 0.05)}


@pytest.mark.parametrize("R", [0.7, 1.3])
def test_S3_circle_closed_form(R):
    Ns = [64, 128, 256]
    errs = []
    for N in Ns:
        g = oracle.OracleGeometry(make_circle_problem(n_outer=N, R=R, pores=()))
        th = 2 * np.pi * np.arange(N) / N
        sig = np.zeros((N, 2))
        for (c, m), (a, b) in _COEF.items():
            sig[:, c] += a * np.cos(m * th) + b * np.sin(m * th)
        y = g.slp_apply(sig.reshape(-1)).reshape(-1, 2)
        errs.append(np.abs(y - _circle_exact(R, N, _COEF)).max())
    slope = -np.polyfit(np.log(Ns), np.log(errs), 1)[0]
    assert slope >= 5.5, (errs, slope)
    assert errs[-1] < 3e-8
    # the constant mode through log R: SLP of sigma = (1, 0) on the unit circle is
    # sigma/4 (SPEC example; int log rho ds = 0, int r r^T/rho^2 ds = pi I)
    g = oracle.OracleGeometry(make_circle_problem(n_outer=256, R=1.0, pores=()))
    y = g.slp_apply(np.tile([1.0, 0.0], 256)).reshape(-1, 2)
    assert np.abs(y - [0.25, 0.0]).max() < 1e-8


def test_S4_normal_is_a_null_vector():
    """C26: S[n] = 0 on a closed curve; the discrete residual decays at 6th order."""
    errs = []
    for N in (64, 128, 256):
        p = make_circle_problem(n_outer=N, R=1.0, pores=((0.1, -0.05, 0.35),), n_pore=N)
        g = oracle.OracleGeometry(p)
        n = g.nrm.copy()
        n[: 2 * N] = 0.0  # normal of the outer curve only
        errs.append(np.abs(g.slp_apply(n)).max())
        n = g.nrm.copy()
        n[2 * N:] = 0.0   # normal of the pore only
        errs[-1] = max(errs[-1], np.abs(g.slp_apply(n)).max())
    assert errs[2] < 2e-10 and errs[1] < errs[0] / 30 and errs[2] < errs[1] / 30, errs


def _stokes_exact(P, c):
    """Polynomial Stokes flow + Stokeslet (force F) + rotlet centred at c (outside the fluid)."""
    X, Y = P[:, 0], P[:, 1]
    rx, ry = X - c[0], Y - c[1]
    r2 = rx * rx + ry * ry
    F = (0.3, -0.2)
    rf = rx * F[0] + ry * F[1]
    us = (-0.5 * np.log(r2) * F[0] + rx * rf / r2) / (4 * np.pi)
    vs = (-0.5 * np.log(r2) * F[1] + ry * rf / r2) / (4 * np.pi)
    return np.stack([X ** 2 + us + 0.2 * ry / r2, -2 * X * Y + vs - 0.2 * rx / r2], 1)


def test_S5_stokes_flow_end_to_end():
    """Solve S sigma = u_exact on the boundary (BD-GMRES, P:l.596-601, 651-663),
    evaluate the trapezoid field (P:l.346-354) inside: converges to the exact
    Stokes flow at high order."""
    errs = []
    for n in (64, 128):
        p = make_circle_problem(n, 1.0, ((0.0, 0.0, 0.3),), n, 1)
        g = oracle.OracleGeometry(p)
        x = g.x.reshape(-1, 2)
        f = _stokes_exact(x, p.pore_c[0]).reshape(-1)
        r = oracle.slp_gmres(g, f, oracle.OracleSLPBD(g), tol=1e-12, max_iter=200)
        assert r["converged"]
        rng = np.random.default_rng(7)
        rad = rng.uniform(0.45, 0.85, 200)
        ang = rng.uniform(0, 2 * np.pi, 200)
        pts = np.stack([rad * np.cos(ang), rad * np.sin(ang)], 1)
        u = g.slp_field(r["x"], pts)
        errs.append(np.abs(u - _stokes_exact(pts, p.pore_c[0])).max())
    assert errs[0] < 3e-4 and errs[1] < 3e-6, errs


def test_S6_slp_block_is_the_restricted_operator():
    g = oracle.OracleGeometry(make_problem(2))
    rng = np.random.default_rng(3)
    for b in (0, 4, g.M):
        lo, hi = g.body_range(b)
        sig = np.zeros(2 * g.N)
        sig[2 * lo:2 * hi] = rng.standard_normal(2 * (hi - lo))
        full = g.slp_apply(sig, rows=np.arange(lo, hi))
        blk = g.slp_block(b) @ sig[2 * lo:2 * hi]
        assert np.abs(full - blk).max() <= 1e-13 * np.abs(full).max()


def test_S7_slp_gmres_matches_dense_gmres():
    p = make_circle_problem(32, 1.0, ((0.1, 0.0, 0.3),), 32, 1)
    g = oracle.OracleGeometry(p)
    n2 = 2 * g.N
    A = np.stack([g.slp_apply(e) for e in np.eye(n2)], 1)
    f = _stokes_exact(g.x.reshape(-1, 2), p.pore_c[0]).reshape(-1)
    a = oracle.slp_gmres(g, f, None, tol=1e-10, max_iter=n2)
    d = oracle.gmres_dense(A, f, None, tol=1e-10, max_iter=n2)
    # the unpreconditioned first-kind system is ill-conditioned (C26): later
    # history entries are rounding-sensitive, so compare the leading ones
    assert abs(a["iters"] - d["iters"]) <= 2
    assert np.abs(a["hist"][:7] - d["hist"][:7]).max() <= 1e-12
    bd = oracle.OracleSLPBD(g)
    Pinv = np.zeros((n2, n2))
    for b in range(g.M + 1):
        lo, hi = g.body_range(b)
        Pinv[2 * lo:2 * hi, 2 * lo:2 * hi] = bd.block_inverse(b)
    # the SLP blocks are nearly singular (C26: n_b), so entries of B_b^-1 are
    # large; compare at rounding level of |B^-1| |A|
    scale = n2 * np.abs(Pinv).max() * np.abs(A).max() * 1e-15
    assert np.abs(Pinv @ A[:, :4] - np.stack([bd.apply(c) for c in A[:, :4].T], 1)).max() <= scale


def test_S8_kernel_symmetry_of_the_assembled_blocks():
    """G(x, y) = G(y, x) and the KR weights depend only on |offset| (C25): on a
    circle with equal arclength weights, B[i, j] = B[j, i]^T as 2x2 blocks (an
    index, transpose or weight mix-up breaks it)."""
    p = make_circle_problem(n_outer=48, R=0.9, pores=())
    g = oracle.OracleGeometry(p)
    B = g.slp_block(0)
    n = g.N
    Bb = B.reshape(n, 2, n, 2)
    for i in range(0, n, 5):
        for j in range(n):
            assert np.abs(Bb[i, :, j, :] - Bb[j, :, i, :].T).max() <= 1e-15 * np.abs(B).max()
