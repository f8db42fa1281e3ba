"""NEXT-2: off-surface velocity evaluation on the GPU.

Parity against the oracle's trapezoid field (oracle.ora_field) on the same
density, and two closed forms through the WHOLE GPU pipeline (BD factor,
GMRES, field): Couette flow (V5) and the paper's Stokeslet/rotlet exact
solution (V6, P:l.943-958)."""
import numpy as np
import pytest

import oracle
from bie_inputs import density, make_problem, rhs_rotation_outer, stokeslet_rotlet_field, stokeslet_rotlet_params

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bie(cuda_ok):
    from paper_1609_04484_b200 import build as b

    b.build()
    import paper_1609_04484_b200 as pkg

    return pkg


def _t(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).reshape(-1)).cuda()


def _interior_points(p, n, margin, seed=5):
    rng = np.random.default_rng(seed)
    L, H = p.meta["L"], p.meta["H"]
    pts = []
    while len(pts) < n:
        q = np.array([rng.uniform(0.5, L - 0.5), rng.uniform(-H + margin, H - margin)])
        if np.all(np.linalg.norm(p.pore_c - q, axis=1) - p.pore_r >= margin):
            pts.append(q)
    return np.array(pts)


@pytest.mark.parametrize("cid,npts", [(2, 300), (3, 1000)])
def test_field_parity_random_density(bie, cid, npts):
    import torch

    p = make_problem(cid)
    g = bie.Geometry.from_problem(p)
    og = oracle.OracleGeometry(p)
    s = density(p)[0]
    pts = _interior_points(p, npts, 0.05)
    out = torch.zeros(2 * npts, dtype=torch.float64, device="cuda")
    bie.field_eval(g, _t(s), _t(pts), out)
    torch.cuda.synchronize()
    u = out.cpu().numpy().reshape(-1, 2)
    ref = og.field(s, pts)
    assert np.abs(u - ref).max() / np.abs(ref).max() <= 1e-12


def test_field_empty_and_errors(bie):
    import torch

    p = make_problem(1)
    g = bie.Geometry.from_problem(p)
    s = _t(density(p)[0])
    empty = torch.zeros(0, dtype=torch.float64, device="cuda")
    bie.field_eval(g, s, empty, empty)
    with pytest.raises(bie.BieError):
        bie.field_eval(g, s, _t(np.zeros(4)), s)  # out aliases sigma


def test_couette_closed_form_gpu_pipeline(bie):
    """V5 through the GPU path: rotating unit circle around a still pore."""
    import torch

    p = make_problem(1)
    g = bie.Geometry.from_problem(p)
    bd = bie.BlockDiag(g)
    f = _t(rhs_rotation_outer(p))
    x = torch.zeros_like(f)
    res = bie.gmres_solve(g, bd, f, x, tol=1e-13, max_iter=100)
    assert res["converged"]
    th = np.linspace(0, 2 * np.pi, 9, endpoint=False)
    A, B = 1 / 0.91, -0.09 / 0.91
    for rad, tol in ((0.5, 1e-12), (0.65, 1e-9)):
        pts = rad * np.stack([np.cos(th), np.sin(th)], 1)
        out = torch.zeros(pts.size, dtype=torch.float64, device="cuda")
        bie.field_eval(g, x, _t(pts), out)
        torch.cuda.synchronize()
        u = out.cpu().numpy().reshape(-1, 2)
        ex = (A * rad + B / rad) * np.stack([-np.sin(th), np.cos(th)], 1)
        assert np.abs(u - ex).max() < tol


def test_stokeslet_rotlet_exact_solution_gpu_pipeline(bie):
    """V6 through the GPU path (P:l.943-958): f from Stokeslets/rotlets outside
    Omega; after the BD-GMRES solve the field reproduces f's formula inside."""
    import torch

    p = make_problem(2)
    g = bie.Geometry.from_problem(p)
    bd = bie.BlockDiag(g)
    cs, lam, mu = stokeslet_rotlet_params(p)
    nodes = g.nodes()
    f = _t(stokeslet_rotlet_field(nodes, cs, lam, mu))
    x = torch.zeros_like(f)
    res = bie.gmres_solve(g, bd, f, x, tol=1e-13, max_iter=400)
    assert res["converged"]
    pts = _interior_points(p, 200, 0.3)
    out = torch.zeros(pts.size, dtype=torch.float64, device="cuda")
    bie.field_eval(g, x, _t(pts), out)
    torch.cuda.synchronize()
    u = out.cpu().numpy().reshape(-1, 2)
    ex = stokeslet_rotlet_field(pts, cs, lam, mu)
    assert np.abs(u - ex).max() / np.abs(ex).max() < 1e-11
