"""NEXT-2 / NEXT-3 at the large configs: the paper's scenarios through the
whole GPU pipeline (geometry -> structured BD -> BD-GMRES -> field), in the
bench's launch configuration.

* Shear flow on ALL curves (P:l.634-638): u_ref = (y, 0) is a Stokes flow in
  Omega_0 represented by the Gamma_0 density alone, so the discrete solution
  has sigma = 0 on every pore (the paper's observation, P:l.733-736; pin V9 of
  the oracle).  Config 3 is compared with the oracle's own solve.
* Stokeslet/rotlet exact solution (P:l.933-958, eq. analyticalBC): after the
  solve the represented field must equal the formula inside Omega.
* Both report the paper's error field eps(x) = | |u| - |u_ref| | / |u_ref|
  (P:l.752-757) on a grid of points that are reliable for the trapezoid rule,
  d(x, Gamma) > sqrt(ds) (P:l.355-358 footnote; bie_inputs.interior_grid).
"""
import numpy as np
import pytest

import oracle
from bie_inputs import (
    interior_grid,
    make_problem,
    node_positions,
    rhs_shear_all,
    stokeslet_rotlet_field,
    stokeslet_rotlet_params,
)

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


def _grid(p):
    return interior_grid(p, int(10 * p.meta["L"]), 24)


def _eps(u, uref, floor):
    """eps(x) of P:l.752-757 where |u_ref| > floor (it divides by |u_ref|)."""
    nu, nr = np.linalg.norm(u, axis=1), np.linalg.norm(uref, axis=1)
    m = nr > floor
    return np.abs(nu[m] - nr[m]) / nr[m]


def _solve(bie, p, f, tol, max_iter):
    import torch

    g = bie.Geometry.from_problem(p)
    bd = bie.BlockDiag(g, structured=True)
    x = torch.zeros(f.size, dtype=torch.float64, device="cuda")
    r = bie.gmres_solve(g, bd, _t(f), x, tol=tol, max_iter=max_iter)
    return g, x, r


def _field(bie, g, x, pts):
    import torch

    out = torch.zeros(pts.size, dtype=torch.float64, device="cuda")
    bie.field_eval(g, x, _t(pts), out)
    torch.cuda.synchronize()
    return out.cpu().numpy().reshape(-1, 2)


@pytest.mark.parametrize("cid", [3, 4])
def test_shear_all_density_vanishes_on_pores(bie, cid):
    p = make_problem(cid)
    f = rhs_shear_all(p)
    g, x, r = _solve(bie, p, f, 1e-11, 3000)
    assert r["converged"]
    s = x.cpu().numpy().reshape(-1, 2)
    wl = p.M * p.n_pore
    ratio = np.abs(s[:wl]).max() / np.abs(s[wl:]).max()
    pts = _grid(p)
    u = _field(bie, g, x, pts)
    eps = _eps(u, np.stack([pts[:, 1], 0 * pts[:, 1]], 1), 0.05)
    print(f"config {cid} shear: {r['iters']} iterations, pore/wall density ratio {ratio:.3e}, "
          f"eps(x) max {eps.max():.3e} median {np.median(eps):.3e} over {eps.size} points")
    assert ratio < 1e-9
    assert eps.max() < 1e-8
    if cid == 3:
        # the oracle's own solve of the same system (BD in its LU-solve form)
        og = oracle.OracleGeometry(p)
        ro = oracle.gmres_bdlu(og, f, oracle.OracleBDLU(og), tol=1e-11, max_iter=3000)
        so = ro["x"].reshape(-1, 2)
        ratio_o = np.abs(so[:wl]).max() / np.abs(so[wl:]).max()
        print(f"  oracle: {ro['iters']} iterations, ratio {ratio_o:.3e}")
        assert abs(ro["iters"] - r["iters"]) <= 1
        assert ratio < 10 * ratio_o + 1e-12
        assert np.abs(s - so).max() / np.abs(so).max() < 1e-7


@pytest.mark.parametrize("cid", [3, 4])
def test_stokeslet_rotlet_error_field(bie, cid):
    p = make_problem(cid)
    cs, lam, mu = stokeslet_rotlet_params(p)
    f = stokeslet_rotlet_field(node_positions(p), cs, lam, mu).reshape(-1)
    g, x, r = _solve(bie, p, f, 1e-12, 3000)
    assert r["converged"]
    pts = _grid(p)
    u = _field(bie, g, x, pts)
    uref = stokeslet_rotlet_field(pts, cs, lam, mu)
    eps = _eps(u, uref, 1e-3 * np.linalg.norm(uref, axis=1).max())
    err = np.abs(u - uref).max() / np.abs(uref).max()
    print(f"config {cid} Stokeslet/rotlet: {r['iters']} iterations, res_true {r['res_true']:.2e}, "
          f"field max rel err {err:.3e}, eps(x) max {eps.max():.3e} median {np.median(eps):.3e} "
          f"over {eps.size} points")
    assert err < 1e-8
    assert eps.max() < 1e-7
