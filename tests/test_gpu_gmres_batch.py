"""NEXT-3: the paper's scenarios (pipe P:l.217-227, shear
P:l.634-638, Stokeslet/rotlet P:l.943-958) solved together by the batched
multi-RHS GMRES; each system must match its own oracle solve (reading C13/C23:
BD histories within 1e-10, equal iteration counts)."""
import numpy as np
import pytest

import oracle
from bie_inputs import (
    density,
    make_problem,
    node_positions,
    rhs_pipe,
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


def _scenarios(p):
    cs, lam, mu = stokeslet_rotlet_params(p)
    return [rhs_pipe(p), rhs_shear_all(p), stokeslet_rotlet_field(node_positions(p), cs, lam, mu).reshape(-1)]


def test_batch_scenarios_match_oracle(bie):
    import torch

    p = make_problem(2)
    g = bie.Geometry.from_problem(p)
    bd = bie.BlockDiag(g)
    og = oracle.OracleGeometry(p)
    obd = oracle.OracleBD(og)
    F = np.stack(_scenarios(p))
    X = torch.zeros(F.size, dtype=torch.float64, device="cuda")
    res = bie.gmres_solve_batch(g, bd, _t(F), X, nrhs=F.shape[0], tol=1e-8, max_iter=500)
    xs = X.cpu().numpy().reshape(F.shape)
    for r in range(F.shape[0]):
        ref = oracle.gmres(og, F[r], obd, tol=1e-8, max_iter=500)
        assert res[r]["iters"] == ref["iters"] and res[r]["converged"]
        big = ref["hist"] > 1e-13
        rel = np.abs(res[r]["hist"][big] - ref["hist"][big]) / ref["hist"][big]
        assert rel.max() <= 1e-10, (r, rel.max())
        assert np.abs(xs[r] - ref["x"]).max() / np.abs(ref["x"]).max() < 1e-9
        assert abs(res[r]["res_true"] - ref["res_true"]) <= 1e-6 * ref["res_true"] + 1e-13


def test_batch_equals_single_solves_many_rhs(bie):
    """17 right-hand sides (two nvec chunks, systems leaving the batch at
    different iterations) vs the single-RHS solver."""
    import torch

    p = make_problem(2)
    g = bie.Geometry.from_problem(p)
    bd = bie.BlockDiag(g)
    F = density(p, nvec=17, vec_id=40)
    F[3] *= 0.0  # a zero right-hand side: converged at iteration 0
    X = torch.zeros(F.size, dtype=torch.float64, device="cuda")
    res = bie.gmres_solve_batch(g, bd, _t(F), X, nrhs=17, tol=1e-8, max_iter=300)
    assert res[3]["iters"] == 0 and res[3]["converged"]
    for r in (0, 5, 16):
        x1 = torch.zeros(2 * p.N, dtype=torch.float64, device="cuda")
        one = bie.gmres_solve(g, bd, _t(F[r]), x1, tol=1e-8, max_iter=300)
        assert res[r]["iters"] == one["iters"]
        rel = np.abs(res[r]["hist"] - one["hist"]) / one["hist"]
        assert rel.max() <= 1e-10


def test_batch_no_pc_and_errors(bie):
    import torch

    p = make_problem(1)
    g = bie.Geometry.from_problem(p)
    F = np.stack(_scenarios_tiny(p))
    X = torch.zeros(F.size, dtype=torch.float64, device="cuda")
    res = bie.gmres_solve_batch(g, None, _t(F), X, nrhs=2, tol=1e-8, max_iter=100)
    assert all(r["converged"] for r in res)
    with pytest.raises(bie.BieError):
        bie.gmres_solve_batch(g, None, _t(F), X, nrhs=0)


def _scenarios_tiny(p):
    from bie_inputs import rhs_rotation_outer, rhs_shear_outer

    return [rhs_rotation_outer(p), rhs_shear_outer(p)]
