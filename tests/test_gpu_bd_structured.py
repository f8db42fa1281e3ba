"""GPU parity of the structured pore BD (NEXT-4; bie_blockdiag_factor_structured):
one reference inverse plus a rank-2 Woodbury term per pore (pin V10) against the
explicit per-body inverses (GPU and oracle), and BD-GMRES with it against the
oracle.  The pore blocks of the completed DLP are well conditioned (second
kind), so the bars are those of the explicit BD: 1e-12 on inverses/applies,
1e-10 on BD-GMRES histories (config 2) and the C23 envelope (config 3 golden)."""
import json
import os

import numpy as np
import pytest

import oracle
from bie_inputs import density, make_problem, rhs_pipe, rhs_shear_all

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def bie(cuda_ok):
    from paper_1609_04484_b200 import build as b

    b.build()
    import paper_1609_04484_b200 as pkg

    return pkg


def _t(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).reshape(-1)).cuda()


@pytest.mark.parametrize("cid", [2, 3, 4])
def test_structured_apply_equals_explicit(bie, cid):
    import torch

    p = make_problem(cid)
    g = bie.Geometry.from_problem(p)
    bd_e = bie.BlockDiag(g)
    bd_s = bie.BlockDiag(g, structured=True)
    for nvec in (1, 3):
        v = _t(density(p, nvec=nvec, vec_id=21))
        ze, zs = torch.zeros_like(v), torch.zeros_like(v)
        bie.blockdiag_apply(bd_e, v, ze, nvec)
        bie.blockdiag_apply(bd_s, v, zs, nvec)
        torch.cuda.synchronize()
        a, b = ze.cpu().numpy().reshape(nvec, -1), zs.cpu().numpy().reshape(nvec, -1)
        for q in range(nvec):
            assert np.abs(a[q] - b[q]).max() <= 1e-12 * np.abs(a[q]).max()


def test_structured_block_inverse_vs_oracle(bie):
    p = make_problem(2)
    g = bie.Geometry.from_problem(p)
    og = oracle.OracleGeometry(p)
    obd = oracle.OracleBD(og)
    bd = bie.BlockDiag(g, structured=True)
    for b in (0, 3, p.M - 1, p.M):
        X = bd.block_inverse(b)
        R = obd.block_inverse(b)
        assert np.abs(X - R).max() <= 1e-12 * np.abs(R).max(), b
        # and it inverts the oracle's block (pin of the Woodbury identity, V10)
        B = og.bd_block(b)
        assert np.abs(B @ X - np.eye(B.shape[0])).max() <= 1e-11


@pytest.mark.parametrize("rhs", [rhs_pipe, rhs_shear_all])
def test_structured_bd_gmres_config2(bie, rhs):
    import torch

    p = make_problem(2)
    g = bie.Geometry.from_problem(p)
    og = oracle.OracleGeometry(p)
    f = rhs(p)
    ref = oracle.gmres(og, f, oracle.OracleBD(og), tol=1e-8, max_iter=300)
    x = torch.zeros(f.size, dtype=torch.float64, device="cuda")
    r = bie.gmres_solve(g, bie.BlockDiag(g, structured=True), _t(f), x, tol=1e-8, max_iter=300)
    assert r["iters"] == ref["iters"] and r["converged"]
    big = ref["hist"] > 1e-13
    assert (np.abs(r["hist"] - ref["hist"])[big] / ref["hist"][big]).max() <= 1e-10


@pytest.mark.parametrize("name", ["config3_bd_pipe", "config4_bd_pipe_prefix", "config4_bd_pipe_full"])
def test_structured_bd_gmres_golden(bie, name):
    """Full-size configs in the bench's launch configuration (config 4 is the
    bench workload): oracle goldens with their C23 envelopes."""
    import torch

    path = os.path.join(GOLDEN, f"gmres_{name}.json")
    if not os.path.exists(path):
        pytest.skip("golden not generated")
    from test_gpu_bd_gmres import _golden, golden_check

    gd = _golden(name)
    p = make_problem(gd["config"])
    g = bie.Geometry.from_problem(p)
    f = rhs_pipe(p)
    x = torch.zeros(f.size, dtype=torch.float64, device="cuda")
    r = bie.gmres_solve(g, bie.BlockDiag(g, structured=True), _t(f), x, tol=gd["tol"], max_iter=gd["max_iter"])
    golden_check(r, gd, name + " (structured BD)")


def test_structured_bd_errors(bie):
    p = make_problem(1)
    g = bie.Geometry.from_problem(p)
    with pytest.raises(ValueError):  # structured BDs cover the whole geometry
        bie.BlockDiag(g, structured=True, bodies=(0, 1))
    bd = bie.BlockDiag(g, structured=True)
    sbd = bie.BlockDiag(g, structured=True, op="slp")
    import torch

    f = _t(density(p, nvec=1)[0])
    x = torch.zeros_like(f)
    with pytest.raises(bie.BieError):  # a DLP-operator handle refused by the SLP solver
        bie.gmres_solve_slp(g, bd, f, x, 1e-8, 10)
    with pytest.raises(bie.BieError):  # and an SLP-operator handle by the DLP solver
        bie.gmres_solve(g, sbd, f, x, 1e-8, 10)
