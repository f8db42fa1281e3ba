"""GPU parity of the block-diagonal preconditioner (A6/A7) and GMRES (A8/A9)
against the CPU oracle, through the C ABI.

Bars (BASELINE.json north_star, readings C13/C14): GMRES iteration count equal
and residual history within 1e-10 relative at tol 1e-8.  BD inverses: the
explicit inverse is unique, so GPU and oracle agree to rounding x cond(B)."""
import json
import os

import numpy as np
import pytest

import oracle
from bie_inputs import density, make_problem, rhs_pipe, rhs_rotation_outer, rhs_shear_all, rhs_shear_outer
from bie_inputs.geometry import make_circle_problem, make_pipe

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def bie(cuda_ok):
    from paper_1609_04484_b200 import build as b

    b.build()
    import paper_1609_04484_b200 as pkg

    return pkg


_cache = {}


def _setup(bie, problem, with_bd=True):
    key = problem.name
    if key not in _cache:
        g = bie.Geometry.from_problem(problem)
        og = oracle.OracleGeometry(problem)
        _cache[key] = dict(g=g, og=og, bd=None, obd=None)
    c = _cache[key]
    if with_bd and c["bd"] is None:
        c["bd"] = bie.BlockDiag(c["g"])
    return c


def _obd(c):
    if c["obd"] is None:
        c["obd"] = oracle.OracleBD(c["og"])
    return c["obd"]


def _t(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).reshape(-1)).cuda()


@pytest.mark.parametrize("cid", [1, 2])
def test_bd_inverse_parity(bie, cid):
    c = _setup(bie, make_problem(cid))
    obd = _obd(c)
    for b in sorted({0, c["og"].M - 1, c["og"].M}):
        gi = c["bd"].block_inverse(b)
        oi = obd.block_inverse(b)
        assert np.abs(gi - oi).max() / np.abs(oi).max() < 1e-12, b
        B = c["og"].bd_block(b)
        assert np.abs(gi @ B - np.eye(B.shape[0])).max() < 1e-12


def test_bd_apply_parity(bie):
    import torch

    c = _setup(bie, make_problem(2))
    obd = _obd(c)
    v = density(c["og"].problem, nvec=5, vec_id=3)
    out = torch.zeros(v.size, dtype=torch.float64, device="cuda")
    bie.blockdiag_apply(c["bd"], _t(v), out, nvec=5)
    torch.cuda.synchronize()
    z = out.cpu().numpy().reshape(5, -1)
    for k in range(5):
        ref = obd.apply(v[k])
        assert np.abs(z[k] - ref).max() / np.abs(ref).max() < 1e-12


@pytest.mark.parametrize("cid", [3, 4])
def test_bd_large_blocks_inverse_property(bie, cid):
    """Sizes the oracle cannot invert in seconds: check B (B^{-1} v) = v with the
    oracle-assembled blocks (wall: 4096^2 / 16384^2; a few pores)."""
    import torch

    p = make_problem(cid)
    c = _setup(bie, p)
    og = c["og"]
    v = density(p, nvec=1, vec_id=9)[0]
    out = torch.zeros(v.size, dtype=torch.float64, device="cuda")
    bie.blockdiag_apply(c["bd"], _t(v), out)
    torch.cuda.synchronize()
    z = out.cpu().numpy()
    for b in (0, p.M // 2, p.M - 1, p.M):
        lo, hi = og.body_range(b)
        B = og.bd_block(b)
        r = B @ z[2 * lo:2 * hi] - v[2 * lo:2 * hi]
        assert np.abs(r).max() / np.abs(v[2 * lo:2 * hi]).max() < 1e-10, b


FLOOR = 1e-13  # estimates below this are rounding noise on both sides (C14)


def _cmp_gmres(res, ref, tol_hist=1e-10):
    assert res["iters"] == ref["iters"], (res["iters"], ref["iters"])
    assert res["converged"] == ref["converged"]
    h, hr = np.asarray(res["hist"]), np.asarray(ref["hist"])
    assert h.shape == hr.shape
    big = hr > FLOOR
    rel = np.abs(h[big] - hr[big]) / np.abs(hr[big])
    assert rel.max() <= tol_hist, rel.max()
    assert np.all(h[~big] <= FLOOR)


CASES = {
    "c1_rotation": (lambda: make_problem(1), rhs_rotation_outer),
    "c1_shear_outer": (lambda: make_problem(1), rhs_shear_outer),
    "c1_offcentre_shear": (lambda: make_circle_problem(64, 1.0, ((0.2, -0.1, 0.3),), 64, 1, "c1off"), rhs_shear_outer),
    "c2_pipe": (lambda: make_problem(2), rhs_pipe),
    "c2_shear_all": (lambda: make_problem(2), rhs_shear_all),
}


@pytest.mark.parametrize("case", list(CASES))
def test_gmres_parity_bd(bie, case):
    """BD-preconditioned histories are well conditioned (the oracle's own history
    moves by ~2e-13 under 1e-15 perturbations of f): strict 1e-10 bar."""
    import torch

    mk, rhs = CASES[case]
    p = mk()
    c = _setup(bie, p)
    f = rhs(p)
    ref = oracle.gmres(c["og"], f, _obd(c), tol=1e-8, max_iter=1000)
    x = torch.zeros(f.size, dtype=torch.float64, device="cuda")
    res = bie.gmres_solve(c["g"], c["bd"], _t(f), x, tol=1e-8, max_iter=1000)
    _cmp_gmres(res, ref)
    xs = x.cpu().numpy()
    assert np.abs(xs - ref["x"]).max() / np.abs(ref["x"]).max() < 1e-9
    assert abs(res["res_true"] - ref["res_true"]) <= 1e-6 * ref["res_true"] + 1e-13
    assert abs(res["res_pc"] - ref["res_pc"]) <= 1e-6 * ref["res_pc"] + 1e-13


def _oracle_envelope(og, f, n_runs=4, eps=1e-13):
    """Oracle no-PC histories under 1e-13 relative perturbations of f (reading C23;
    1e-13 is the GPU-vs-oracle matvec agreement level)."""
    runs = []
    for s in range(n_runs):
        rng = np.random.default_rng(100 + s)
        runs.append(oracle.gmres(og, f * (1 + eps * rng.standard_normal(f.size)), None, tol=1e-8, max_iter=1000))
    return runs


@pytest.mark.parametrize("case", list(CASES))
def test_gmres_parity_nopc(bie, case):
    """No-PC histories are ill conditioned (reading C23: the oracle's own history
    moves by up to 13% on config 2, and the off-centre tiny case changes its
    iteration count, under 1e-15 perturbations of f).  The GPU history must
    lie within 10x the oracle's own perturbation envelope (floor 1e-10), and
    its iteration count within the perturbed oracle runs' range."""
    import torch

    mk, rhs = CASES[case]
    p = mk()
    c = _setup(bie, p, with_bd=False)
    f = rhs(p)
    ref = oracle.gmres(c["og"], f, None, tol=1e-8, max_iter=1000)
    runs = _oracle_envelope(c["og"], f)
    x = torch.zeros(f.size, dtype=torch.float64, device="cuda")
    res = bie.gmres_solve(c["g"], None, _t(f), x, tol=1e-8, max_iter=1000)
    its = [r["iters"] for r in runs] + [ref["iters"]]
    assert min(its) - 1 <= res["iters"] <= max(its) + 1, (res["iters"], its)
    n = min([res["iters"]] + its) + 1
    hr = ref["hist"][:n]
    env = np.max([np.abs(r["hist"][:n] - hr) / hr for r in runs], axis=0)
    env = np.maximum.accumulate(env)  # a chaotic divergence only grows
    big = hr > FLOOR
    rel = np.abs(res["hist"][:n] - hr) / hr
    assert np.all(rel[big] <= np.maximum(1e-10, 10 * env[big])), (rel.max(), env.max())
    assert res["converged"] and res["res_true"] < 1e-7


def test_gmres_single_body_one_iteration(bie):
    import torch

    p = make_pipe(0, 10.0, 256, 0, (0.1, 0.2), 0.05, 16)
    c = _setup(bie, p)
    f = rhs_pipe(p)
    x = torch.zeros(f.size, dtype=torch.float64, device="cuda")
    res = bie.gmres_solve(c["g"], c["bd"], _t(f), x, tol=1e-8, max_iter=20)
    assert res["iters"] == 1 and res["converged"]


def test_gmres_cap_not_converged(bie):
    import torch

    p = make_problem(2)
    c = _setup(bie, p)
    f = rhs_pipe(p)
    x = torch.zeros(f.size, dtype=torch.float64, device="cuda")
    res = bie.gmres_solve(c["g"], None, _t(f), x, tol=1e-8, max_iter=7)
    assert res["iters"] == 7 and not res["converged"]
    ref = oracle.gmres(c["og"], f, None, tol=1e-8, max_iter=7)
    _cmp_gmres(res, ref)


def test_gmres_deterministic(bie):
    import torch

    p = make_problem(2)
    c = _setup(bie, p)
    f = _t(rhs_pipe(p))
    outs = []
    for _ in range(2):
        x = torch.zeros_like(f)
        r = bie.gmres_solve(c["g"], c["bd"], f, x, tol=1e-8, max_iter=200)
        outs.append((r["hist"], x.cpu().numpy()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("name", ["config3_bd_pipe", "config4_none_pipe_prefix", "config4_bd_pipe_prefix",
                                  "config4_bd_pipe_full"])
def test_gmres_golden(bie, name):
    """Large configs: histories produced by tools/make_golden.py (oracle only;
    config 4's BD uses the oracle's LU-solve form of the same operator)."""
    import torch

    path = os.path.join(GOLDEN, f"gmres_{name}.json")
    if not os.path.exists(path):
        pytest.skip(f"golden {path} not generated")
    gd = json.load(open(path))
    p = make_problem(gd["config"])
    use_bd = gd["pc"] in ("bd", "bdlu")
    c = _setup(bie, p, with_bd=use_bd)
    f = rhs_pipe(p)
    assert abs(np.linalg.norm(f) - gd["f_norm"]) < 1e-12 * gd["f_norm"]
    x = torch.zeros(f.size, dtype=torch.float64, device="cuda")
    res = bie.gmres_solve(c["g"], c["bd"] if use_bd else None, _t(f), x, tol=gd["tol"], max_iter=gd["max_iter"])
    assert res["iters"] == gd["iters"] and res["converged"] == gd["converged"]
    hr = np.asarray(gd["hist"])
    env = np.maximum.accumulate(np.asarray(gd.get("envelope", np.zeros(hr.size))))
    rel = np.abs(np.asarray(res["hist"]) - hr) / hr
    # 1e-10 bar, relaxed only where the oracle's own history moves more under
    # 1e-13 perturbations of f (reading C23)
    assert np.all(rel <= np.maximum(1e-10, 10 * env)), (rel.max(), env.max())


def test_abi_handle_and_argument_errors(bie):
    """Wrong-geometry blockdiag, bad nvec, aliasing, double destroy -> BIE_EINVAL."""
    import ctypes

    import torch

    p1, p2 = make_problem(1), make_pipe(0, 10.0, 256, 0, (0.1, 0.2), 0.05, 16)
    c1, c2 = _setup(bie, p1), _setup(bie, p2)
    f = _t(rhs_rotation_outer(p1))
    x = torch.zeros_like(f)
    with pytest.raises(bie.BieError) as ei:
        bie.gmres_solve(c1["g"], c2["bd"], f, x)
    assert ei.value.code == -1 and "another geometry" in str(ei.value)
    v = torch.zeros(17 * 2 * p1.N, dtype=torch.float64, device="cuda")
    out = torch.zeros_like(v)
    with pytest.raises(bie.BieError):
        bie.dlp_apply(c1["g"], v, out, nvec=17)
    with pytest.raises(bie.BieError):
        bie.blockdiag_apply(c1["bd"], v, v, nvec=1)
    with pytest.raises(bie.BieError):
        bie.gmres_solve(c1["g"], c1["bd"], f, f)
    # a blockdiag handle passed where a geometry is expected (handle-kind check)
    assert bie.lib().bie_geometry_info(ctypes.c_void_p(c1["bd"].h.value), ctypes.byref(ctypes.c_int()),
                                       ctypes.byref(ctypes.c_int())) == -1


def test_pinned_host_end_to_end(bie):
    """bie_dlp_apply_host with pinned torch buffers (the e2e path of bench.py)."""
    import torch

    from paper_1609_04484_b200._bie import dlp_apply_host_ptr

    p = make_problem(2)
    c = _setup(bie, p, with_bd=False)
    s = density(p, nvec=4)
    hs = torch.from_numpy(s.reshape(-1).copy()).pin_memory()
    ho = torch.zeros_like(hs).pin_memory()
    dlp_apply_host_ptr(c["g"], hs.data_ptr(), ho.data_ptr(), nvec=4)
    ref = c["og"].apply(s)
    y = ho.numpy().reshape(4, -1)
    for v in range(4):
        assert np.abs(y[v] - ref[v]).max() / np.abs(ref[v]).max() <= 1e-12
