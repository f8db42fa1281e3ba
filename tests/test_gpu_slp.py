"""GPU parity of the single-layer operator with the Kapur-Rokhlin correction
(NEXT-1; P:l.270-330) against the CPU oracle, through the C ABI.

Bars: matvec and field evaluation max-norm relative 1e-12 per vector (as C15);
BD inverses and GMRES histories of the nearly singular SLP blocks follow the
conditioning readings C23/C26 (envelopes measured with the oracle here)."""
import json
import os

import numpy as np
import pytest

import oracle
from bie_inputs import density, make_problem, rhs_pipe, rhs_shear_all
from bie_inputs.geometry import make_circle_problem

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module")
def bie(cuda_ok):
    from paper_1609_04484_b200 import build as b

    b.build()
    import paper_1609_04484_b200 as pkg

    return pkg


_cache = {}


def _setup(bie, problem):
    key = problem.name
    if key not in _cache:
        _cache[key] = (bie.Geometry.from_problem(problem), oracle.OracleGeometry(problem))
    return _cache[key]


def _t(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).reshape(-1)).cuda()


def _gpu_slp(bie, g, s, nvec, flags=0):
    import torch

    sig = _t(s)
    out = torch.full_like(sig, float("nan"))
    bie.slp_apply(g, sig, out, nvec, flags)
    torch.cuda.synchronize()
    return out.cpu().numpy().reshape(nvec, -1)


def _relerr(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


def _rows(p, n=1024):
    """Sampled target rows incl. every KR seam: first/last nodes of pores and wall."""
    N = p.N
    r = [np.linspace(0, N - 1, n).astype(np.int64), [0, 1, 5, 6, 7, N - 7, N - 6, N - 1]]
    if p.M:
        for k in (0, 1, p.M // 2, p.M - 1):
            lo = k * p.n_pore
            r.append([lo, lo + 1, lo + 6, lo + p.n_pore - 6, lo + p.n_pore - 1])
        w0 = p.M * p.n_pore
        r.append([w0, w0 + 1, w0 + 6, w0 + 7])
    return np.unique(np.concatenate(r)).astype(np.int32)


@pytest.mark.parametrize("cid", [1, 2])
@pytest.mark.parametrize("flags", [0, 2])  # symmetric path, one-sided path
def test_slp_matvec_full_parity(bie, cid, flags):
    p = make_problem(cid)
    g, og = _setup(bie, p)
    s = density(p, nvec=1)
    y = _gpu_slp(bie, g, s, 1, flags)[0]
    ref = og.slp_apply(s[0])
    assert _relerr(y, ref) <= TOL


@pytest.mark.parametrize("nvec", [4, 16, 3])
def test_slp_matvec_multivector(bie, nvec):
    p = make_problem(2)
    g, og = _setup(bie, p)
    s = density(p, nvec=nvec, vec_id=11)
    y = _gpu_slp(bie, g, s, nvec)
    ref = og.slp_apply(s)
    for v in range(nvec):
        assert _relerr(y[v], ref[v]) <= TOL


@pytest.mark.parametrize("cid", [3, 4])
def test_slp_matvec_sampled_rows_large(bie, cid):
    """Full-size configs in the launch configuration the bench uses (nvec = 1,
    symmetric path), checked on sampled rows incl. every curve seam."""
    p = make_problem(cid)
    g, og = _setup(bie, p)
    s = density(p, nvec=1)
    y = _gpu_slp(bie, g, s, 1)[0].reshape(-1, 2)
    rows = _rows(p)
    ref = og.slp_apply(s[0], rows=rows).reshape(-1, 2)
    assert np.abs(y[rows] - ref).max() / np.abs(ref).max() <= TOL


def test_slp_apply_rows_matches_full(bie):
    import torch

    p = make_problem(2)
    g, og = _setup(bie, p)
    s = density(p, nvec=2, vec_id=3)
    full = _gpu_slp(bie, g, s, 2)
    rb, re_ = 100, p.N - 250
    out = torch.zeros(2 * 2 * (re_ - rb), dtype=torch.float64, device="cuda")
    bie.slp_apply_rows(g, _t(s), out, rb, re_, nvec=2)
    torch.cuda.synchronize()
    o = out.cpu().numpy().reshape(2, -1)
    for v in range(2):
        assert _relerr(o[v], full[v, 2 * rb:2 * re_]) <= 1e-13


def test_slp_field_parity(bie):
    import torch

    p = make_problem(2)
    g, og = _setup(bie, p)
    s = density(p, nvec=1)[0]
    rng = np.random.default_rng(4)
    tg = np.stack([rng.uniform(0.2, 9.8, 777), rng.uniform(-0.8, 0.8, 777)], 1)
    out = torch.zeros(2 * 777, dtype=torch.float64, device="cuda")
    bie.slp_field_eval(g, _t(s), _t(tg), out)
    torch.cuda.synchronize()
    ref = og.slp_field(s, tg)
    assert _relerr(out.cpu().numpy().reshape(-1, 2), ref) <= TOL


def test_kr_weights_library_equals_oracle(bie):
    assert np.abs(bie.kr_weights() - oracle.kr_weights()).max() <= 4 * np.spacing(26.0)


def test_slp_blockdiag_inverse_and_apply(bie):
    """BD inverses of nearly singular blocks (C26): compare as backward errors --
    B_b X_gpu = I to the block's conditioning, and the GPU apply equals X_gpu v."""
    import torch

    p = make_problem(2)
    g, og = _setup(bie, p)
    bd = bie.BlockDiag(g, op="slp")
    for b in (0, 7, p.M):
        B = og.slp_block(b)
        X = bd.block_inverse(b)
        cond = np.linalg.cond(B)
        res = np.abs(B @ X - np.eye(B.shape[0])).max()
        assert res <= 50 * cond * 1e-16, (b, res, cond)
        Xo = oracle.OracleSLPBD(og).block_inverse(b) if b == 0 else None
        if Xo is not None:
            assert np.abs(X - Xo).max() / np.abs(Xo).max() <= 50 * cond * 1e-16
    v = density(p, nvec=1, vec_id=9)[0]
    z = torch.zeros(2 * p.N, dtype=torch.float64, device="cuda")
    bie.blockdiag_apply(bd, _t(v), z)
    torch.cuda.synchronize()
    zc = z.cpu().numpy()
    for b in (0, p.M):
        lo, hi = og.body_range(b)
        ref = bd.block_inverse(b) @ v[2 * lo:2 * hi]
        assert np.abs(zc[2 * lo:2 * hi] - ref).max() <= 1e-12 * np.abs(ref).max()


EPS_FILE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "round2", "disagreement.json")


def _slp_perturbation(cid):
    """Measured GPU-vs-oracle disagreement of the SLP primitives (matvec, BD
    apply) and the Krylov primitives (tools/measure_disagreement.py)."""
    d = json.load(open(EPS_FILE))[f"config{cid}"]
    return {"A": max(x["rms"] for x in d["slp_matvec"]), "P": max(x["rms"] for x in d["slp_bd"]),
            "dot": d["dot"]["rms"], "norm": d["norm"]["rms"], "sub": d["sub"]["rms"]}


def _envelope(og, f, max_iter, cid):
    """Oracle self-sensitivity of the SLP BD-GMRES history (C23/C26): three runs
    with every iteration primitive perturbed at its measured GPU-vs-oracle
    disagreement (the near-singular SLP blocks make P^-1 the dominant term)."""
    a = oracle.slp_gmres(og, f, oracle.OracleSLPBD(og), tol=1e-8, max_iter=max_iter)
    runs = []
    for s_ in range(3):
        with oracle.perturbed(_slp_perturbation(cid), seed=3000 + s_):
            runs.append(oracle.slp_gmres(og, f, oracle.OracleSLPBD(og), tol=1e-8, max_iter=max_iter))
    k = min([len(a["hist"])] + [len(r["hist"]) for r in runs])
    env = np.max([np.abs(r["hist"][:k] - a["hist"][:k]) / a["hist"][:k] for r in runs], axis=0)
    return a, np.maximum.accumulate(env), {a["iters"]} | {r["iters"] for r in runs}


@pytest.mark.parametrize("cid", [1, 2])
def test_slp_bd_gmres_parity(bie, cid):
    import torch

    p = make_problem(cid)
    g, og = _setup(bie, p)
    f = rhs_pipe(p) if cid > 1 else np.ascontiguousarray(
        np.stack([-og.x.reshape(-1, 2)[:, 1], og.x.reshape(-1, 2)[:, 0]], 1).reshape(-1))
    ref, env, its = _envelope(og, f, 300, cid)
    bd = bie.BlockDiag(g, op="slp")
    x = torch.zeros(2 * p.N, dtype=torch.float64, device="cuda")
    r = bie.gmres_solve_slp(g, bd, _t(f), x, 1e-8, 300)
    assert r["converged"] and ref["converged"]
    assert min(its) <= r["iters"] <= max(its), (r["iters"], its)
    k = min(len(r["hist"]), len(env))
    bar = np.maximum(1e-10, 2 * env[:k])
    rel = np.abs(r["hist"][:k] - ref["hist"][:k]) / ref["hist"][:k]
    print(f"SLP config {cid}: max GPU dev {rel.max():.3e}, max env {env.max():.3e}, dev/bar {(rel / bar).max():.3f}")
    assert np.all(rel <= bar), (rel.max(), np.argmax(rel / bar))


def test_slp_gmres_nopc_leading_history(bie):
    """Unpreconditioned first-kind system: the leading history entries are well
    conditioned (test_oracle_slp S7); later ones are not (C26)."""
    import torch

    p = make_problem(1)
    g, og = _setup(bie, p)
    f = density(p, nvec=1, vec_id=2)[0]
    ref = oracle.slp_gmres(og, f, None, tol=1e-8, max_iter=60)
    x = torch.zeros(2 * p.N, dtype=torch.float64, device="cuda")
    r = bie.gmres_solve_slp(g, None, _t(f), x, 1e-8, 60)
    assert np.abs(r["hist"][:7] - ref["hist"][:7]).max() / ref["hist"][:7].min() <= 1e-10


def _stokes_exact(P, c):
    X, Y = P[:, 0], P[:, 1]
    rx, ry = X - c[0], Y - c[1]
    r2 = rx * rx + ry * ry
    F = (0.3, -0.2)
    rf = rx * F[0] + ry * F[1]
    us = (-0.5 * np.log(r2) * F[0] + rx * rf / r2) / (4 * np.pi)
    vs = (-0.5 * np.log(r2) * F[1] + ry * rf / r2) / (4 * np.pi)
    return np.stack([X ** 2 + us + 0.2 * ry / r2, -2 * X * Y + vs - 0.2 * rx / r2], 1)


def test_slp_stokes_flow_end_to_end_gpu(bie):
    """The whole SLP pipeline on the GPU (BD factor, BD-GMRES, field) recovers an
    exact Stokes flow as the oracle does (test_oracle_slp S5)."""
    import torch

    p = make_circle_problem(128, 1.0, ((0.0, 0.0, 0.3),), 128, 1)
    g = bie.Geometry.from_problem(p)
    xy = g.nodes()
    f = _stokes_exact(xy, p.pore_c[0]).reshape(-1)
    bd = bie.BlockDiag(g, op="slp")
    x = torch.zeros(2 * p.N, dtype=torch.float64, device="cuda")
    r = bie.gmres_solve_slp(g, bd, _t(f), x, 1e-12, 200)
    assert r["converged"]
    rng = np.random.default_rng(7)
    rad, ang = rng.uniform(0.45, 0.85, 200), rng.uniform(0, 2 * np.pi, 200)
    pts = np.stack([rad * np.cos(ang), rad * np.sin(ang)], 1)
    u = torch.zeros(400, dtype=torch.float64, device="cuda")
    bie.slp_field_eval(g, x, _t(pts), u)
    torch.cuda.synchronize()
    assert np.abs(u.cpu().numpy().reshape(-1, 2) - _stokes_exact(pts, p.pore_c[0])).max() < 3e-6


def test_slp_batch_gmres_matches_single(bie):
    import torch

    p = make_problem(2)
    g, og = _setup(bie, p)
    bd = bie.BlockDiag(g, op="slp")
    F = np.stack([rhs_pipe(p), rhs_shear_all(p)])  # physical (zero-flux) data, C26
    X = torch.zeros(F.size, dtype=torch.float64, device="cuda")
    rb = bie.gmres_solve_batch_slp(g, bd, _t(F), X, 2, 1e-8, 300)
    for q in range(2):
        x = torch.zeros(2 * p.N, dtype=torch.float64, device="cuda")
        rs = bie.gmres_solve_slp(g, bd, _t(F[q]), x, 1e-8, 300)
        assert abs(rb[q]["iters"] - rs["iters"]) <= 1
        k = min(len(rb[q]["hist"]), len(rs["hist"]))
        # batched (nvec-wide) and single applications round differently; the BD
        # SLP history is sensitive at the 1e-6 level (C26)
        assert (np.abs(rb[q]["hist"][:k] - rs["hist"][:k]) / rs["hist"][:k]).max() < 1e-4


def test_slp_abi_errors(bie):
    import torch

    p = make_problem(1)
    g, _ = _setup(bie, p)
    s = _t(density(p, nvec=1)[0])
    o = torch.zeros_like(s)
    with pytest.raises(bie.BieError):
        bie.slp_apply(g, s, o, 1, 1)  # BIE_D_ONLY is not an SLP flag
    with pytest.raises(bie.BieError):
        bie.slp_apply(g, s, s, 1)     # aliasing
    dlp_bd = bie.BlockDiag(g)
    with pytest.raises(bie.BieError):
        bie.gmres_solve_slp(g, dlp_bd, s, o, 1e-8, 10)
    slp_bd = bie.BlockDiag(g, op="slp")
    with pytest.raises(bie.BieError):
        bie.gmres_solve(g, slp_bd, s, o, 1e-8, 10)


@pytest.mark.parametrize("n", [64, 100, 16])
def test_single_curve_no_pores(bie, n):
    """Edge case: a geometry with no pores (M = 0), node counts below one
    512-block and not a multiple of the 32-node chunk; DLP and SLP parity."""
    p = make_circle_problem(n_outer=n, R=1.3, pores=())
    g = bie.Geometry.from_problem(p)
    og = oracle.OracleGeometry(p)
    s = density(p, nvec=2, vec_id=1)
    y = _gpu_slp(bie, g, s, 2)
    ref = og.slp_apply(s)
    for v in range(2):
        assert _relerr(y[v], ref[v]) <= TOL
    import torch

    sig = _t(s)
    out = torch.full_like(sig, float("nan"))
    bie.dlp_apply(g, sig, out, 2)
    torch.cuda.synchronize()
    yd = out.cpu().numpy().reshape(2, -1)
    refd = og.apply(s)
    for v in range(2):
        assert _relerr(yd[v], refd[v]) <= TOL


def test_slp_one_sided_sampled_config3(bie):
    p = make_problem(3)
    g, og = _setup(bie, p)
    s = density(p, nvec=1, vec_id=5)
    y = _gpu_slp(bie, g, s, 1, 2)[0].reshape(-1, 2)
    rows = _rows(p, 512)
    ref = og.slp_apply(s[0], rows=rows).reshape(-1, 2)
    assert np.abs(y[rows] - ref).max() / np.abs(ref).max() <= TOL


def test_slp_matvec_config5_sampled_rows(bie):
    """Config 5 (N = 1.06M), the symmetric SLP path, 128 strided rows vs the oracle."""
    p = make_problem(5)
    g, og = _setup(bie, p)
    s = density(p, nvec=1)
    y = _gpu_slp(bie, g, s, 1)[0].reshape(-1, 2)
    rows = _rows(p, 128)
    ref = og.slp_apply(s[0], rows=rows).reshape(-1, 2)
    assert np.abs(y[rows] - ref).max() / np.abs(ref).max() <= TOL


@pytest.mark.parametrize("n_pore", [16, 18])
def test_minimum_nodes_per_pore(bie, n_pore):
    """Edge case: the smallest allowed pores (16 nodes, and a non-power-of-two
    count), where the +-6 KR neighbourhoods cover most of the curve."""
    p = make_circle_problem(n_outer=32, R=1.0, pores=((0.3, 0.1, 0.2), (-0.4, -0.2, 0.15)), n_pore=n_pore)
    g = bie.Geometry.from_problem(p)
    og = oracle.OracleGeometry(p)
    s = density(p, nvec=1, vec_id=6)
    assert _relerr(_gpu_slp(bie, g, s, 1)[0], og.slp_apply(s[0])) <= TOL
    import torch

    sig = _t(s)
    out = torch.full_like(sig, float("nan"))
    bie.dlp_apply(g, sig, out, 1)
    torch.cuda.synchronize()
    assert _relerr(out.cpu().numpy(), og.apply(s[0])) <= TOL


@pytest.mark.parametrize("scale", [1e-5, 1e5])
@pytest.mark.parametrize("flags", [0, 2])  # symmetric path, one-sided path
def test_length_scale_extremes(bie, scale, flags):
    """Edge case: the same geometry at 1e-5 and 1e5 length units (rho^2 from
    ~1e-17 to ~4e10: the table logs' mantissa and exponent tables over ~90
    binades); SLP and DLP parity on N = 1,792 (several 512-blocks)."""
    import torch

    s_ = scale
    p = make_circle_problem(n_outer=1024, R=1.0 * s_, n_pore=256, name=f"scaled{s_:g}",
                            pores=((0.3 * s_, 0.1 * s_, 0.2 * s_), (-0.4 * s_, -0.2 * s_, 0.15 * s_),
                                   (0.1 * s_, -0.5 * s_, 0.12 * s_)))
    g = bie.Geometry.from_problem(p)
    og = oracle.OracleGeometry(p)
    s = density(p, nvec=1, vec_id=8)
    assert _relerr(_gpu_slp(bie, g, s, 1, flags)[0], og.slp_apply(s[0])) <= TOL
    sig = _t(s)
    out = torch.full_like(sig, float("nan"))
    bie.dlp_apply(g, sig, out, 1, flags)
    torch.cuda.synchronize()
    assert _relerr(out.cpu().numpy(), og.apply(s[0])) <= TOL


@pytest.mark.parametrize("cid", [1, 2, 3])
def test_structured_slp_bd_inverse(bie, cid):
    """Rotating-frame block-circulant pore inverses (bie_blockdiag_factor_structured_slp):
    B_k X_k = I to the block's conditioning against the oracle's assembled SLP
    block (C26: backward error, the blocks are nearly singular), for pores of
    different radii; the wall is the explicit inverse of bie_blockdiag_factor_slp."""
    p = make_problem(cid)
    g, og = _setup(bie, p)
    bd = bie.BlockDiag(g, op="slp", structured=True)
    radii = np.asarray(p.pore_r)
    for b in sorted({0, int(np.argmin(radii)), int(np.argmax(radii)), p.M - 1}):
        B = og.slp_block(b)
        X = bd.block_inverse(b)
        cond = np.linalg.cond(B)
        res = np.abs(B @ X - np.eye(B.shape[0])).max()
        assert res <= 50 * cond * 1e-16, (b, res, cond)
    if cid <= 2:
        Bw = og.slp_block(p.M)
        Xw = bd.block_inverse(p.M)
        assert np.abs(Bw @ Xw - np.eye(Bw.shape[0])).max() <= 50 * np.linalg.cond(Bw) * 1e-16


def test_structured_slp_bd_apply(bie):
    """The structured apply equals X_k v with X_k = its own materialised inverse
    (1e-12), pore by pore and on the wall, for nvec = 1 and 3."""
    import torch

    p = make_problem(2)
    g, og = _setup(bie, p)
    bd = bie.BlockDiag(g, op="slp", structured=True)
    for nvec in (1, 3):
        v = density(p, nvec=nvec, vec_id=11)
        z = torch.zeros(v.size, dtype=torch.float64, device="cuda")
        bie.blockdiag_apply(bd, _t(v), z, nvec)
        torch.cuda.synchronize()
        zc = z.cpu().numpy().reshape(nvec, -1)
        for b in (0, 4, p.M):
            lo, hi = og.body_range(b)
            X = bd.block_inverse(b)
            for q in range(nvec):
                ref = X @ v[q, 2 * lo:2 * hi]
                assert np.abs(zc[q, 2 * lo:2 * hi] - ref).max() <= 1e-12 * np.abs(ref).max(), (nvec, b, q)


@pytest.mark.parametrize("cid", [2, 3])
def test_structured_slp_bd_gmres(bie, cid):
    """BD-GMRES on the SLP system with the structured pore inverses converges in
    the explicit-inverse solve's iteration count (+-1: the two inverses of the
    nearly singular blocks differ at cond x eps, C26) to the same solution."""
    import torch

    p = make_problem(cid)
    g, _ = _setup(bie, p)
    f = _t(rhs_pipe(p))
    xs, xe = torch.zeros_like(f), torch.zeros_like(f)
    rs = bie.gmres_solve_slp(g, bie.BlockDiag(g, op="slp", structured=True), f, xs, 1e-8, 1000)
    re_ = bie.gmres_solve_slp(g, bie.BlockDiag(g, op="slp"), f, xe, 1e-8, 1000)
    assert rs["converged"] and re_["converged"]
    assert abs(rs["iters"] - re_["iters"]) <= 1, (rs["iters"], re_["iters"])
    # the densities differ in the near-null directions S n_b = O(h^6) (C26), which
    # the BD-preconditioned residual does not see; the velocity they represent
    # inside the fluid (reliable points, d > sqrt(ds)) agrees
    from bie_inputs.geometry import interior_grid

    pts = interior_grid(p, int(4 * p.meta["L"]), 12)
    us, ue = torch.zeros(pts.size, dtype=torch.float64, device="cuda"), torch.zeros(pts.size, dtype=torch.float64,
                                                                                   device="cuda")
    bie.slp_field_eval(g, xs, _t(pts), us)
    bie.slp_field_eval(g, xe, _t(pts), ue)
    torch.cuda.synchronize()
    us, ue = us.cpu().numpy(), ue.cpu().numpy()
    dev = np.abs(us - ue).max() / np.abs(ue).max()
    print(f"config {cid}: iterations {rs['iters']} / {re_['iters']}, res_true {rs['res_true']:.2e} / "
          f"{re_['res_true']:.2e}, interior field deviation {dev:.2e} on {len(pts)} points")
    # both solutions carry the first-kind system's residual (C26): the structured
    # inverse is exact for the ideal circulant block, the explicit one for the
    # assembled block; they differ by cond x eps in the near-null directions, so
    # the fields agree to the explicit solve's own true residual
    assert dev <= 10 * re_["res_true"], (dev, re_["res_true"])
