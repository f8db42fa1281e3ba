"""GPU parity of the completed DLP matvec (A2-A5) against the CPU oracle,
through the C ABI.  Bar (BASELINE.json north_star, reading C15):
max_i |y_gpu - y_ora| / max_i |y_ora| <= 1e-12 per density vector."""
import numpy as np
import pytest

import oracle
from bie_inputs import density, make_problem
from bie_inputs.geometry import make_circle_problem, make_pipe

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


def _gpu_apply(bie, g, s, nvec, flags=0):
    import torch

    sig = torch.from_numpy(np.ascontiguousarray(s).reshape(-1)).cuda()
    out = torch.full_like(sig, float("nan"))
    bie.dlp_apply(g, sig, out, nvec, flags)
    torch.cuda.synchronize()
    return out.cpu().numpy().reshape(nvec, -1)


def _relerr(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


def _rows(N, n=1536):
    r = np.unique(np.concatenate([np.linspace(0, N - 1, n).astype(np.int64), [0, 1, N - 2, N - 1]]))
    return r.astype(np.int32)


@pytest.mark.parametrize("cid", [1, 2])
@pytest.mark.parametrize("flags", [0, 1])
def test_matvec_full_parity_small(bie, cid, flags):
    p = make_problem(cid)
    g, og = _setup(bie, p)
    s = density(p, nvec=1)
    y = _gpu_apply(bie, g, s, 1, flags)
    ref = og.apply(s, flags=flags)
    assert np.all(np.isfinite(y))
    assert _relerr(y[0], ref[0]) <= TOL


@pytest.mark.parametrize("nvec", [2, 3, 4, 5, 8, 11, 16])
def test_matvec_nvec_parity(bie, nvec):
    p = make_problem(2)
    g, og = _setup(bie, p)
    s = density(p, nvec=nvec)
    y = _gpu_apply(bie, g, s, nvec)
    ref = og.apply(s)
    for v in range(nvec):
        assert _relerr(y[v], ref[v]) <= TOL, v


@pytest.mark.parametrize("cid", [3, 4])
def test_matvec_sampled_rows_parity(bie, cid):
    p = make_problem(cid)
    g, og = _setup(bie, p)
    s = density(p, nvec=1)
    y = _gpu_apply(bie, g, s, 1).reshape(-1, 2)
    rows = _rows(p.N)
    ref = og.apply(s, rows=rows).reshape(-1, 2)
    assert np.abs(y[rows] - ref).max() / np.abs(ref).max() <= TOL


def test_matvec_config5_sampled_rows(bie):
    """Config 5 (N = 1.06M): 256 strided rows x all sources vs the oracle."""
    p = make_problem(5)
    g, og = _setup(bie, p)
    s = density(p, nvec=1)
    y = _gpu_apply(bie, g, s, 1).reshape(-1, 2)
    rows = _rows(p.N, 256)
    ref = og.apply(s, rows=rows).reshape(-1, 2)
    assert np.abs(y[rows] - ref).max() / np.abs(ref).max() <= TOL


@pytest.mark.parametrize("cid,nvec", [(4, 16), (5, 4), (5, 16)])
def test_matvec_multivector_sampled_rows_large(bie, cid, nvec):
    """The bench's matvec sweeps (config 4 nvec 16; config 5 nvec 4/16, the
    one-sided multi-vector kernels at full size) on strided sampled rows."""
    p = make_problem(cid)
    g, og = _setup(bie, p)
    s = density(p, nvec=nvec, vec_id=40)
    y = _gpu_apply(bie, g, s, nvec)
    rows = _rows(p.N, 128)
    ref = og.apply(s, rows=rows)
    for v in range(nvec):
        yv = y[v].reshape(-1, 2)[rows]
        rv = ref[v].reshape(-1, 2)
        assert np.abs(yv - rv).max() / np.abs(rv).max() <= TOL


def test_gauss_identity_on_gpu(bie):
    """Property at any size (V1): D_ONLY of a constant density = -1/2 e.
    Config 4 tolerance: the trapezoid near-field error at its closest pore
    pair (gap 0.02, r ~ 0.03) is 8.7e-9 in the oracle itself (C18,
    tests/test_oracle_pins.py::test_V1_gauss_config4_worst_rows)."""
    for cid, tol in ((2, 1e-12), (4, 2e-8)):
        p = make_problem(cid)
        g, _ = _setup(bie, p)
        e = np.tile([0.3, -0.7], p.N)[None, :]
        y = _gpu_apply(bie, g, e, 1, flags=1)
        assert np.abs(y[0] + 0.5 * e[0]).max() < tol


@pytest.mark.parametrize("shape", ["nopores", "ragged", "circle_multi"])
def test_matvec_edge_geometries(bie, shape):
    if shape == "nopores":
        p = make_pipe(0, 10.0, 256, 0, (0.1, 0.2), 0.05, 16)
    elif shape == "ragged":
        p = make_pipe(31, 6.0, 262, 7, (0.1, 0.3), 0.05, 18)
    else:
        p = make_circle_problem(96, 1.0, ((0.3, 0.2, 0.2), (-0.4, -0.1, 0.25), (0.0, -0.6, 0.1)), 34,
                                config_id=41, name="circle_multi")
    g, og = _setup(bie, p)
    s = density(p, nvec=3)
    y = _gpu_apply(bie, g, s, 3)
    ref = og.apply(s)
    for v in range(3):
        assert _relerr(y[v], ref[v]) <= TOL


def test_rows_variant_matches_full(bie):
    import torch

    p = make_problem(2)
    g, og = _setup(bie, p)
    s = density(p, nvec=2)
    sig = torch.from_numpy(s.reshape(-1).copy()).cuda()
    full = torch.zeros_like(sig)
    bie.dlp_apply(g, sig, full, 2)
    rb, re_ = 333, 1501
    part = torch.zeros(2 * 2 * (re_ - rb), dtype=torch.float64, device="cuda")
    bie.dlp_apply_rows(g, sig, part, rb, re_, 2)
    torch.cuda.synchronize()
    f = full.cpu().numpy().reshape(2, -1, 2)[:, rb:re_]
    q = part.cpu().numpy().reshape(2, -1, 2)
    assert np.abs(f - q).max() <= 1e-14 * np.abs(f).max()


def test_host_variant_matches_device(bie):
    p = make_problem(2)
    g, og = _setup(bie, p)
    s = density(p, nvec=1)
    out = np.zeros_like(s)
    bie.dlp_apply_host(g, np.ascontiguousarray(s), out, 1)
    assert _relerr(out[0], og.apply(s)[0]) <= TOL


def test_deterministic_repeat(bie):
    p = make_problem(3)
    g, _ = _setup(bie, p)
    s = density(p, nvec=1)
    a = _gpu_apply(bie, g, s, 1)
    b = _gpu_apply(bie, g, s, 1)
    assert np.array_equal(a, b)


def test_apply_errors(bie):
    import torch

    p = make_problem(1)
    g, _ = _setup(bie, p)
    x = torch.zeros(2 * p.N, dtype=torch.float64, device="cuda")
    with pytest.raises(bie.BieError):
        bie.dlp_apply(g, x, x, 1)  # aliasing
    y = torch.zeros_like(x)
    with pytest.raises(bie.BieError):
        bie.dlp_apply(g, x, y, 1, flags=7)
    with pytest.raises(ValueError):
        bie.dlp_apply(g, x.float(), y, 1)


@pytest.mark.parametrize("cid", [1, 2, 3])
def test_symmetric_vs_one_sided(bie, cid):
    """The pair-reusing nvec=1 kernel and the one-sided kernel agree to rounding."""
    p = make_problem(cid)
    g, _ = _setup(bie, p)
    s = density(p, nvec=1, vec_id=4)
    a = _gpu_apply(bie, g, s, 1, 0)
    b = _gpu_apply(bie, g, s, 1, 2)  # BIE_ONE_SIDED
    assert _relerr(a[0], b[0]) <= 1e-13


def test_symmetric_ragged_sizes(bie):
    """Block/chunk edges: N not a multiple of 512 or 32, tiny N (no off-block units)."""
    for p in (make_pipe(31, 6.0, 262, 7, (0.1, 0.3), 0.05, 18),
              make_circle_problem(16, 1.0, (), 64, 50, "c16"),
              make_pipe(32, 12.0, 1000, 9, (0.1, 0.3), 0.05, 66)):
        g, og = _setup(bie, p)
        s = density(p, nvec=1)
        y = _gpu_apply(bie, g, s, 1)
        assert _relerr(y[0], og.apply(s)[0]) <= TOL, p.name


def test_d_only_symmetric_path_large(bie):
    """BIE_D_ONLY at nvec = 1 takes the symmetric kernel: sampled rows of config 4."""
    p = make_problem(4)
    g, og = _setup(bie, p)
    s = density(p, nvec=1, vec_id=2)
    y = _gpu_apply(bie, g, s, 1, flags=1).reshape(-1, 2)
    rows = _rows(p.N, 512)
    ref = og.apply(s, flags=1, rows=rows).reshape(-1, 2)
    assert np.abs(y[rows] - ref).max() / np.abs(ref).max() <= TOL


def test_side_stream_and_profile_hooks(bie):
    """Async on a caller stream; profiling hooks and the launch counter."""
    import torch

    p = make_problem(2)
    g, og = _setup(bie, p)
    s = density(p, nvec=1)
    sig = torch.from_numpy(s.reshape(-1).copy()).cuda()
    out = torch.zeros_like(sig)
    st = torch.cuda.Stream()
    n0 = bie.launch_count()
    bie.profile_begin(g)
    with torch.cuda.stream(st):
        for _ in range(3):
            bie.dlp_apply(g, sig, out, 1, stream=st)
    st.synchronize()
    pr = bie.profile_end(g)
    assert pr["applies"] == 3 and pr["pairs_ms"] > 0 and pr["epilogue_ms"] > 0
    assert bie.launch_count() - n0 >= 3 * 4  # moments, quad, sym, diag, epilogue per apply
    assert _relerr(out.cpu().numpy(), og.apply(s)[0]) <= TOL


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_node_table_bit_exact(bie, cid):
    """A1 parity (reading C27): the device node table equals the oracle's bit
    for bit -- positions, normals, tangents, weights and curvature are one
    fixed sequence of IEEE operations on the same inputs on both sides."""
    p = make_problem(cid)
    g = bie.Geometry.from_problem(p)
    og = oracle.OracleGeometry(p)
    t = g.node_table()
    g.close()
    assert np.array_equal(t["pos"], og.x)
    assert np.array_equal(t["nrm"], og.nrm)
    assert np.array_equal(t["tan"], og.tan)
    assert np.array_equal(t["w"], og.w)
    assert np.array_equal(t["kappa"], og.kn)


@pytest.mark.parametrize("cid", [3, 4])
def test_matvec_all_rows_parity(bie, cid):
    """Every row (not a sample) of the config-3/4 completed matvec at 1e-12."""
    p = make_problem(cid)
    g, og = _setup(bie, p)
    s = density(p, nvec=1, vec_id=70)
    y = _gpu_apply(bie, g, s, 1)
    ref = og.apply(s)
    assert _relerr(y[0], ref[0]) <= TOL


@pytest.mark.parametrize("cid", [2, 3])
def test_power_of_two_scaling_bitwise(bie, cid):
    """Degenerate magnitudes: the operator is linear and every step of the GPU
    path (pair sums in fixed-point limbs whose window follows max |Q|, the
    in-block sums, the completion terms) scales exactly by a power of two, so
    A(2^k sigma) = 2^k A(sigma) BITWISE for k = +-300 -- and A(0) = 0 exactly."""
    p = make_problem(cid)
    g, _ = _setup(bie, p)
    s = density(p, nvec=1)
    a = _gpu_apply(bie, g, s, 1)
    for k in (300, -300):
        b = _gpu_apply(bie, g, np.ldexp(s, k), 1)
        assert np.array_equal(np.ldexp(a, k), b), k
    z = _gpu_apply(bie, g, np.zeros_like(s), 1)
    assert np.array_equal(z, np.zeros_like(z))
