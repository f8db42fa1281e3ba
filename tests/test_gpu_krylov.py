"""GPU unit tests of the exported Krylov building blocks (bie_krylov_*; include/bie.h,
reading C13) against numpy in fp64: the kernels bie_gmres_solve uses, which a
row-sharded driver (paper_1609_04484_b200.dist) calls directly.  Sizes span several
4096-element dot chunks plus a ragged tail; nv spans the 4-vector CTA groups."""
import numpy as np
import pytest

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


@pytest.mark.parametrize("n", [100, 4096, 3 * 4096 + 77])
@pytest.mark.parametrize("nv", [1, 7, 17, 51])
def test_dots_and_axpy(bie, n, nv):
    import torch

    rng = np.random.default_rng(n * 100 + nv)
    ldv = n + 13  # a basis stored with padding between vectors
    V = rng.standard_normal((nv, ldv))
    w = rng.standard_normal(n)
    out = torch.zeros(nv, dtype=torch.float64, device="cuda")
    bie.Krylov.dots(_t(V), ldv, nv, _t(w), n, out)
    ref = V[:, :n] @ w
    # rounding bound of any summation order (Higham, gamma_n = n u / (1 - n u))
    scale = np.abs(V[:, :n]) @ np.abs(w)
    assert np.all(np.abs(out.cpu().numpy() - ref) <= n * 1.2e-16 * scale)

    c = rng.standard_normal(nv)
    y0 = rng.standard_normal(n)
    for alpha, beta in ((1.0, 0.0), (-1.0, 1.0), (0.5, -2.0)):
        y = _t(y0)
        bie.Krylov.axpy(_t(V), ldv, nv, _t(c), alpha, beta, y, n)
        ref = beta * y0 + alpha * (c @ V[:, :n])
        bound = abs(beta) * np.abs(y0) + abs(alpha) * (np.abs(c) @ np.abs(V[:, :n]))
        assert np.all(np.abs(y.cpu().numpy() - ref) <= (nv + 3) * 1.2e-16 * bound), (alpha, beta)


def test_scale_and_sqrt(bie):
    import torch

    rng = np.random.default_rng(5)
    n = 2 * 4096 + 3
    x = rng.standard_normal(n)
    s = np.array([3.7])
    y = torch.zeros(n, dtype=torch.float64, device="cuda")
    bie.Krylov.scale(_t(x), _t(s), y, n)
    assert np.array_equal(y.cpu().numpy(), x / 3.7)  # one correctly rounded division per element
    v = rng.random(9) * 10
    o = torch.zeros(9, dtype=torch.float64, device="cuda")
    bie.Krylov.sqrt(_t(v), o, 9)
    assert np.array_equal(o.cpu().numpy(), np.sqrt(v))


@pytest.mark.parametrize("K", [1, 5, 40])
def test_givens_trisolve_least_squares(bie, K):
    """K Givens steps on a random upper-Hessenberg matrix, then the triangular
    solve: y must be the least-squares solution of min ||beta e1 - Hbar y||
    (numpy lstsq) and scal[3] the relative residual -- quantities independent
    of the rotations' sign convention."""
    import torch

    rng = np.random.default_rng(K)
    ldh = K + 2
    Hbar = np.triu(rng.standard_normal((K + 1, K)), -1) + 3.0 * np.eye(K + 1, K)
    Hbar[np.arange(1, K + 1), np.arange(K)] = np.abs(Hbar[np.arange(1, K + 1), np.arange(K)])  # ||w|| >= 0
    beta = 2.5
    H = torch.zeros(ldh * (K + 1), dtype=torch.float64, device="cuda")
    cs = torch.zeros(K + 1, dtype=torch.float64, device="cuda")
    sn = torch.zeros_like(cs)
    g = torch.zeros(K + 2, dtype=torch.float64, device="cuda")
    g[0] = beta
    scal = torch.zeros(8, dtype=torch.float64, device="cuda")
    scal[0] = beta
    cols = np.zeros_like(Hbar)
    for k in range(K):
        h2 = 0.25 * rng.standard_normal(k + 1)
        h = Hbar[: k + 1, k] - h2
        cols[: k + 1, k] = h + h2  # the column the kernel forms
        cols[k + 1, k] = Hbar[k + 1, k]
        scal[1] = 1.0
        scal[2] = Hbar[k + 1, k]
        bie.Krylov.givens(H, ldh, cs, sn, g, _t(h), _t(h2), k, scal)
    y = torch.zeros(K, dtype=torch.float64, device="cuda")
    bie.Krylov.trisolve(H, ldh, g, y, K)
    rhs = np.zeros(K + 1)
    rhs[0] = beta
    ref, *_ = np.linalg.lstsq(cols, rhs, rcond=None)
    assert np.abs(y.cpu().numpy() - ref).max() <= 1e-12 * np.abs(ref).max()
    # relative residual from a Householder QR (evaluating ||rhs - cols y|| would
    # only see rounding noise when the residual is tiny)
    Q, _ = np.linalg.qr(cols, mode="complete")
    res = abs((Q.T @ rhs)[K]) / beta
    assert abs(scal[3].item() - res) <= 1e-10 * res, (scal[3].item(), res)
    assert scal[4].item() == 0.0  # no breakdown flagged (H[k+1,k] > 1e-14 scal[1])
    # a zero subdiagonal (the Krylov space is invariant) is flagged
    scal[2] = 0.0
    bie.Krylov.givens(H, ldh, cs, sn, g, _t(np.ones(K + 1)), _t(np.zeros(K + 1)), K, scal)
    assert scal[4].item() == 1.0 and scal[3].item() == 0.0
