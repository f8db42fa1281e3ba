"""Pins for the shared input generator (bie_inputs): closed forms of the
Gaussian-mollified wall (reading C8) and the packing invariants (C16)."""
import math

import numpy as np
import pytest

from bie_inputs import CONFIGS, density, make_problem, mollified_rectangle, node_positions
from bie_inputs.geometry import circle_outer, make_pipe


def _shoelace(xy, dxy, T):
    n = xy.shape[0]
    return 0.5 * np.sum(xy[:, 0] * dxy[:, 1] - xy[:, 1] * dxy[:, 0]) * T / n


@pytest.mark.parametrize("L,n", [(10.0, 512), (100.0, 8192)])
def test_mollified_area_closed_form(L, n):
    # Each mollified corner loses delta^2/2 of area: A = 2LH - 2 delta^2 (C8).
    H, d = 1.0, 0.2
    xy, dxy, ddxy, T = mollified_rectangle(L, H, d, n)
    assert abs(_shoelace(xy, dxy, T) - (2 * L * H - 2 * d * d)) < 1e-12 * L


def test_mollified_closure_and_derivatives():
    L, H, d, n = 10.0, 1.0, 0.2, 4096
    xy, dxy, ddxy, T = mollified_rectangle(L, H, d, n)
    h = T / n
    # closure: x(P) = x(0) -- evaluate one extra sample at s = P
    xy2, _, _, _ = mollified_rectangle(L, H, d, n)
    assert np.allclose(xy2[0], [L / 2, -H])
    # centred differences of x and x' reproduce x' and x'' (periodic wrap)
    fd1 = (np.roll(xy, -1, 0) - np.roll(xy, 1, 0)) / (2 * h)
    fd2 = (np.roll(dxy, -1, 0) - np.roll(dxy, 1, 0)) / (2 * h)
    assert np.abs(fd1 - dxy).max() < 2e-4  # O(h^2 x''')
    assert np.abs(fd2 - ddxy).max() < 2e-3
    # the wrap-around difference is a valid derivative too -> the curve closes
    assert np.linalg.norm(xy[0] - (xy[-1] + h * dxy[-1])) < 1e-3
    # stays inside |y| <= H, flat far from corners
    assert np.abs(xy[:, 1]).max() <= H + 1e-15
    mid = np.argmin(np.abs(xy[:, 0] - L / 2) + np.abs(xy[:, 1] - H))
    assert abs(xy[mid, 1] - H) < 1e-12


def test_mollified_perimeter_spectral():
    # SPEC S:l.83: trapezoid arclength converges spectrally.
    L, H, d = 10.0, 1.0, 0.2
    per = []
    for n in (256, 512, 1024):
        xy, dxy, _, T = mollified_rectangle(L, H, d, n)
        per.append(np.sum(np.linalg.norm(dxy, axis=1)) * T / n)
    assert abs(per[1] - per[2]) < 1e-12
    assert abs(per[0] - per[2]) < 1e-6
    assert per[2] < 2 * L + 4 * H  # smoothing shortens the rectangle


def test_circle_outer():
    xy, dxy, ddxy, T = circle_outer(64, 1.0)
    assert abs(_shoelace(xy, dxy, T) - math.pi) < 1e-14
    assert np.allclose(ddxy, -xy)


@pytest.mark.parametrize("cid", [2, 3, 4])
def test_packing_invariants(cid):
    p = make_problem(cid)
    c = CONFIGS[cid]
    assert p.M == c["M"] and p.N == c["M"] * c["n_pore"] + c["n_outer"]
    assert np.all(p.pore_r >= c["r"][0]) and np.all(p.pore_r <= c["r"][1])
    L, H, gw = p.meta["L"], p.meta["H"], p.meta["wall_gap"]
    assert gw >= c["gap"] and gw >= 4 * (2 * L + 4 * H) / c["n_outer"] - 1e-15
    # pore-pore gaps (brute force over all pairs)
    cc, rr = p.pore_c, p.pore_r
    if p.M <= 1000:
        dd = np.linalg.norm(cc[:, None, :] - cc[None, :, :], axis=2) - rr[:, None] - rr[None, :]
        np.fill_diagonal(dd, np.inf)
        assert dd.min() >= c["gap"]
    # pore-wall: inside the flat part of the pipe with the wall gap
    assert np.all(cc[:, 1] + rr <= H - gw + 1e-12) and np.all(cc[:, 1] - rr >= -H + gw - 1e-12)
    assert np.all(cc[:, 0] - rr >= H + gw - 1e-12) and np.all(cc[:, 0] + rr <= L - H - gw + 1e-12)


def test_packing_deterministic_and_known_attempts():
    # Attempt counts of the seeded rejection sampler (C16) are a fingerprint
    # of the draw order r, cx, cy.
    assert [make_problem(c).meta["attempts"] for c in (2, 3, 4)] == [15, 141, 1440]
    a, b = make_problem(2), make_problem(2)
    assert np.array_equal(a.pore_c, b.pore_c)


def test_packing_failure_raises():
    with pytest.raises(RuntimeError):
        make_pipe(9, 4.0, 256, 50, (0.3, 0.4), 0.05, 16)


def test_density_seeded():
    p = make_problem(2)
    d1 = density(p, nvec=2)
    d2 = density(p, vec_id=1)
    assert d1.shape == (2, 2 * p.N)
    assert np.array_equal(d1[1], d2[0])
    assert abs(d1.mean()) < 0.05 and abs(d1.std() - 1) < 0.05


def test_node_positions_order():
    p = make_problem(2)
    pts = node_positions(p)
    assert pts.shape == (p.N, 2)
    k = 4
    ring = pts[k * p.n_pore:(k + 1) * p.n_pore]
    assert np.allclose(np.linalg.norm(ring - p.pore_c[k], axis=1), p.pore_r[k])
    assert np.allclose(ring[0], p.pore_c[k] + [p.pore_r[k], 0.0])
    assert np.array_equal(pts[p.M * p.n_pore:], p.outer_xy)
