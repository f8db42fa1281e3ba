"""Synthetic porous-pipe geometries (BASELINE.json configs[0..4]).

Citations are PAPER.md line numbers (P:l.N) and the readings (C-numbers) that
DESIGN.md lists.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy.special import ndtr  # standard normal CDF (Phi)

_INV_SQRT_2PI = 1.0 / math.sqrt(2.0 * math.pi)


def _phi(z):
    return _INV_SQRT_2PI * np.exp(-0.5 * z * z)


@dataclass
class Problem:
    """Raw geometry inputs, exactly what bie_geometry_create() takes.

    Dof order (P:l.734-736): pores 1..M first (each n_pore nodes, theta_j =
    2 pi j / n_pore from theta = 0, CCW; reading C12), then the outer wall
    Gamma_0 (n_outer nodes at t_j = j T / n_outer, CCW).
    """

    name: str
    outer_xy: np.ndarray  # (n_outer, 2) float64
    outer_dxy: np.ndarray  # (n_outer, 2) dx/dt
    outer_ddxy: np.ndarray  # (n_outer, 2) d2x/dt2
    period: float  # T
    pore_c: np.ndarray  # (M, 2)
    pore_r: np.ndarray  # (M,)
    n_pore: int
    config_id: int = 0
    meta: dict = field(default_factory=dict)

    @property
    def n_outer(self) -> int:
        return int(self.outer_xy.shape[0])

    @property
    def M(self) -> int:
        return int(self.pore_r.shape[0])

    @property
    def N(self) -> int:
        return self.M * self.n_pore + self.n_outer


def circle_outer(n: int, radius: float = 1.0, center=(0.0, 0.0)):
    """Circle samples at t_j = 2 pi j / n, CCW (config 1 outer curve)."""
    t = 2.0 * np.pi * np.arange(n) / n
    c, s = np.cos(t), np.sin(t)
    xy = np.stack([center[0] + radius * c, center[1] + radius * s], axis=1)
    dxy = np.stack([-radius * s, radius * c], axis=1)
    ddxy = np.stack([-radius * c, -radius * s], axis=1)
    return xy, dxy, ddxy, 2.0 * np.pi


def mollified_rectangle(L: float, H: float, delta: float, n: int):
    """Gaussian-mollified rectangle [0,L]x[-H,H] (reading C8; P:l.191-195).

    Arclength-of-the-rectangle parameter s in [0, P), P = 2L + 4H, start at
    (L/2, -H) heading +x, CCW.  Each corner turns the tangent by a step
    smoothed with the normal CDF of width delta:
      x'(s)  = t0 + sum_c dt_c Phi(z_c),       z_c = (s - s_c)/delta
      x''(s) = sum_c dt_c phi(z_c)/delta
      x(s)   = (L/2,-H) + s t0 + sum_c dt_c delta [psi(z_c) - psi(z_c^0)],
               psi(z) = z Phi(z) + phi(z), z_c^0 = -s_c/delta.
    Samples at s_j = j P / n, period T = P.
    """
    P = 2.0 * L + 4.0 * H
    s_c = np.array([L / 2, L / 2 + 2 * H, 3 * L / 2 + 2 * H, 3 * L / 2 + 4 * H])
    tang = np.array([[1.0, 0.0], [0.0, 1.0], [-1.0, 0.0], [0.0, -1.0], [1.0, 0.0]])
    dt = tang[1:] - tang[:-1]  # (4,2)
    s = P * np.arange(n) / n
    z = (s[:, None] - s_c[None, :]) / delta  # (n,4)
    z0 = -s_c / delta
    Phi = ndtr(z)
    ph = _phi(z)
    psi = z * Phi + ph
    psi0 = z0 * ndtr(z0) + _phi(z0)
    t0 = tang[0]
    dxy = t0[None, :] + Phi @ dt
    ddxy = (ph / delta) @ dt
    xy = np.array([L / 2, -H])[None, :] + s[:, None] * t0[None, :] + (delta * (psi - psi0[None, :])) @ dt
    return xy, dxy, ddxy, P


def pack_pores(rng, M, r_lo, r_hi, gap, L, H, wall_gap, max_attempts=10**6):
    """Seeded rejection packing (reading C16).

    Per attempt draw r ~ U[r_lo, r_hi], then cx ~ U[H+r+g_w, L-H-r-g_w], then
    cy ~ U[-H+r+g_w, H-r-g_w]; accept when the gap to every accepted pore is
    >= gap.  Raises RuntimeError after max_attempts (SPEC S:l.88 cap).
    """
    cs = np.zeros((M, 2))
    rs = np.zeros(M)
    k = 0
    attempts = 0
    # coarse grid for neighbour lookup
    cell = 2 * r_hi + gap
    grid: dict = {}
    while k < M:
        attempts += 1
        if attempts > max_attempts:
            raise RuntimeError(f"pore packing failed after {max_attempts} attempts ({k}/{M} placed)")
        r = rng.uniform(r_lo, r_hi)
        cx = rng.uniform(H + r + wall_gap, L - H - r - wall_gap)
        cy = rng.uniform(-H + r + wall_gap, H - r - wall_gap)
        gx, gy = int(math.floor(cx / cell)), int(math.floor(cy / cell))
        ok = True
        for ix in (gx - 1, gx, gx + 1):
            for iy in (gy - 1, gy, gy + 1):
                for q in grid.get((ix, iy), ()):
                    d = math.hypot(cx - cs[q, 0], cy - cs[q, 1]) - r - rs[q]
                    if d < gap:
                        ok = False
                        break
                if not ok:
                    break
            if not ok:
                break
        if not ok:
            continue
        cs[k] = (cx, cy)
        rs[k] = r
        grid.setdefault((gx, gy), []).append(k)
        k += 1
    return cs, rs, attempts


# BASELINE.json configs[0..4]; H = 1 (reading C9), delta = 0.2 H (C8),
# min gaps for configs 3 and 5 per reading C19.
CONFIGS = {
    1: dict(kind="circle", n_outer=64, M=1, n_pore=64),
    2: dict(kind="pipe", L=10.0, n_outer=512, M=10, r=(0.1, 0.3), gap=0.05, n_pore=128),
    3: dict(kind="pipe", L=40.0, n_outer=2048, M=100, r=(0.05, 0.2), gap=0.05, n_pore=256),
    4: dict(kind="pipe", L=100.0, n_outer=8192, M=1000, r=(0.03, 0.12), gap=0.02, n_pore=128),
    5: dict(kind="pipe", L=200.0, n_outer=16384, M=4096, r=(0.02, 0.08), gap=0.02, n_pore=256),
}
H_DEFAULT = 1.0
DELTA_FRAC = 0.2


def make_pipe(config_id, L, n_outer, M, r, gap, n_pore, H=H_DEFAULT, seed=None):
    delta = DELTA_FRAC * H
    xy, dxy, ddxy, T = mollified_rectangle(L, H, delta, n_outer)
    h_wall = (2 * L + 4 * H) / n_outer
    g_w = max(gap, 4.0 * h_wall)
    rng = np.random.default_rng(config_id if seed is None else seed)
    if M > 0:
        cs, rs, attempts = pack_pores(rng, M, r[0], r[1], gap, L, H, g_w)
    else:
        cs, rs, attempts = np.zeros((0, 2)), np.zeros(0), 0
    return Problem(
        name=f"config{config_id}" if seed is None else f"pipe_L{L}_M{M}_seed{seed}",
        outer_xy=xy, outer_dxy=dxy, outer_ddxy=ddxy, period=T,
        pore_c=cs, pore_r=rs, n_pore=n_pore, config_id=config_id,
        meta=dict(L=L, H=H, delta=delta, gap=gap, wall_gap=g_w, attempts=attempts),
    )


def make_circle_problem(n_outer=64, R=1.0, pores=((0.0, 0.0, 0.3),), n_pore=64, config_id=1, name=None):
    xy, dxy, ddxy, T = circle_outer(n_outer, R)
    pc = np.array([[p[0], p[1]] for p in pores], dtype=np.float64).reshape(-1, 2)
    pr = np.array([p[2] for p in pores], dtype=np.float64)
    return Problem(
        name=name or f"circle{n_outer}_M{len(pores)}", outer_xy=xy, outer_dxy=dxy, outer_ddxy=ddxy,
        period=T, pore_c=pc, pore_r=pr, n_pore=n_pore, config_id=config_id, meta=dict(R=R),
    )


def make_problem(config_id: int) -> Problem:
    """BASELINE.json configs[config_id - 1] (config ids 1..5)."""
    c = CONFIGS[config_id]
    if c["kind"] == "circle":
        return make_circle_problem(c["n_outer"], 1.0, ((0.0, 0.0, 0.3),), c["n_pore"], 1, "config1")
    return make_pipe(config_id, c["L"], c["n_outer"], c["M"], c["r"], c["gap"], c["n_pore"])


def density(problem_or_N, config_id=None, vec_id=0, nvec=1):
    """Densities i.i.d. N(0,1), interleaved (sx, sy) per node (reading C17).

    Vector v of a batch uses default_rng([config_id, 2, vec_id + v]).
    Returns shape (nvec, 2N).
    """
    if isinstance(problem_or_N, Problem):
        N = problem_or_N.N
        cid = problem_or_N.config_id if config_id is None else config_id
    else:
        N = int(problem_or_N)
        cid = 0 if config_id is None else config_id
    out = np.empty((nvec, 2 * N))
    for v in range(nvec):
        out[v] = np.random.default_rng([cid, 2, vec_id + v]).standard_normal(2 * N)
    return out


def pore_node_positions(problem: Problem) -> np.ndarray:
    """Pore collocation points c_k + r_k (cos th_j, sin th_j), th_j = 2 pi j/n (C12)."""
    th = 2.0 * np.pi * np.arange(problem.n_pore) / problem.n_pore
    ring = np.stack([np.cos(th), np.sin(th)], axis=1)
    pts = problem.pore_c[:, None, :] + problem.pore_r[:, None, None] * ring[None, :, :]
    return pts.reshape(-1, 2)


def node_positions(problem: Problem) -> np.ndarray:
    """All collocation points in dof order (pores first, then Gamma_0)."""
    return np.concatenate([pore_node_positions(problem), problem.outer_xy], axis=0)


def interior_grid(problem: Problem, nx: int, ny: int):
    """Evaluation points for the error field eps(x) (P:l.752-757): a regular
    nx x ny grid over the pipe's bounding box, keeping only points inside the
    fluid domain that are RELIABLE for the trapezoid rule -- farther than
    sqrt(ds) from every boundary, ds the local node spacing of that boundary
    (P:l.355-358 footnote).  Pure sampling; returns (P, 2)."""
    L, H = problem.meta["L"], problem.meta["H"]
    xs = (np.arange(nx) + 0.5) * L / nx
    ys = -H + (np.arange(ny) + 0.5) * 2 * H / ny
    P = np.stack(np.meshgrid(xs, ys, indexing="ij"), axis=-1).reshape(-1, 2)
    keep = np.ones(P.shape[0], dtype=bool)
    if problem.M:
        ds_p = 2 * np.pi * problem.pore_r / problem.n_pore
        for k in range(problem.M):
            d = np.hypot(P[:, 0] - problem.pore_c[k, 0], P[:, 1] - problem.pore_c[k, 1]) - problem.pore_r[k]
            keep &= d > np.sqrt(ds_p[k])
    w = problem.outer_xy
    seg = np.roll(w, -1, axis=0) - w
    ds_w = np.hypot(seg[:, 0], seg[:, 1]).max()
    # inside Gamma_0 (the mollified rectangle lies within [0, L] x [-H, H]) and far from it
    from scipy.spatial import cKDTree

    dw, _ = cKDTree(w).query(P)
    keep &= dw > np.sqrt(ds_w) + ds_w
    keep &= (np.abs(P[:, 1]) < H) & (P[:, 0] > 0) & (P[:, 0] < L)
    return P[keep]
