"""Boundary data f at the collocation points (problem data, not the method).

Layout: (2N,) interleaved (fx, fy) per node in dof order (pores, then Gamma_0).
"""
from __future__ import annotations

import numpy as np

from .geometry import Problem, node_positions


def _pack(problem: Problem, f_pores: np.ndarray, f_outer: np.ndarray) -> np.ndarray:
    return np.concatenate([f_pores.reshape(-1, 2), f_outer.reshape(-1, 2)], axis=0).reshape(-1).copy()


def rhs_pipe(problem: Problem, k: float = 1.0, H: float | None = None) -> np.ndarray:
    """Pipe flow, P:l.217-227 (eq. noslip_bcs), reading C10:
    f = (k (H^2 - y^2), 0) on Gamma_0, f = 0 on every pore."""
    H = problem.meta.get("H", 1.0) if H is None else H
    y = problem.outer_xy[:, 1]
    fo = np.stack([k * (H * H - y * y), np.zeros_like(y)], axis=1)
    return _pack(problem, np.zeros((problem.M * problem.n_pore, 2)), fo)


def rhs_rotation_outer(problem: Problem) -> np.ndarray:
    """Tiny config (reading C11): rigid rotation f = (-y, x) on the outer curve, no-slip on pores."""
    x, y = problem.outer_xy[:, 0], problem.outer_xy[:, 1]
    return _pack(problem, np.zeros((problem.M * problem.n_pore, 2)), np.stack([-y, x], axis=1))


def rhs_shear_outer(problem: Problem) -> np.ndarray:
    """Shear (y, 0) on the outer curve only, no-slip on pores (C11 companion case)."""
    y = problem.outer_xy[:, 1]
    return _pack(problem, np.zeros((problem.M * problem.n_pore, 2)), np.stack([y, np.zeros_like(y)], axis=1))


def rhs_shear_all(problem: Problem) -> np.ndarray:
    """Shear flow on ALL boundaries, u_ref = (y, 0) (P:l.634-638)."""
    p = node_positions(problem)
    return np.stack([p[:, 1], np.zeros(p.shape[0])], axis=1).reshape(-1).copy()


def stokeslet_rotlet_params(problem: Problem, seed: int = 7, c0=None):
    """Singularity data for eq. analyticalBC (P:l.943-958): c_0 outside Omega_0,
    c_k inside pore k (its centre), lambda_k ~ N(0,1)^2, mu_k ~ N(0,1)."""
    rng = np.random.default_rng([problem.config_id, 13, seed])
    if c0 is None:
        if problem.meta.get("L") is not None:
            L, H = problem.meta["L"], problem.meta["H"]
            c0 = np.array([L / 2, 3.0 * H])
        else:
            c0 = np.array([0.0, 2.5 * problem.meta.get("R", 1.0)])
    cs = np.concatenate([np.asarray(c0, dtype=np.float64)[None, :], problem.pore_c], axis=0)
    lam = rng.standard_normal((cs.shape[0], 2))
    mu = rng.standard_normal(cs.shape[0])
    return cs, lam, mu


def stokeslet_rotlet_field(points: np.ndarray, cs: np.ndarray, lam: np.ndarray, mu: np.ndarray) -> np.ndarray:
    """Eq. analyticalBC (P:l.943-948), (x,y)^perp = (y,-x) (P:l.956):
    f(x) = sum_k (-log|x-c_k| I + (x-c_k)(x-c_k)^T/|x-c_k|^2) lam_k + (x-c_k)^perp/|x-c_k|^2 mu_k.
    Returns (P, 2)."""
    out = np.zeros((points.shape[0], 2))
    for k in range(cs.shape[0]):
        r = points - cs[k][None, :]
        rho2 = np.sum(r * r, axis=1)
        rl = r @ lam[k]
        out += -0.5 * np.log(rho2)[:, None] * lam[k][None, :] + (rl / rho2)[:, None] * r
        perp = np.stack([r[:, 1], -r[:, 0]], axis=1)
        out += (mu[k] / rho2)[:, None] * perp
    return out
