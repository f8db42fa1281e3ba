"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Python (ctypes) front-end of oracle/bie_oracle.c, the plain-C definition of the
completed double-layer operator, the single-layer operator with Kapur-Rokhlin
corrections (NEXT-1), the block-diagonal preconditioner and GMRES (see that
file's header for citations and pins), plus kr_weights(), the Kapur-Rokhlin
correction weights computed here in 40-digit decimal arithmetic.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package.  It shares no code with paper_1609_04484_b200 and the
product path never imports it.
"""
from __future__ import annotations

import ctypes
import decimal
import os
import subprocess
from fractions import Fraction

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bie_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O3", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC", "-std=c11"]

D_ONLY = 1


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lquadmath", "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int)
        L.ora_nodes.restype = ctypes.c_int
        L.ora_nodes.argtypes = [dp, dp, dp, ctypes.c_int, ctypes.c_double, dp, dp, ctypes.c_int, ctypes.c_int,
                                dp, dp, dp, dp, dp]
        L.ora_pore_template.restype = None
        L.ora_pore_template.argtypes = [ctypes.c_int, dp]
        L.ora_apply.restype = None
        L.ora_apply.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp, dp, dp, dp, dp, dp,
                                dp, dp, ctypes.c_int, ctypes.c_uint, ip, ctypes.c_int]
        L.ora_field.restype = None
        L.ora_field.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp, dp, dp, dp, dp, dp,
                                ctypes.c_int, dp]
        L.ora_bd_block.restype = None
        L.ora_bd_block.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp, dp, dp, dp, dp, dp,
                                   ctypes.c_int, dp]
        L.ora_lu.restype = ctypes.c_int
        L.ora_lu.argtypes = [ctypes.c_int, dp, ip]
        L.ora_lu_inverse.restype = None
        L.ora_lu_inverse.argtypes = [ctypes.c_int, dp, ip, dp]
        L.ora_bd_factor.restype = ctypes.c_void_p
        L.ora_bd_factor.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp, dp, dp, dp, dp, dp, ip]
        L.ora_bd_apply.restype = None
        L.ora_bd_apply.argtypes = [ctypes.c_void_p, dp, dp]
        L.ora_bd_block_inverse.restype = ctypes.c_int
        L.ora_bd_block_inverse.argtypes = [ctypes.c_void_p, ctypes.c_int, dp]
        L.ora_bd_free.restype = None
        L.ora_bd_free.argtypes = [ctypes.c_void_p]
        L.ora_gmres_dense.restype = ctypes.c_int
        L.ora_gmres_dense.argtypes = [ctypes.c_int, dp, dp, dp, dp, ctypes.c_double, ctypes.c_int, dp, dp, dp, ip]
        L.ora_bdlu_factor.restype = ctypes.c_void_p
        L.ora_bdlu_factor.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp, dp, dp, dp, dp, dp, ip]
        L.ora_bdlu_apply.restype = None
        L.ora_bdlu_apply.argtypes = [ctypes.c_void_p, dp, dp]
        L.ora_bdlu_free.restype = None
        L.ora_bdlu_free.argtypes = [ctypes.c_void_p]
        L.ora_gmres_bdlu.restype = ctypes.c_int
        L.ora_gmres_bdlu.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp, dp, dp, dp, dp, dp,
                                     ctypes.c_void_p, dp, dp, ctypes.c_double, ctypes.c_int, dp, dp, dp, ip]
        L.ora_slp_apply.restype = None
        L.ora_slp_apply.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp, dp, dp, dp, ctypes.c_int, ip,
                                    ctypes.c_int]
        L.ora_slp_field.restype = None
        L.ora_slp_field.argtypes = [ctypes.c_int, dp, dp, dp, dp, ctypes.c_int, dp]
        L.ora_slp_block.restype = None
        L.ora_slp_block.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp, dp, ctypes.c_int, dp]
        L.ora_slp_bd_factor.restype = ctypes.c_void_p
        L.ora_slp_bd_factor.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp, dp, ip]
        L.ora_slp_bdlu_factor.restype = ctypes.c_void_p
        L.ora_slp_bdlu_factor.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp, dp, ip]
        L.ora_slp_gmres.restype = ctypes.c_int
        L.ora_slp_gmres.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp, dp, ctypes.c_void_p, ctypes.c_int,
                                    dp, dp, ctypes.c_double, ctypes.c_int, dp, dp, dp, ip]
        L.ora_gmres_set_perturbation.restype = None
        L.ora_gmres_set_perturbation.argtypes = [dp, ctypes.c_ulonglong]
        L.ora_cgs_dots.restype = None
        L.ora_cgs_dots.argtypes = [ctypes.c_int, ctypes.c_int, dp, dp, dp]
        L.ora_cgs_sub.restype = None
        L.ora_cgs_sub.argtypes = [ctypes.c_int, ctypes.c_int, dp, dp, dp]
        L.ora_gmres.restype = ctypes.c_int
        L.ora_gmres.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp, dp, dp, dp, dp, dp,
                                ctypes.c_void_p, dp, dp, ctypes.c_double, ctypes.c_int, dp, dp, dp, ip]
        _lib = L
    return _lib


def _d(a):
    if a is None:
        return ctypes.POINTER(ctypes.c_double)()
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _i(a):
    if a is None:
        return ctypes.POINTER(ctypes.c_int)()
    assert a.dtype == np.int32 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


def _c(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class OracleGeometry:
    """Node table (A1) of one problem, derived by the oracle from the raw inputs."""

    def __init__(self, problem):
        self.problem = problem
        p = problem
        self.N, self.M, self.n_pore = p.N, p.M, p.n_pore
        self.pc = _c(p.pore_c.reshape(-1)) if p.M else np.zeros(2)
        self.pr = _c(p.pore_r) if p.M else np.zeros(1)
        N = self.N
        self.x = np.zeros(2 * N)
        self.nrm = np.zeros(2 * N)
        self.w = np.zeros(N)
        self.tan = np.zeros(2 * N)
        self.kn = np.zeros(N)
        n = lib().ora_nodes(_d(_c(p.outer_xy.reshape(-1))), _d(_c(p.outer_dxy.reshape(-1))),
                            _d(_c(p.outer_ddxy.reshape(-1))), p.n_outer, float(p.period), _d(self.pc),
                            _d(self.pr), p.M, p.n_pore, _d(self.x), _d(self.nrm), _d(self.w), _d(self.tan),
                            _d(self.kn))
        assert n == N

    def _geo(self):
        return (self.N, self.M, self.n_pore, _d(self.x), _d(self.nrm), _d(self.w), _d(self.tan), _d(self.kn),
                _d(self.pc), _d(self.pr))

    def apply(self, sigma, flags: int = 0, rows=None):
        """out = A sigma (completed operator; D_ONLY -> PV sum + self term).

        sigma: (2N,) or (nvec, 2N).  rows: optional int array of target nodes
        -> output (nvec, 2*len(rows)) holding only those rows."""
        s = _c(sigma)
        squeeze = s.ndim == 1
        s = s.reshape(-1, 2 * self.N)
        nvec = s.shape[0]
        r = None if rows is None else np.ascontiguousarray(rows, dtype=np.int32)
        nr = self.N if r is None else r.shape[0]
        out = np.zeros((nvec, 2 * nr))
        lib().ora_apply(*self._geo(), _d(s), _d(out), nvec, flags, _i(r), 0 if r is None else nr)
        return out[0] if squeeze else out

    def field(self, sigma, targets):
        """Off-surface velocity u = D[sigma] + completion fields at targets (P,2)."""
        t = _c(targets).reshape(-1)
        out = np.zeros(t.shape[0])
        lib().ora_field(self.N, self.M, self.n_pore, _d(self.x), _d(self.nrm), _d(self.w), _d(self.pc),
                        _d(self.pr), _d(_c(sigma)), _d(t), t.shape[0] // 2, _d(out))
        return out.reshape(-1, 2)

    def bd_block(self, b: int):
        n = self.n_pore if b < self.M else self.N - self.M * self.n_pore
        B = np.zeros((2 * n, 2 * n))
        lib().ora_bd_block(*self._geo(), b, _d(B))
        return B

    def body_range(self, b: int):
        if b < self.M:
            return b * self.n_pore, (b + 1) * self.n_pore
        return self.M * self.n_pore, self.N

    # --- NEXT-1: single-layer operator with Kapur-Rokhlin corrections ---
    def _slp(self):
        if not hasattr(self, "_gam"):
            self._gam = kr_weights()
        return self.N, self.M, self.n_pore, _d(self.x), _d(self.w), _d(self._gam)

    def slp_apply(self, sigma, rows=None):
        """out = A_SLP sigma (P:l.310-330): sigma (2N,) or (nvec, 2N); optional target rows."""
        s = _c(sigma)
        squeeze = s.ndim == 1
        s = s.reshape(-1, 2 * self.N)
        r = None if rows is None else np.ascontiguousarray(rows, dtype=np.int32)
        nr = self.N if r is None else r.shape[0]
        out = np.zeros((s.shape[0], 2 * nr))
        lib().ora_slp_apply(*self._slp(), _d(s), _d(out), s.shape[0], _i(r), 0 if r is None else nr)
        return out[0] if squeeze else out

    def slp_field(self, sigma, targets):
        """Off-surface u(x) = sum_j w_j G(x, x_j) sigma_j (P:l.346-354) at targets (P, 2)."""
        t = _c(targets).reshape(-1)
        out = np.zeros(t.shape[0])
        lib().ora_slp_field(self.N, _d(self.x), _d(self.w), _d(_c(sigma)), _d(t), t.shape[0] // 2, _d(out))
        return out.reshape(-1, 2)

    def slp_block(self, b: int):
        lo, hi = self.body_range(b)
        B = np.zeros((2 * (hi - lo), 2 * (hi - lo)))
        lib().ora_slp_block(*self._slp(), b, _d(B))
        return B


class OracleBD:
    """Explicit per-body inverses (A6); apply is A7."""

    def __init__(self, geom: OracleGeometry):
        bad = ctypes.c_int(0)
        self.geom = geom
        self.h = lib().ora_bd_factor(*geom._geo(), ctypes.byref(bad))
        if not self.h:
            raise MemoryError("oracle BD allocation failed")
        if bad.value:
            lib().ora_bd_free(self.h)
            self.h = None
            raise np.linalg.LinAlgError(f"singular BD block for body {bad.value - 1}")

    def apply(self, v):
        v = _c(v)
        out = np.zeros_like(v)
        lib().ora_bd_apply(self.h, _d(v), _d(out))
        return out

    def block_inverse(self, b: int):
        lo, hi = self.geom.body_range(b)
        n2 = 2 * (hi - lo)
        out = np.zeros((n2, n2))
        assert lib().ora_bd_block_inverse(self.h, b, _d(out)) == 0
        return out

    def __del__(self):
        if getattr(self, "h", None):
            lib().ora_bd_free(self.h)
            self.h = None


class OracleBDLU:
    """The BD preconditioner in LU form (forward/back substitution per apply) --
    the same operator as OracleBD without forming explicit inverses."""

    def __init__(self, geom: OracleGeometry):
        bad = ctypes.c_int(0)
        self.geom = geom
        self.h = lib().ora_bdlu_factor(*geom._geo(), ctypes.byref(bad))
        if not self.h:
            raise MemoryError("oracle BD-LU allocation failed")
        if bad.value:
            lib().ora_bdlu_free(self.h)
            self.h = None
            raise np.linalg.LinAlgError(f"singular BD block for body {bad.value - 1}")

    def apply(self, v):
        v = _c(v)
        out = np.zeros_like(v)
        lib().ora_bdlu_apply(self.h, _d(v), _d(out))
        return out

    def __del__(self):
        if getattr(self, "h", None):
            lib().ora_bdlu_free(self.h)
            self.h = None


class OracleSLPBD(OracleBD):
    """Explicit per-body inverses of the SLP blocks (NEXT-1, P:l.651-657)."""

    def __init__(self, geom: OracleGeometry):
        bad = ctypes.c_int(0)
        self.geom = geom
        self.h = lib().ora_slp_bd_factor(*geom._slp(), ctypes.byref(bad))
        if not self.h:
            raise MemoryError("oracle SLP BD allocation failed")
        if bad.value:
            lib().ora_bd_free(self.h)
            self.h = None
            raise np.linalg.LinAlgError(f"singular SLP BD block for body {bad.value - 1}")


class OracleSLPBDLU(OracleBDLU):
    """The SLP BD preconditioner in LU form."""

    def __init__(self, geom: OracleGeometry):
        bad = ctypes.c_int(0)
        self.geom = geom
        self.h = lib().ora_slp_bdlu_factor(*geom._slp(), ctypes.byref(bad))
        if not self.h:
            raise MemoryError("oracle SLP BD-LU allocation failed")
        if bad.value:
            lib().ora_bdlu_free(self.h)
            self.h = None
            raise np.linalg.LinAlgError(f"singular SLP BD block for body {bad.value - 1}")


def slp_gmres(geom: OracleGeometry, f, pc=None, tol=1e-8, max_iter=1000):
    """Left-preconditioned GMRES on the SLP system (pc: None, OracleSLPBD or OracleSLPBDLU)."""
    kind = 0 if pc is None else 2 if isinstance(pc, OracleBDLU) else 1
    x = np.zeros(2 * geom.N)
    hist, rp, rt, conv = _gmres_out(max_iter)
    it = lib().ora_slp_gmres(*geom._slp(), None if pc is None else pc.h, kind, _d(_c(f)), _d(x), tol, max_iter,
                             _d(hist), ctypes.byref(rp), ctypes.byref(rt), ctypes.byref(conv))
    return dict(x=x, iters=it, hist=hist[: it + 1].copy(), res_pc=rp.value, res_true=rt.value,
                converged=bool(conv.value))


# ---------------------------------------------------------------------------
# Kapur-Rokhlin sixth-order correction weights (P:l.321-330; reading C24 of
# DESIGN.md).  The rule  h sum_{j != 0} f(jh) + h sum_{0<|k|<=6} gamma_|k| f(kh)
# for f = phi(x) log|x| + psi(x) (periodic, singular node excluded) is exact
# to O(h^7 log h) when, with Navot's generalised Euler-Maclaurin expansion of
# the punctured trapezoid sum,
#     I - T'_h = h phi(0)(log h - log 2 pi) + 2 sum_{l>=1} zeta'(-2l) h^{2l+1} phi^(2l)(0)/(2l)!,
#   2 sum_k gamma_k k^(2l)        = [l == 0]          l = 0, 1, 2   (smooth part psi)
#   2 sum_k gamma_k k^(2l) log k  = 2 zeta'(-2l)      l = 0, 1, 2   (log part phi)
# with zeta'(0) = -log(2 pi)/2 and zeta'(-2l) = (-1)^l (2l)! zeta(2l+1) / (2 (2 pi)^(2l)).
# Everything below is plain 40-digit decimal arithmetic (Euler-Maclaurin for
# zeta(3), zeta(5); Machin for pi; Gauss-Jordan for the 6 x 6 system).
# ---------------------------------------------------------------------------
_KR_DIGITS = 40


def _bernoulli(n):
    """B_0..B_n as Fractions (B_1 = -1/2) from sum_{k<m} C(m+1, k) B_k = -(m+1) B_m."""
    B = [Fraction(0)] * (n + 1)
    B[0] = Fraction(1)
    for m in range(1, n + 1):
        acc = Fraction(0)
        c = 1  # C(m+1, k)
        for k in range(m):
            acc += c * B[k]
            c = c * (m + 1 - k) // (k + 1)
        B[m] = -acc / (m + 1)
    return B


def _zeta(s, D):
    """zeta(s), integer s >= 2: sum_{n<Nz} n^-s + Euler-Maclaurin tail at Nz = 40."""
    Nz, K = 40, 12
    total = sum(D(1) / D(n) ** s for n in range(1, Nz))
    total += D(Nz) ** (1 - s) / (s - 1) + D(1) / (2 * D(Nz) ** s)
    B = _bernoulli(2 * K)
    rising = D(s)  # s (s+1) ... (s + 2k - 2)
    fact = D(2)    # (2k)!
    for k in range(1, K + 1):
        b = D(B[2 * k].numerator) / D(B[2 * k].denominator)
        total += b / fact * rising / D(Nz) ** (s + 2 * k - 1)
        rising *= D(s + 2 * k - 1) * D(s + 2 * k)
        fact *= D(2 * k + 1) * D(2 * k + 2)
    return total


def _atan_inv(n, D):
    """atan(1/n) by its Taylor series."""
    x = D(1) / D(n)
    x2 = x * x
    term, total, k = x, D(0), 0
    eps = D(10) ** (-(_KR_DIGITS + 5))
    while abs(term) > eps:
        total += term / (2 * k + 1) if k % 2 == 0 else -term / (2 * k + 1)
        term *= x2
        k += 1
    return total


def kr_weights(order: int = 6):
    """gamma_1..gamma_6 of the sixth-order Kapur-Rokhlin log correction (float64)."""
    assert order == 6
    with decimal.localcontext() as ctx:
        ctx.prec = _KR_DIGITS + 10
        D = decimal.Decimal
        pi = 16 * _atan_inv(5, D) - 4 * _atan_inv(239, D)
        two_pi = 2 * pi
        zeta_p = [-(two_pi.ln()) / 2,
                  -D(2) * _zeta(3, D) / (2 * two_pi ** 2),
                  D(24) * _zeta(5, D) / (2 * two_pi ** 4)]
        rows = []
        for l in range(3):
            rows.append([2 * D(k) ** (2 * l) for k in range(1, 7)] + [D(1) if l == 0 else D(0)])
        for l in range(3):
            rows.append([2 * D(k) ** (2 * l) * D(k).ln() for k in range(1, 7)] + [2 * zeta_p[l]])
        n = 6
        for c in range(n):  # Gauss-Jordan, partial pivoting
            p = max(range(c, n), key=lambda r: abs(rows[r][c]))
            rows[c], rows[p] = rows[p], rows[c]
            piv = rows[c][c]
            rows[c] = [v / piv for v in rows[c]]
            for r in range(n):
                if r != c and rows[r][c] != 0:
                    f = rows[r][c]
                    rows[r] = [a - f * b for a, b in zip(rows[r], rows[c])]
        return np.array([float(rows[k][n]) for k in range(n)])


def gmres_bdlu(geom: OracleGeometry, f, bdlu: OracleBDLU, tol=1e-8, max_iter=1000):
    x = np.zeros(2 * geom.N)
    hist, rp, rt, conv = _gmres_out(max_iter)
    it = lib().ora_gmres_bdlu(*geom._geo(), bdlu.h, _d(_c(f)), _d(x), tol, max_iter, _d(hist), ctypes.byref(rp),
                              ctypes.byref(rt), ctypes.byref(conv))
    return dict(x=x, iters=it, hist=hist[: it + 1].copy(), res_pc=rp.value, res_true=rt.value,
                converged=bool(conv.value))


PERTURB_KEYS = ("A", "P", "dot", "norm", "sub")


class perturbed:
    """Sensitivity runs for the GMRES parity envelope (reading C23):
    inside the block every primitive of the oracle's GMRES iteration gets
    seeded Gaussian noise at the given level (keys of PERTURB_KEYS: A v,
    P^-1 v, CGS inner products, norms, CGS subtractions -- see the C source).
    Test infrastructure only; outside the block the oracle is unperturbed."""

    def __init__(self, eps: dict, seed: int = 0):
        self.eps = np.array([float(eps.get(k, 0.0)) for k in PERTURB_KEYS])
        self.seed = int(seed)

    def __enter__(self):
        lib().ora_gmres_set_perturbation(_d(self.eps), self.seed)
        return self

    def __exit__(self, *exc):
        lib().ora_gmres_set_perturbation(_d(np.zeros(5)), 0)


def cgs_dots(V, w):
    """out[j] = V_j . w with the oracle GMRES's own sequential sums (V: [nv, n])."""
    V = _c(V)
    nv, n = V.shape
    out = np.zeros(nv)
    lib().ora_cgs_dots(n, nv, _d(V), _d(_c(w)), _d(out))
    return out


def cgs_sub(V, h, w):
    """w - V^T h with the oracle GMRES's own loop (returns a new array)."""
    V = _c(V)
    nv, n = V.shape
    w = _c(w).copy()
    lib().ora_cgs_sub(n, nv, _d(V), _d(_c(h)), _d(w))
    return w


def pore_template(n: int) -> np.ndarray:
    """(cos, sin)(2 pi j / n), j < n, correctly rounded (reading C27) -> [n, 2]."""
    out = np.zeros(2 * n)
    lib().ora_pore_template(n, _d(out))
    return out.reshape(n, 2)


def lu(A):
    A = _c(A).copy()
    n = A.shape[0]
    piv = np.zeros(n, dtype=np.int32)
    rc = lib().ora_lu(n, _d(A), _i(piv))
    return A, piv, rc


def lu_inverse(LU, piv):
    n = LU.shape[0]
    out = np.zeros((n, n))
    lib().ora_lu_inverse(n, _d(_c(LU)), _i(piv), _d(out))
    return out


def _gmres_out(max_iter):
    return np.zeros(max_iter + 1), ctypes.c_double(0), ctypes.c_double(0), ctypes.c_int(0)


def gmres_dense(A, f, Pinv=None, tol=1e-8, max_iter=100):
    A = _c(A)
    n = A.shape[0]
    x = np.zeros(n)
    hist, rp, rt, conv = _gmres_out(max_iter)
    it = lib().ora_gmres_dense(n, _d(A), _d(None if Pinv is None else _c(Pinv)), _d(_c(f)), _d(x), tol,
                               max_iter, _d(hist), ctypes.byref(rp), ctypes.byref(rt), ctypes.byref(conv))
    return dict(x=x, iters=it, hist=hist[: it + 1].copy(), res_pc=rp.value, res_true=rt.value,
                converged=bool(conv.value))


def gmres(geom: OracleGeometry, f, bd: OracleBD | None = None, tol=1e-8, max_iter=1000):
    x = np.zeros(2 * geom.N)
    hist, rp, rt, conv = _gmres_out(max_iter)
    it = lib().ora_gmres(*geom._geo(), None if bd is None else bd.h, _d(_c(f)), _d(x), tol, max_iter,
                         _d(hist), ctypes.byref(rp), ctypes.byref(rt), ctypes.byref(conv))
    return dict(x=x, iters=it, hist=hist[: it + 1].copy(), res_pc=rp.value, res_true=rt.value,
                converged=bool(conv.value))
