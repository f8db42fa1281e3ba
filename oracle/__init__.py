"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Python (ctypes) front-end of oracle/bie_oracle.c, the plain-C definition of the
completed double-layer operator, the block-diagonal preconditioner and GMRES
(see that file's header for citations and pins).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package.  It shares no code with paper_1609_04484_b200 and the
product path never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

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
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
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


def gmres_bdlu(geom: OracleGeometry, f, bdlu: OracleBDLU, tol=1e-8, max_iter=1000):
    x = np.zeros(2 * geom.N)
    hist, rp, rt, conv = _gmres_out(max_iter)
    it = lib().ora_gmres_bdlu(*geom._geo(), bdlu.h, _d(_c(f)), _d(x), tol, max_iter, _d(hist), ctypes.byref(rp),
                              ctypes.byref(rt), ctypes.byref(conv))
    return dict(x=x, iters=it, hist=hist[: it + 1].copy(), res_pc=rp.value, res_true=rt.value,
                converged=bool(conv.value))


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
