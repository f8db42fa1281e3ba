"""ctypes binding of libbie.so (names mirror include/bie.h)."""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# BIE_CHECKED=1 selects the checked build (allocation canaries, NaN-filled fresh
# memory, device bounds checks) -- a test configuration
_LIB_PATH = os.path.join(_HERE, "lib", "libbie_checked.so" if os.environ.get("BIE_CHECKED") == "1" else "libbie.so")

BIE_OK = 0
BIE_EINVAL = -1
BIE_EGEOM = -2
BIE_ESINGULAR = -3
BIE_ECUDA = -4
BIE_ENOMEM = -5
BIE_ECHECK = -6
BIE_FULL = 0
BIE_D_ONLY = 1
BIE_MAX_NVEC = 16

_CODES = {BIE_EINVAL: "BIE_EINVAL", BIE_EGEOM: "BIE_EGEOM", BIE_ESINGULAR: "BIE_ESINGULAR",
          BIE_ECUDA: "BIE_ECUDA", BIE_ENOMEM: "BIE_ENOMEM", BIE_ECHECK: "BIE_ECHECK"}

EXPORTED_SYMBOLS = (
    "bie_geometry_create", "bie_geometry_destroy", "bie_geometry_info", "bie_geometry_nodes",
    "bie_dlp_apply", "bie_dlp_apply_rows", "bie_dlp_apply_host",
    "bie_blockdiag_factor", "bie_blockdiag_apply", "bie_blockdiag_destroy", "bie_blockdiag_block_inverse",
    "bie_gmres_solve", "bie_last_error", "bie_profile_begin", "bie_profile_end", "bie_launch_count",
    "bie_field_eval", "bie_gmres_solve_batch", "bie_blockdiag_factor_range", "bie_blockdiag_rows",
    "bie_krylov_dots", "bie_krylov_axpy", "bie_krylov_scale", "bie_krylov_sqrt", "bie_krylov_givens",
    "bie_krylov_trisolve", "bie_dlp_sym_info", "bie_dlp_pairs_partial", "bie_dlp_epilogue_rows",
    "bie_kr_weights", "bie_slp_apply", "bie_slp_apply_rows", "bie_slp_field_eval", "bie_blockdiag_factor_slp",
    "bie_gmres_solve_slp", "bie_gmres_solve_batch_slp", "bie_blockdiag_factor_structured",
    "bie_blockdiag_factor_structured_slp",
    "bie_slp_pairs_partial", "bie_slp_epilogue_rows", "bie_blockdiag_factor_range_slp",
    "bie_geometry_node_table", "bie_pore_template", "bie_gmres_solve_host", "bie_fp64_peak",
    "bie_debug_check",
)


class BieError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_CODES.get(code, code)}: {msg}")
        self.code = code


_lib = None


def lib_path() -> str:
    return _LIB_PATH


def lib():
    """Load libbie.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"libbie.so not built: {_LIB_PATH} missing (run __graft_entry__.build())")
    L = ctypes.CDLL(_LIB_PATH)
    vp, dp, ip = ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)
    c_int, c_uint, c_double = ctypes.c_int, ctypes.c_uint, ctypes.c_double
    sig = {
        "bie_geometry_create": [dp, dp, dp, c_int, c_double, dp, dp, c_int, c_int, ctypes.POINTER(vp)],
        "bie_geometry_destroy": [vp],
        "bie_geometry_info": [vp, ip, ip],
        "bie_geometry_nodes": [vp, dp],
        "bie_geometry_node_table": [vp, dp, dp, dp, dp, dp],
        "bie_pore_template": [c_int, dp],
        "bie_dlp_apply": [vp, vp, vp, c_int, c_uint, vp],
        "bie_dlp_apply_rows": [vp, vp, vp, c_int, c_uint, c_int, c_int, vp],
        "bie_dlp_apply_host": [vp, dp, dp, c_int, c_uint, vp],
        "bie_blockdiag_factor": [vp, ctypes.POINTER(vp), vp],
        "bie_blockdiag_apply": [vp, vp, vp, c_int, vp],
        "bie_blockdiag_destroy": [vp],
        "bie_blockdiag_block_inverse": [vp, c_int, dp, ctypes.c_longlong],
        "bie_gmres_solve": [vp, vp, vp, vp, c_double, c_int, dp, ip, dp, dp, ip, vp],
        "bie_gmres_solve_host": [vp, vp, vp, vp, c_double, c_int, dp, ip, dp, dp, ip, vp],
        "bie_fp64_peak": [c_int, dp, dp, vp],
        "bie_debug_check": [ip, ip],
        "bie_field_eval": [vp, vp, vp, c_int, vp, vp],
        "bie_gmres_solve_batch": [vp, vp, vp, vp, c_int, c_double, c_int, dp, ip, dp, dp, ip, vp],
        "bie_blockdiag_factor_range": [vp, c_int, c_int, ctypes.POINTER(vp), vp],
        "bie_blockdiag_rows": [vp, ip, ip],
        "bie_krylov_dots": [vp, ctypes.c_longlong, c_int, vp, ctypes.c_longlong, vp, vp],
        "bie_krylov_axpy": [vp, ctypes.c_longlong, c_int, vp, c_double, c_double, vp, ctypes.c_longlong, vp],
        "bie_krylov_scale": [vp, vp, vp, ctypes.c_longlong, vp],
        "bie_krylov_sqrt": [vp, vp, c_int, vp],
        "bie_krylov_givens": [vp, c_int, vp, vp, vp, vp, vp, c_int, vp, vp],
        "bie_krylov_trisolve": [vp, c_int, vp, vp, c_int, vp],
        "bie_dlp_sym_info": [vp, ctypes.POINTER(ctypes.c_longlong), ip],
        "bie_dlp_pairs_partial": [vp, vp, vp, ctypes.c_longlong, ctypes.c_longlong, c_int, c_int, vp],
        "bie_dlp_epilogue_rows": [vp, vp, vp, vp, c_int, c_int, c_uint, vp],
        "bie_kr_weights": [dp],
        "bie_slp_apply": [vp, vp, vp, c_int, c_uint, vp],
        "bie_slp_apply_rows": [vp, vp, vp, c_int, c_int, c_int, vp],
        "bie_slp_field_eval": [vp, vp, vp, c_int, vp, vp],
        "bie_blockdiag_factor_slp": [vp, ctypes.POINTER(vp), vp],
        "bie_blockdiag_factor_structured": [vp, ctypes.POINTER(vp), vp],
        "bie_blockdiag_factor_structured_slp": [vp, ctypes.POINTER(vp), vp],
        "bie_slp_pairs_partial": [vp, vp, vp, ctypes.c_longlong, ctypes.c_longlong, c_int, c_int, vp],
        "bie_slp_epilogue_rows": [vp, vp, vp, vp, c_int, c_int, vp],
        "bie_blockdiag_factor_range_slp": [vp, c_int, c_int, ctypes.POINTER(vp), vp],
        "bie_gmres_solve_slp": [vp, vp, vp, vp, c_double, c_int, dp, ip, dp, dp, ip, vp],
        "bie_gmres_solve_batch_slp": [vp, vp, vp, vp, c_int, c_double, c_int, dp, ip, dp, dp, ip, vp],
        "bie_profile_begin": [vp],
        "bie_profile_end": [vp, dp, dp, dp, ip],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = c_int
    L.bie_last_error.argtypes = []
    L.bie_last_error.restype = ctypes.c_char_p
    L.bie_launch_count.argtypes = []
    L.bie_launch_count.restype = ctypes.c_longlong
    _lib = L
    return L


def _check(rc: int):
    if rc != BIE_OK:
        raise BieError(rc, lib().bie_last_error().decode(errors="replace"))


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _stream_ptr(stream):
    if stream is None:
        import torch

        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _dev_ptr(t, name, n_expected=None):
    import torch

    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor on a CUDA device")
    if not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous float64 CUDA tensor")
    if n_expected is not None and t.numel() < n_expected:
        raise ValueError(f"{name} has {t.numel()} elements, needs {n_expected}")
    return ctypes.c_void_p(t.data_ptr())


class Geometry:
    """bie_geometry_t: device node table + matvec workspace (A1)."""

    def __init__(self, outer_xy, outer_dxy, outer_ddxy, period, pore_c, pore_r, nodes_per_pore):
        L = lib()
        c = lambda a: np.ascontiguousarray(a, dtype=np.float64).reshape(-1)  # noqa: E731
        self._arrays = [c(outer_xy), c(outer_dxy), c(outer_ddxy), c(pore_c), c(pore_r)]
        n_outer = self._arrays[0].size // 2
        M = self._arrays[4].size
        h = ctypes.c_void_p()
        _check(L.bie_geometry_create(_dp(self._arrays[0]), _dp(self._arrays[1]), _dp(self._arrays[2]), n_outer,
                                     float(period), _dp(self._arrays[3]) if M else None,
                                     _dp(self._arrays[4]) if M else None, M, int(nodes_per_pore), ctypes.byref(h)))
        self.h = h
        N, Mo = ctypes.c_int(), ctypes.c_int()
        _check(L.bie_geometry_info(h, ctypes.byref(N), ctypes.byref(Mo)))
        self.N, self.M = N.value, Mo.value
        self.n_pore = int(nodes_per_pore) if M else 0

    @classmethod
    def from_problem(cls, p):
        """Duck-typed: any object with outer_xy/outer_dxy/outer_ddxy/period/pore_c/pore_r/n_pore."""
        return cls(p.outer_xy, p.outer_dxy, p.outer_ddxy, p.period, p.pore_c, p.pore_r, p.n_pore)

    def nodes(self) -> np.ndarray:
        out = np.zeros(2 * self.N)
        _check(lib().bie_geometry_nodes(self.h, _dp(out)))
        return out.reshape(-1, 2)

    def node_table(self) -> dict:
        """The device node table (A1) copied to host: pos, nrm, tan [N, 2], w, kappa [N]."""
        N = self.N
        t = {k: np.zeros(2 * N) for k in ("pos", "nrm", "tan")}
        t.update({k: np.zeros(N) for k in ("w", "kappa")})
        _check(lib().bie_geometry_node_table(self.h, _dp(t["pos"]), _dp(t["nrm"]), _dp(t["tan"]), _dp(t["w"]),
                                             _dp(t["kappa"])))
        return t

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            _check(lib().bie_geometry_destroy(self.h))
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fp64_peak(iters: int = 20000, stream=None) -> dict:
    """bie_fp64_peak: measured DFMA-chain FP64 rate of this device (TFLOP/s) and its duration."""
    tf, ms = ctypes.c_double(), ctypes.c_double()
    _check(lib().bie_fp64_peak(int(iters), ctypes.byref(tf), ctypes.byref(ms), _stream_ptr(stream)))
    return dict(tflops=tf.value, ms=ms.value)


def pore_template(n: int) -> np.ndarray:
    """(cos, sin)(2 pi j / n), correctly rounded (bie_pore_template, host only) -> [n, 2]."""
    out = np.zeros(2 * n)
    _check(lib().bie_pore_template(int(n), _dp(out)))
    return out.reshape(n, 2)


def debug_check() -> int:
    """bie_debug_check: verify allocation canaries and device bounds checks
    (checked build); returns the number of allocations verified, -1 in the
    normal build.  Raises BieError(BIE_ECHECK) on a violation."""
    n, line = ctypes.c_int(), ctypes.c_int()
    _check(lib().bie_debug_check(ctypes.byref(n), ctypes.byref(line)))
    return n.value


def launch_count() -> int:
    """Kernels launched by libbie.so in this process so far (bie_launch_count)."""
    return int(lib().bie_launch_count())


def profile_begin(g: Geometry):
    _check(lib().bie_profile_begin(g.h))


def profile_end(g: Geometry) -> dict:
    """Summed CUDA-event durations (ms) of the matvec phases since profile_begin."""
    m, p, e, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
    _check(lib().bie_profile_end(g.h, ctypes.byref(m), ctypes.byref(p), ctypes.byref(e), ctypes.byref(n)))
    return dict(moments_ms=m.value, pairs_ms=p.value, epilogue_ms=e.value, applies=n.value)


def dlp_apply(g: Geometry, sigma, out, nvec: int = 1, flags: int = BIE_FULL, stream=None):
    """out = A sigma on the device (bie_dlp_apply); sigma/out: float64 CUDA [nvec*2N]."""
    n = nvec * 2 * g.N
    _check(lib().bie_dlp_apply(g.h, _dev_ptr(sigma, "sigma", n), _dev_ptr(out, "out", n), nvec, flags,
                               _stream_ptr(stream)))
    return out


def dlp_sym_info(g: Geometry):
    """(units, blocks) of the symmetric all-pairs work list (bie_dlp_sym_info)."""
    u, b = ctypes.c_longlong(), ctypes.c_int()
    _check(lib().bie_dlp_sym_info(g.h, ctypes.byref(u), ctypes.byref(b)))
    return u.value, b.value


def dlp_pairs_partial(g: Geometry, sigma, out_full, units, blocks, stream=None):
    """Pair sums of a slice of the symmetric work into a full [2N] vector (bie_dlp_pairs_partial)."""
    _check(lib().bie_dlp_pairs_partial(g.h, _dev_ptr(sigma, "sigma", 2 * g.N), _dev_ptr(out_full, "out", 2 * g.N),
                                       int(units[0]), int(units[1]), int(blocks[0]), int(blocks[1]),
                                       _stream_ptr(stream)))
    return out_full


def dlp_epilogue_rows(g: Geometry, sigma, pairsum_rows, out_rows, row_begin: int, row_end: int,
                      flags: int = BIE_FULL, stream=None):
    """out_rows = pairsum_rows + local operator terms on [row_begin, row_end) (bie_dlp_epilogue_rows)."""
    n = 2 * (row_end - row_begin)
    _check(lib().bie_dlp_epilogue_rows(g.h, _dev_ptr(sigma, "sigma", 2 * g.N), _dev_ptr(pairsum_rows, "pairsum", n),
                                       _dev_ptr(out_rows, "out", n), row_begin, row_end, flags, _stream_ptr(stream)))
    return out_rows


def field_eval(g: Geometry, sigma, targets, out, stream=None):
    """Off-surface velocity u(x) at targets [P,2] from density sigma [2N] (bie_field_eval)."""
    ntgt = targets.numel() // 2
    _check(lib().bie_field_eval(g.h, _dev_ptr(sigma, "sigma", 2 * g.N), _dev_ptr(targets, "targets", 2 * ntgt),
                                ntgt, _dev_ptr(out, "out", 2 * ntgt), _stream_ptr(stream)))
    return out


def dlp_apply_rows(g: Geometry, sigma, out, row_begin: int, row_end: int, nvec: int = 1, flags: int = BIE_FULL,
                   stream=None):
    _check(lib().bie_dlp_apply_rows(g.h, _dev_ptr(sigma, "sigma", nvec * 2 * g.N),
                                    _dev_ptr(out, "out", nvec * 2 * (row_end - row_begin)), nvec, flags,
                                    row_begin, row_end, _stream_ptr(stream)))
    return out


def dlp_apply_host(g: Geometry, sigma_host: np.ndarray, out_host: np.ndarray, nvec: int = 1,
                   flags: int = BIE_FULL, stream=None):
    """End-to-end: host buffers in and out (bie_dlp_apply_host); synchronises."""
    assert sigma_host.dtype == np.float64 and out_host.dtype == np.float64
    assert sigma_host.size >= nvec * 2 * g.N and out_host.size >= nvec * 2 * g.N
    st = _stream_ptr(stream) if stream is not None else ctypes.c_void_p(0)
    _check(lib().bie_dlp_apply_host(g.h, _dp(sigma_host), _dp(out_host), nvec, flags, st))
    return out_host


def dlp_apply_host_ptr(g: Geometry, sigma_ptr: int, out_ptr: int, nvec: int = 1, flags: int = BIE_FULL,
                       stream=None):
    """Same as dlp_apply_host for raw (e.g. pinned torch) host pointers."""
    st = _stream_ptr(stream) if stream is not None else ctypes.c_void_p(0)
    dp = ctypes.POINTER(ctypes.c_double)
    _check(lib().bie_dlp_apply_host(g.h, ctypes.cast(sigma_ptr, dp), ctypes.cast(out_ptr, dp), nvec, flags, st))


class BlockDiag:
    """bie_blockdiag_t: explicit per-body inverses (A6).  bodies=(b0, b1) factors
    only that body range (row sharding); its apply takes local vectors.
    op="slp": blocks of the single-layer operator (bie_blockdiag_factor_slp).
    structured=True: DLP pore blocks from one reference inverse + rank-2
    Woodbury terms (bie_blockdiag_factor_structured); with op="slp", pore
    blocks as rotating-frame block-circulant inverses
    (bie_blockdiag_factor_structured_slp)."""

    def __init__(self, g: Geometry, stream=None, bodies=None, op: str = "dlp", structured: bool = False):
        h = ctypes.c_void_p()
        self.op = op
        if structured:
            if bodies is not None:
                raise ValueError("the structured pore BD is built for the whole geometry")
            fn = lib().bie_blockdiag_factor_structured_slp if op == "slp" else lib().bie_blockdiag_factor_structured
            _check(fn(g.h, ctypes.byref(h), _stream_ptr(stream)))
        elif op == "slp":
            if bodies is None:
                _check(lib().bie_blockdiag_factor_slp(g.h, ctypes.byref(h), _stream_ptr(stream)))
            else:
                _check(lib().bie_blockdiag_factor_range_slp(g.h, int(bodies[0]), int(bodies[1]), ctypes.byref(h),
                                                            _stream_ptr(stream)))
        elif bodies is None:
            _check(lib().bie_blockdiag_factor(g.h, ctypes.byref(h), _stream_ptr(stream)))
        else:
            _check(lib().bie_blockdiag_factor_range(g.h, int(bodies[0]), int(bodies[1]), ctypes.byref(h),
                                                    _stream_ptr(stream)))
        self.h = h
        self.g = g
        rb, re_ = ctypes.c_int(), ctypes.c_int()
        _check(lib().bie_blockdiag_rows(h, ctypes.byref(rb), ctypes.byref(re_)))
        self.rows = (rb.value, re_.value)

    def block_inverse(self, body: int) -> np.ndarray:
        g = self.g
        n = g.n_pore if body < g.M else g.N - g.M * g.n_pore
        out = np.zeros((2 * n, 2 * n))
        _check(lib().bie_blockdiag_block_inverse(self.h, body, _dp(out), out.size))
        return out

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            _check(lib().bie_blockdiag_destroy(self.h))
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def blockdiag_factor(g: Geometry, stream=None) -> BlockDiag:
    return BlockDiag(g, stream)


class Krylov:
    """Thin wrappers of the bie_krylov_* building blocks (device tensors)."""

    @staticmethod
    def dots(V, ldv: int, nv: int, w, n: int, out, stream=None):
        _check(lib().bie_krylov_dots(_dev_ptr(V, "V"), ldv, nv, _dev_ptr(w, "w"), n, _dev_ptr(out, "out", nv),
                                     _stream_ptr(stream)))

    @staticmethod
    def axpy(V, ldv: int, nv: int, c, alpha: float, beta: float, y, n: int, stream=None):
        _check(lib().bie_krylov_axpy(_dev_ptr(V, "V"), ldv, nv, _dev_ptr(c, "c"), float(alpha), float(beta),
                                     _dev_ptr(y, "y"), n, _stream_ptr(stream)))

    @staticmethod
    def scale(x, s, y, n: int, stream=None):
        _check(lib().bie_krylov_scale(_dev_ptr(x, "x"), _dev_ptr(s, "s"), _dev_ptr(y, "y"), n, _stream_ptr(stream)))

    @staticmethod
    def sqrt(inp, out, n: int, stream=None):
        _check(lib().bie_krylov_sqrt(_dev_ptr(inp, "in"), _dev_ptr(out, "out"), n, _stream_ptr(stream)))

    @staticmethod
    def givens(H, ldh: int, cs, sn, g, h, h2, k: int, scal, stream=None):
        _check(lib().bie_krylov_givens(_dev_ptr(H, "H"), ldh, _dev_ptr(cs, "cs"), _dev_ptr(sn, "sn"),
                                       _dev_ptr(g, "g"), _dev_ptr(h, "h"), _dev_ptr(h2, "h2"), k,
                                       _dev_ptr(scal, "scal"), _stream_ptr(stream)))

    @staticmethod
    def trisolve(H, ldh: int, g, y, iters: int, stream=None):
        _check(lib().bie_krylov_trisolve(_dev_ptr(H, "H"), ldh, _dev_ptr(g, "g"), _dev_ptr(y, "y"), iters,
                                         _stream_ptr(stream)))


def blockdiag_apply(bd: BlockDiag, inp, out, nvec: int = 1, stream=None):
    n = nvec * 2 * (bd.rows[1] - bd.rows[0])
    _check(lib().bie_blockdiag_apply(bd.h, _dev_ptr(inp, "in", n), _dev_ptr(out, "out", n), nvec,
                                     _stream_ptr(stream)))
    return out


def gmres_solve_batch(g: Geometry, bd: BlockDiag | None, F, X, nrhs: int, tol: float = 1e-8, max_iter: int = 1000,
                      stream=None):
    """bie_gmres_solve_batch: nrhs independent solves with batched operator applications.
    F, X: float64 CUDA [nrhs * 2N].  Returns a list of per-system dicts."""
    hist = np.zeros(nrhs * (max_iter + 1))
    it = np.zeros(nrhs, dtype=np.int32)
    conv = np.zeros(nrhs, dtype=np.int32)
    rp, rt = np.zeros(nrhs), np.zeros(nrhs)
    ip_ = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))  # noqa: E731
    n = nrhs * 2 * g.N
    _check(lib().bie_gmres_solve_batch(g.h, None if bd is None else bd.h, _dev_ptr(F, "F", n), _dev_ptr(X, "X", n),
                                       int(nrhs), float(tol), int(max_iter), _dp(hist), ip_(it), _dp(rp), _dp(rt),
                                       ip_(conv), _stream_ptr(stream)))
    hist = hist.reshape(nrhs, max_iter + 1)
    return [dict(iters=int(it[r]), hist=hist[r, : it[r] + 1].copy(), res_pc=float(rp[r]), res_true=float(rt[r]),
                 converged=bool(conv[r])) for r in range(nrhs)]


def gmres_solve(g: Geometry, bd: BlockDiag | None, f, x, tol: float = 1e-8, max_iter: int = 1000, stream=None):
    """bie_gmres_solve; returns dict(iters, hist, res_pc, res_true, converged)."""
    hist = np.zeros(max_iter + 1)
    it, conv = ctypes.c_int(0), ctypes.c_int(0)
    rp, rt = ctypes.c_double(0), ctypes.c_double(0)
    _check(lib().bie_gmres_solve(g.h, None if bd is None else bd.h, _dev_ptr(f, "f", 2 * g.N),
                                 _dev_ptr(x, "x", 2 * g.N), float(tol), int(max_iter), _dp(hist), ctypes.byref(it),
                                 ctypes.byref(rp), ctypes.byref(rt), ctypes.byref(conv), _stream_ptr(stream)))
    return dict(iters=it.value, hist=hist[: it.value + 1].copy(), res_pc=rp.value, res_true=rt.value,
                converged=bool(conv.value))


def _host_ptr(a, name, n):
    """Address of a host float64 buffer (numpy array or CPU torch tensor, pinned or not)."""
    if isinstance(a, np.ndarray):
        if a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"] or a.size < n:
            raise ValueError(f"{name} must be a contiguous float64 array with >= {n} elements")
        return ctypes.c_void_p(a.ctypes.data)
    import torch

    if not isinstance(a, torch.Tensor) or a.is_cuda or a.dtype != torch.float64 or not a.is_contiguous() \
            or a.numel() < n:
        raise ValueError(f"{name} must be a contiguous float64 host tensor with >= {n} elements")
    return ctypes.c_void_p(a.data_ptr())


def gmres_solve_host(g: Geometry, bd: BlockDiag | None, f_host, x_host, tol: float = 1e-8, max_iter: int = 1000,
                     stream=None):
    """bie_gmres_solve_host: f_host / x_host are HOST buffers [2N] (pinned for async DMA);
    H2D copy, solve and D2H copy inside the call, which returns after x_host is written."""
    hist = np.zeros(max_iter + 1)
    it, conv = ctypes.c_int(0), ctypes.c_int(0)
    rp, rt = ctypes.c_double(0), ctypes.c_double(0)
    _check(lib().bie_gmres_solve_host(g.h, None if bd is None else bd.h, _host_ptr(f_host, "f_host", 2 * g.N),
                                      _host_ptr(x_host, "x_host", 2 * g.N), float(tol), int(max_iter), _dp(hist),
                                      ctypes.byref(it), ctypes.byref(rp), ctypes.byref(rt), ctypes.byref(conv),
                                      _stream_ptr(stream)))
    return dict(iters=it.value, hist=hist[: it.value + 1].copy(), res_pc=rp.value, res_true=rt.value,
                converged=bool(conv.value))


# --- NEXT-1: single-layer operator with the Kapur-Rokhlin correction ---------
def kr_weights() -> np.ndarray:
    """gamma_1..gamma_6 as libbie.so computes them (bie_kr_weights)."""
    out = np.zeros(6)
    _check(lib().bie_kr_weights(_dp(out)))
    return out


def slp_apply(g: Geometry, sigma, out, nvec: int = 1, flags: int = 0, stream=None):
    """out = A_SLP sigma on the device (bie_slp_apply); flags 0 or BIE_ONE_SIDED (2)."""
    n = nvec * 2 * g.N
    _check(lib().bie_slp_apply(g.h, _dev_ptr(sigma, "sigma", n), _dev_ptr(out, "out", n), nvec, flags,
                               _stream_ptr(stream)))
    return out


def slp_apply_rows(g: Geometry, sigma, out, row_begin: int, row_end: int, nvec: int = 1, stream=None):
    _check(lib().bie_slp_apply_rows(g.h, _dev_ptr(sigma, "sigma", nvec * 2 * g.N),
                                    _dev_ptr(out, "out", nvec * 2 * (row_end - row_begin)), nvec, row_begin, row_end,
                                    _stream_ptr(stream)))
    return out


def slp_field_eval(g: Geometry, sigma, targets, out, stream=None):
    """Off-surface SLP velocity at targets [P,2] (bie_slp_field_eval)."""
    ntgt = targets.numel() // 2
    _check(lib().bie_slp_field_eval(g.h, _dev_ptr(sigma, "sigma", 2 * g.N), _dev_ptr(targets, "targets", 2 * ntgt),
                                    ntgt, _dev_ptr(out, "out", 2 * ntgt), _stream_ptr(stream)))
    return out


def gmres_solve_slp(g: Geometry, bd: BlockDiag | None, f, x, tol: float = 1e-8, max_iter: int = 1000, stream=None):
    """bie_gmres_solve_slp; bd from BlockDiag(g, op="slp") or None."""
    hist = np.zeros(max_iter + 1)
    it, conv = ctypes.c_int(0), ctypes.c_int(0)
    rp, rt = ctypes.c_double(0), ctypes.c_double(0)
    _check(lib().bie_gmres_solve_slp(g.h, None if bd is None else bd.h, _dev_ptr(f, "f", 2 * g.N),
                                     _dev_ptr(x, "x", 2 * g.N), float(tol), int(max_iter), _dp(hist),
                                     ctypes.byref(it), ctypes.byref(rp), ctypes.byref(rt), ctypes.byref(conv),
                                     _stream_ptr(stream)))
    return dict(iters=it.value, hist=hist[: it.value + 1].copy(), res_pc=rp.value, res_true=rt.value,
                converged=bool(conv.value))


def gmres_solve_batch_slp(g: Geometry, bd: BlockDiag | None, F, X, nrhs: int, tol: float = 1e-8,
                          max_iter: int = 1000, stream=None):
    hist = np.zeros(nrhs * (max_iter + 1))
    it = np.zeros(nrhs, dtype=np.int32)
    conv = np.zeros(nrhs, dtype=np.int32)
    rp, rt = np.zeros(nrhs), np.zeros(nrhs)
    ip_ = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))  # noqa: E731
    n = nrhs * 2 * g.N
    _check(lib().bie_gmres_solve_batch_slp(g.h, None if bd is None else bd.h, _dev_ptr(F, "F", n),
                                           _dev_ptr(X, "X", n), int(nrhs), float(tol), int(max_iter), _dp(hist),
                                           ip_(it), _dp(rp), _dp(rt), ip_(conv), _stream_ptr(stream)))
    hist = hist.reshape(nrhs, max_iter + 1)
    return [dict(iters=int(it[r]), hist=hist[r, : it[r] + 1].copy(), res_pc=float(rp[r]), res_true=float(rt[r]),
                 converged=bool(conv[r])) for r in range(nrhs)]


def slp_pairs_partial(g: Geometry, sigma, out_full, units, blocks, stream=None):
    """SLP pair sums of a slice of the symmetric work into a full [2N] vector (bie_slp_pairs_partial)."""
    _check(lib().bie_slp_pairs_partial(g.h, _dev_ptr(sigma, "sigma", 2 * g.N), _dev_ptr(out_full, "out", 2 * g.N),
                                       int(units[0]), int(units[1]), int(blocks[0]), int(blocks[1]),
                                       _stream_ptr(stream)))
    return out_full


def slp_epilogue_rows(g: Geometry, sigma, pairsum_rows, out_rows, row_begin: int, row_end: int, stream=None):
    """out_rows = pairsum_rows + KR corrections on [row_begin, row_end) (bie_slp_epilogue_rows)."""
    n = 2 * (row_end - row_begin)
    _check(lib().bie_slp_epilogue_rows(g.h, _dev_ptr(sigma, "sigma", 2 * g.N), _dev_ptr(pairsum_rows, "pairsum", n),
                                       _dev_ptr(out_rows, "out", n), row_begin, row_end, _stream_ptr(stream)))
    return out_rows

