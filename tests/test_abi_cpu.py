"""C-ABI contract checks that need no GPU: the library loads, exports every
symbol include/bie.h declares, and argument validation fails loudly before
any device call."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bie():
    from paper_1609_04484_b200 import build as b

    b.build()
    import paper_1609_04484_b200 as pkg

    return pkg


def _declared():
    hdr = open(os.path.join(ROOT, "include", "bie.h")).read()
    return sorted(set(re.findall(r"BIE_API\s+(?:int|long long|const char \*)\s*(bie_\w+)\(", hdr)))


def test_header_declares_boundary():
    names = _declared()
    for n in ("bie_geometry_create", "bie_dlp_apply", "bie_blockdiag_factor", "bie_blockdiag_apply",
              "bie_gmres_solve", "bie_last_error"):
        assert n in names


def test_library_exports_every_declared_symbol(bie):
    L = bie.lib()
    for n in _declared():
        assert hasattr(L, n), n
    assert set(_declared()) == set(bie.EXPORTED_SYMBOLS)
    out = subprocess.run(["nm", "-D", "--defined-only", bie.lib_path()], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (bie_\w+)", out))
    assert exported == set(_declared())  # nothing else leaks


def test_sass_is_sm100a(bie):
    out = subprocess.run(["cuobjdump", "-lelf", bie.lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_invalid_arguments_fail_before_device(bie):
    L = bie.lib()
    h = ctypes.c_void_p()
    xy = np.zeros(2 * 32)
    dp = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))  # noqa: E731
    # odd / too small node counts (S:l.55-57)
    assert L.bie_geometry_create(dp(xy), dp(xy), dp(xy), 15, 1.0, None, None, 0, 0, ctypes.byref(h)) == -1
    assert b"even" in L.bie_last_error()
    assert L.bie_geometry_create(dp(xy), dp(xy), dp(xy), 32, 1.0, None, None, 1, 32, ctypes.byref(h)) == -1
    assert L.bie_geometry_create(None, dp(xy), dp(xy), 32, 1.0, None, None, 0, 0, ctypes.byref(h)) == -1
    # non-positive radius -> BIE_EGEOM
    c = np.zeros(2)
    r = np.array([-0.1])
    assert L.bie_geometry_create(dp(xy), dp(xy), dp(xy), 32, 1.0, dp(c), dp(r), 1, 32, ctypes.byref(h)) == -2
    # null handles -> BIE_EINVAL
    assert L.bie_dlp_apply(None, None, None, 1, 0, None) == -1
    assert L.bie_geometry_destroy(None) == -1
    assert L.bie_blockdiag_apply(None, None, None, 1, None) == -1
    assert L.bie_gmres_solve(None, None, None, None, 1e-8, 10, None, None, None, None, None, None) == -1


def test_binding_raises_without_library(tmp_path, monkeypatch):
    import paper_1609_04484_b200._bie as m

    monkeypatch.setattr(m, "_LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(m, "_lib", None)
    with pytest.raises(ImportError):
        m.lib()


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1609_04484_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", src).replace("no oracle", ""), f


def test_kr_weights_library_matches_oracle(bie):
    """bie_kr_weights needs no device: the library's long-double solve of the
    C24 conditions agrees with the oracle's 40-digit one to a few ulp."""
    import oracle

    assert np.abs(bie.kr_weights() - oracle.kr_weights()).max() <= 4 * np.spacing(26.0)


def test_krylov_entry_points_validate_arguments(bie):
    """bie_krylov_*: bad arguments return BIE_EINVAL before any device access
    (a host buffer stands in for the non-null pointers); n = 0 is a no-op."""
    L = bie._bie.lib()
    buf = np.zeros(64)
    p = buf.ctypes.data
    assert L.bie_krylov_dots(None, 8, 1, p, 8, p, None) == -1
    assert L.bie_krylov_dots(p, 8, 0, p, 8, p, None) == -1  # nv < 1
    assert L.bie_krylov_dots(p, 8, 1, p, -1, p, None) == -1  # n < 0
    assert L.bie_krylov_axpy(p, 8, 1, None, 1.0, 0.0, p, 8, None) == -1
    assert L.bie_krylov_axpy(p, 8, 1, p, 1.0, 0.0, p, 0, None) == 0  # empty: nothing launched
    assert L.bie_krylov_scale(p, None, p, 8, None) == -1
    assert L.bie_krylov_scale(p, p, p, 0, None) == 0
    assert L.bie_krylov_sqrt(p, p, 0, None) == -1
    assert L.bie_krylov_givens(p, 4, p, p, p, p, p, 3, p, None) == -1  # ldh < k + 2
    assert L.bie_krylov_givens(p, 8, p, p, p, p, None, 3, p, None) == -1
    assert L.bie_krylov_trisolve(p, 4, p, p, 5, None) == -1  # ldh < iters
    assert L.bie_krylov_trisolve(p, 4, p, p, 0, None) == 0
    assert b"krylov" in L.bie_last_error()


def test_slp_entry_points_validate_arguments(bie):
    L = bie._bie.lib()
    assert L.bie_slp_apply(None, None, None, 1, 0, None) == -1
    assert L.bie_slp_apply_rows(None, None, None, 1, 0, 1, None) == -1
    assert L.bie_slp_field_eval(None, None, None, 1, None, None) == -1
    assert L.bie_blockdiag_factor_slp(None, None, None) == -1
    assert L.bie_gmres_solve_slp(None, None, None, None, 1e-8, 10, None, None, None, None, None, None) == -1
    assert L.bie_kr_weights(None) == -1


def test_geometry_validation_rejects_bad_pores(bie):
    """Disjoint pores inside Gamma_0 (S:l.36) are checked on the host before any
    device work: overlapping, wall-crossing and outside pores -> BIE_EGEOM."""
    from bie_inputs.geometry import circle_outer

    L = bie.lib()
    h = ctypes.c_void_p()
    xy, dxy, ddxy, T = circle_outer(64, 1.0)
    dp = lambda a: np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(ctypes.POINTER(ctypes.c_double))  # noqa: E731
    keep = []

    def create(cs, rs):
        c = np.ascontiguousarray(np.array(cs, dtype=np.float64).reshape(-1))
        r = np.ascontiguousarray(np.array(rs, dtype=np.float64))
        a = [np.ascontiguousarray(x.reshape(-1)) for x in (xy, dxy, ddxy)]
        keep.append((a, c, r))
        return L.bie_geometry_create(dp(a[0]), dp(a[1]), dp(a[2]), 64, T, dp(c), dp(r), len(rs), 32,
                                     ctypes.byref(h))

    assert create([[0.0, 0.0], [0.25, 0.0]], [0.2, 0.1]) == -2
    assert b"overlap" in L.bie_last_error()
    assert create([[0.9, 0.0]], [0.2]) == -2
    assert b"crosses" in L.bie_last_error()
    assert create([[3.0, 0.0]], [0.1]) == -2
    assert b"outside" in L.bie_last_error()
    # a valid geometry passes validation (then needs a device: BIE_ECUDA on a CPU-only host)
    rc = create([[0.0, 0.0], [0.5, 0.0]], [0.2, 0.2])
    assert rc != -2 and rc != -1


@pytest.mark.parametrize("cid", [2, 3, 5])
def test_config_geometries_pass_validation(bie, cid):
    from bie_inputs import make_problem

    p = make_problem(cid)
    L = bie.lib()
    h = ctypes.c_void_p()
    arrs = [np.ascontiguousarray(a, dtype=np.float64).reshape(-1) for a in
            (p.outer_xy, p.outer_dxy, p.outer_ddxy, p.pore_c, p.pore_r)]
    dp = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))  # noqa: E731
    rc = L.bie_geometry_create(dp(arrs[0]), dp(arrs[1]), dp(arrs[2]), p.n_outer, float(p.period), dp(arrs[3]),
                               dp(arrs[4]), p.M, p.n_pore, ctypes.byref(h))
    if rc == 0:
        L.bie_geometry_destroy(h)
    assert rc not in (-1, -2), L.bie_last_error()


@pytest.mark.parametrize("n", [16, 18, 30, 64, 100, 128, 256, 1000, 4096])
def test_pore_template_correctly_rounded(bie, n):
    """Reading C27: the library's pore template (double-double Taylor series,
    host code, no device) and the oracle's (libquadmath) are independent
    implementations of one uniquely defined value -- cos/sin(2 pi j / n)
    correctly rounded -- so they must agree bit for bit.  Also pinned to the
    exact values at the octant points and to numpy within a few ulp."""
    import oracle

    u = bie.pore_template(n)
    assert np.array_equal(u, oracle.pore_template(n))
    th = 2 * np.pi * np.arange(n) / n
    assert np.abs(u - np.stack([np.cos(th), np.sin(th)], 1)).max() < 2e-15
    assert np.array_equal(u[0], [1.0, 0.0])
    if n % 4 == 0:
        assert np.array_equal(np.abs(u[n // 4]), [0.0, 1.0]) and np.array_equal(u[n // 2], [-1.0, 0.0])
    if n % 8 == 0:
        assert u[n // 8][0] == u[n // 8][1] == np.float64(np.sqrt(0.5))
