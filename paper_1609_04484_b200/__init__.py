"""B200-native hot path of arxiv 1609.04484 (2D Stokes BIE-GMRES in porous media).

Thin ctypes binding of the C ABI declared in include/bie.h and implemented by
paper_1609_04484_b200/lib/libbie.so (CUDA, sm_100a).  Argument marshalling
only: every step of the path runs in the library's kernels.  There is no CPU
fallback -- importing the binding on a machine without the built library, or
calling a compute entry point without a CUDA device, raises.
"""
from ._bie import (  # noqa: F401
    BIE_D_ONLY,
    BIE_FULL,
    BIE_MAX_NVEC,
    BieError,
    BlockDiag,
    Geometry,
    Krylov,
    blockdiag_apply,
    blockdiag_factor,
    dlp_apply,
    dlp_apply_host,
    dlp_apply_rows,
    dlp_epilogue_rows,
    dlp_pairs_partial,
    dlp_sym_info,
    field_eval,
    gmres_solve,
    gmres_solve_host,
    gmres_solve_batch,
    gmres_solve_batch_slp,
    gmres_solve_slp,
    kr_weights,
    launch_count,
    debug_check,
    pore_template,
    fp64_peak,
    profile_begin,
    profile_end,
    slp_apply,
    slp_apply_rows,
    slp_epilogue_rows,
    slp_field_eval,
    slp_pairs_partial,
    lib,
    lib_path,
    EXPORTED_SYMBOLS,
)
