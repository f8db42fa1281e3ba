"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NO arithmetic of the method (no layer-potential kernel, no
quadrature weights, no normals, no preconditioner, no Krylov step).  It only
produces the problem data both sides consume:

* samples of the outer wall curve Gamma_0 (x, x', x'' at equispaced parameter
  values) -- PAPER.md l.191-204 ("mollification of the rectangle [0,L]x[-H,H]"),
  reading C8 of DESIGN.md (Gaussian-mollified rectangle);
* pore centres / radii by seeded rejection sampling -- reading C16;
* density vectors i.i.d. N(0,1) -- reading C17;
* boundary data f: pipe flow (eq. noslip_bcs), shear
  (l.634-638), rigid rotation (reading C11), Stokeslet/rotlet combination
  (l.943-958, eq. analyticalBC).

The pore node positions c + r(cos th, sin th) are evaluated here only to
tabulate boundary data f at the collocation points; both the oracle and the
CUDA library derive their own node tables (normals, weights, curvature) from
the raw inputs.
"""
from .geometry import (  # noqa: F401
    CONFIGS,
    Problem,
    make_problem,
    circle_outer,
    mollified_rectangle,
    pack_pores,
    density,
    pore_node_positions,
    node_positions,
    interior_grid,
)
from .rhs import (  # noqa: F401
    rhs_pipe,
    rhs_rotation_outer,
    rhs_shear_outer,
    rhs_shear_all,
    stokeslet_rotlet_params,
    stokeslet_rotlet_field,
)
