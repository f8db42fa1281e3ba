"""One small pass over every kernel family of libbie.so, for compute-sanitizer
(memcheck, racecheck, synccheck):

  python tools/sanitize_run.py            (configs 1-2 everywhere; config 3 for
                                           the cooperative BD panel of the wall)

DLP and SLP, symmetric and one-sided all-pairs kernels, nvec 1/2/4/16, D_ONLY,
field evaluation, explicit / structured / SLP BD factor and apply, GMRES
(device and host buffers), batched GMRES, the sharded slices
(bie_dlp_pairs_partial + bie_dlp_epilogue_rows, body-range BD) and the Krylov
primitives.  Prints one line per stage; any sanitizer error is reported by the
tool itself.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1609_04484_b200 as bie
from bie_inputs import density, make_problem, rhs_pipe, rhs_shear_all

BIE_ONE_SIDED = 2


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).reshape(-1)).cuda()


def stage(name):
    torch.cuda.synchronize()
    print("ok", name, flush=True)


def main():
    for cid in (1, 2):
        p = make_problem(cid)
        g = bie.Geometry.from_problem(p)
        n = 2 * p.N
        for nvec in (1, 2, 4, 16):
            s = t(density(p, nvec=nvec))
            o = torch.zeros_like(s)
            bie.dlp_apply(g, s, o, nvec)
            bie.slp_apply(g, s, o, nvec)
        s1 = t(density(p, nvec=1))
        o1 = torch.zeros_like(s1)
        for fl in (1, BIE_ONE_SIDED, 1 | BIE_ONE_SIDED):
            bie.dlp_apply(g, s1, o1, 1, fl)
        bie.slp_apply(g, s1, o1, 1, BIE_ONE_SIDED)
        stage(f"config {cid} matvecs")
        pts = t(np.array([[0.01, 0.02], [0.3, -0.4]]) if cid == 1 else np.array([[0.5, 0.0], [9.5, 0.5]]))
        fo = torch.zeros_like(pts)
        bie.field_eval(g, s1, pts, fo)
        bie.slp_field_eval(g, s1, pts, fo)
        stage(f"config {cid} fields")
        bds = {"explicit": bie.BlockDiag(g), "structured": bie.BlockDiag(g, structured=True)}
        bslp = bie.BlockDiag(g, op="slp")
        for b in list(bds.values()) + [bslp]:
            bie.blockdiag_apply(b, s1, o1)
        stage(f"config {cid} BD factor/apply")
        f = t(rhs_pipe(p))
        x = torch.zeros_like(f)
        for b in bds.values():
            bie.gmres_solve(b.g if hasattr(b, "g") else g, b, f, x, 1e-8, 200)
        bie.gmres_solve(g, None, f, x, 1e-8, 50)
        bie.gmres_solve_slp(g, bslp, f, x, 1e-8, 100)
        fh = f.cpu().pin_memory()
        xh = torch.zeros_like(fh).pin_memory()
        bie.gmres_solve_host(g, bds["structured"], fh, xh, 1e-8, 200)
        F = t(np.stack([rhs_pipe(p), rhs_shear_all(p), density(p, nvec=1)[0]]))
        X = torch.zeros_like(F)
        bie.gmres_solve_batch(g, bds["explicit"], F, X, 3, 1e-8, 200)
        stage(f"config {cid} GMRES (single, host, batched, SLP)")
        units, blocks = bie.dlp_sym_info(g)
        full = torch.zeros_like(s1)
        part = torch.zeros_like(s1)
        for (ub, ue), (b0, b1) in (((0, units // 2), (0, blocks // 2)), ((units // 2, units), (blocks // 2, blocks))):
            bie.dlp_pairs_partial(g, s1, part, (ub, ue), (b0, b1))
            full += part
        rows = torch.zeros_like(s1)
        bie.dlp_epilogue_rows(g, s1, full, rows, 0, p.N)
        bie.slp_pairs_partial(g, s1, part, (0, units), (0, blocks))
        bie.slp_epilogue_rows(g, s1, part, rows, 0, p.N)
        if p.M > 1:
            br = bie.BlockDiag(g, bodies=(0, p.M // 2))
            rb, re_ = br.rows
            bie.blockdiag_apply(br, s1[2 * rb:2 * re_].contiguous(), o1[2 * rb:2 * re_])
        stage(f"config {cid} sharded slices")
        V = t(density(p, nvec=8))
        h = torch.zeros(8, dtype=torch.float64, device="cuda")
        bie.Krylov.dots(V, n, 8, s1, n, h)
        bie.Krylov.axpy(V, n, 8, h, -1.0, 1.0, o1, n)
        stage(f"config {cid} Krylov primitives")
        g.close()
    p = make_problem(3)  # the wall block (4096 rows) takes the cooperative panel kernel
    g = bie.Geometry.from_problem(p)
    bd = bie.BlockDiag(g, structured=True)
    s = t(density(p, nvec=1))
    o = torch.zeros_like(s)
    bie.blockdiag_apply(bd, s, o)
    bie.dlp_apply(g, s, o, 1)
    stage("config 3 coop BD panel + matvec")


if __name__ == "__main__":
    main()
