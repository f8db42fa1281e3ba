"""Structured (rotating-frame circulant) vs explicit SLP BD: factor time,
apply time, BD-GMRES iterations/time at configs 3-4 (and the factor + apply at
config 5, where explicit pore inverses would need 17 GB)."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem, rhs_pipe


def timed(fn, reps=1):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps): r = fn()
    torch.cuda.synchronize(); return r, (time.perf_counter() - t) / reps


for cid in (3, 4, 5):
    p = make_problem(cid); g = bie.Geometry.from_problem(p)
    out = dict(cfg=cid, N=p.N)
    kinds = (True,) if cid == 5 else (True, False)
    for st in kinds:
        bd, tf = timed(lambda: bie.BlockDiag(g, op="slp", structured=st))
        v = torch.randn(2 * p.N, dtype=torch.float64, device="cuda"); z = torch.zeros_like(v)
        bie.blockdiag_apply(bd, v, z)
        _, ta = timed(lambda: bie.blockdiag_apply(bd, v, z), 20)
        rec = dict(factor_s=tf, apply_ms=ta * 1e3)
        if cid < 5:
            f = torch.from_numpy(rhs_pipe(p)).cuda(); x = torch.zeros_like(f)
            r, ts = timed(lambda: bie.gmres_solve_slp(g, bd, f, x, 1e-8, 2000))
            rec.update(iters=r["iters"], gmres_s=ts, res_true=r["res_true"])
        out["structured" if st else "explicit"] = rec
        del bd
    print(json.dumps(out), flush=True)
