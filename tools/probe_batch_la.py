"""Batched BD-GMRES (3 scenarios) vs 3 single graph-loop solves, configs 2 and 3."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem, rhs_pipe, rhs_shear_all, node_positions, stokeslet_rotlet_field, stokeslet_rotlet_params

for cid in (2, 3):
    p = make_problem(cid); g = bie.Geometry.from_problem(p); bd = bie.BlockDiag(g, structured=True)
    cs, lam, mu = stokeslet_rotlet_params(p)
    F = np.stack([rhs_pipe(p), rhs_shear_all(p), stokeslet_rotlet_field(node_positions(p), cs, lam, mu).reshape(-1)])
    Ft = torch.from_numpy(F.reshape(-1).copy()).cuda(); X = torch.zeros_like(Ft); n2 = 2 * p.N
    for _ in range(2):
        rb = bie.gmres_solve_batch(g, bd, Ft, X, nrhs=3, tol=1e-8, max_iter=1000)
        for r in range(3):
            bie.gmres_solve(g, bd, Ft[r * n2:(r + 1) * n2], X[r * n2:(r + 1) * n2], tol=1e-8, max_iter=1000)
    torch.cuda.synchronize(); t = time.perf_counter()
    rb = bie.gmres_solve_batch(g, bd, Ft, X, nrhs=3, tol=1e-8, max_iter=1000)
    torch.cuda.synchronize(); tb = time.perf_counter() - t
    t = time.perf_counter()
    rs = [bie.gmres_solve(g, bd, Ft[r * n2:(r + 1) * n2], X[r * n2:(r + 1) * n2], tol=1e-8, max_iter=1000) for r in range(3)]
    torch.cuda.synchronize(); ts = time.perf_counter() - t
    print(json.dumps(dict(cfg=cid, batched_ms=tb * 1e3, sequential_ms=ts * 1e3, iters_b=[r["iters"] for r in rb],
                          iters_s=[r["iters"] for r in rs])), flush=True)
