"""BD-GMRES solve time, CUDA-graph loop vs host-driven loop (BIE_GMRES_GRAPH),
configs 1-3: iterations, ms per solve (median of 7), bitwise agreement of the
histories and solutions of the two forms."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem, rhs_pipe, rhs_rotation_outer

for cid in (1, 2, 3):
    p = make_problem(cid); g = bie.Geometry.from_problem(p); bd = bie.BlockDiag(g, structured=True)
    f = torch.from_numpy(rhs_pipe(p) if cid > 1 else rhs_rotation_outer(p)).cuda(); x = torch.zeros_like(f)
    out = dict(cfg=cid, N=p.N)
    sols = {}
    for mode in ("1", "0"):
        os.environ["BIE_GMRES_GRAPH"] = mode
        for _ in range(2): r = bie.gmres_solve(g, bd, f, x, tol=1e-8, max_iter=1000)
        ts = []
        for _ in range(7):
            torch.cuda.synchronize(); t = time.perf_counter()
            r = bie.gmres_solve(g, bd, f, x, tol=1e-8, max_iter=1000)
            torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
        sols[mode] = (np.asarray(r["hist"]).copy(), x.cpu().numpy().copy(), r["iters"])
        out["graph" if mode == "1" else "host"] = dict(iters=r["iters"], ms=float(np.median(ts)) * 1e3,
                                                      us_per_iter=float(np.median(ts)) * 1e6 / max(1, r["iters"]))
    out["bitwise_equal"] = bool(np.array_equal(sols["1"][0], sols["0"][0]) and np.array_equal(sols["1"][1], sols["0"][1]))
    print(json.dumps(out), flush=True)
