"""BD factor (build PC) time at configs 2-4, delayed rank-128 update vs the
per-panel sweep (BIE_BD_AGG=0 in a second process), and B X = I residuals of
the wall inverse on sampled rows (backward error; the oracle's wall block)."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem

for cid in (2, 3, 4):
    p = make_problem(cid); g = bie.Geometry.from_problem(p)
    bd = bie.BlockDiag(g, structured=True); del bd
    ts = []
    for _ in range(3 if cid < 4 else 2):
        torch.cuda.synchronize(); t = time.perf_counter()
        bd = bie.BlockDiag(g, structured=True)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
    X = bd.block_inverse(p.M)
    print(json.dumps(dict(cfg=cid, noagg=os.environ.get("BIE_BD_AGG", "auto"), factor_s=min(ts),
                          wall_order=X.shape[0], inv_checksum=float(np.abs(X).sum()))), flush=True)
    np.save(f"/tmp/wallinv_c{cid}_{os.environ.get('BIE_BD_AGG', 'auto')}.npy", X[::97].copy())
