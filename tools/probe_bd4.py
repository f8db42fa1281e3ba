"""BD factor (build PC) of one config (default 4), timed with CUDA-synchronised
wall clocks: used for the A/B runs of the wall factor's schedule
(BIE_BD_LOOKAHEAD, BIE_BD_AGGK, BIE_BD_AGG) and, with --once, as the ncu
target for its launch list.  Prints a checksum of the wall inverse so that runs
of different schedules can be compared (they are bitwise equal)."""
import hashlib, json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem

cid = int(next((a for a in sys.argv[1:] if a.isdigit()), 4))
once = "--once" in sys.argv
p = make_problem(cid)
g = bie.Geometry.from_problem(p)
ts = []
for _ in range(1 if once else 4):
    torch.cuda.synchronize(); t = time.perf_counter()
    bd = bie.BlockDiag(g, structured=True)
    torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
    if not once:
        del bd
if not once:
    bd = bie.BlockDiag(g, structured=True)
X = bd.block_inverse(p.M)
env = {k: os.environ[k] for k in ("BIE_BD_LOOKAHEAD", "BIE_BD_AGGK", "BIE_BD_AGG") if k in os.environ}
print(json.dumps(dict(cfg=cid, env=env, factor_s=[round(t, 4) for t in ts], wall_order=int(X.shape[0]),
                      sha=hashlib.sha256(X.tobytes()).hexdigest()[:16], finite=bool(np.isfinite(X).all()))), flush=True)
