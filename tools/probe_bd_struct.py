"""BD factor and apply times: explicit per-body inverses vs structured pore blocks."""
import json, sys, time
import torch
sys.path.insert(0, '.')
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem, density
for cid in [int(c) for c in sys.argv[1:]] or [4]:
    p = make_problem(cid); g = bie.Geometry.from_problem(p)
    v = torch.from_numpy(density(p)[0]).cuda(); o = torch.zeros_like(v)
    for structured in (False, True, False, True):
        torch.cuda.synchronize(); t = time.time(); bd = bie.BlockDiag(g, structured=structured); torch.cuda.synchronize()
        tf = time.time() - t
        for _ in range(3): bie.blockdiag_apply(bd, v, o)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): bie.blockdiag_apply(bd, v, o)
        e1.record(); torch.cuda.synchronize()
        print(json.dumps(dict(cfg=cid, structured=structured, factor_s=tf, apply_ms=e0.elapsed_time(e1) / 20)), flush=True)
        del bd
