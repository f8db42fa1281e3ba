"""Matvec times at nvec 2 and 8 (one-sided variants), DLP and SLP, config on argv."""
import json, sys
import torch
sys.path.insert(0, '.')
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem, density
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
p = make_problem(cid); g = bie.Geometry.from_problem(p)
for op in ("dlp", "slp"):
    fn = bie.dlp_apply if op == "dlp" else bie.slp_apply
    for nvec in (2, 8):
        s = torch.from_numpy(density(p, nvec=nvec).reshape(-1)).cuda(); o = torch.zeros_like(s)
        for _ in range(2): fn(g, s, o, nvec, 0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3): fn(g, s, o, nvec, 0)
        e1.record(); torch.cuda.synchronize()
        print(json.dumps(dict(op=op, cfg=cid, nvec=nvec, ms=e0.elapsed_time(e1) / 3)), flush=True)
