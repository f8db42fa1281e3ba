"""SLP matvec times (bie_slp_apply) at nvec 4 and 16, config 4."""
import json, sys
import torch
sys.path.insert(0, '.')
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem, density
p = make_problem(4); g = bie.Geometry.from_problem(p)
for nvec in (4, 16):
    s = torch.from_numpy(density(p, nvec=nvec).reshape(-1)).cuda(); o = torch.zeros_like(s)
    for _ in range(2): bie.slp_apply(g, s, o, nvec)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): bie.slp_apply(g, s, o, nvec)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(json.dumps(dict(op="slp", cfg=4, nvec=nvec, ms=round(ms, 3), gpairs=round(nvec * p.N * p.N / ms / 1e6, 1))), flush=True)
