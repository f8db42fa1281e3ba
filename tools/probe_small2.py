"""Matvec at small N: symmetric vs one-sided path."""
import json, sys, time
import torch
sys.path.insert(0, '.')
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem
from bie_inputs.geometry import make_pipe, CONFIGS
for cid in (1, 2, 3):
    p = make_problem(cid); g = bie.Geometry.from_problem(p)
    s = torch.randn(2 * p.N, dtype=torch.float64, device="cuda"); o = torch.zeros_like(s)
    res = {}
    for flags in (0, 2):
        for _ in range(3): bie.dlp_apply(g, s, o, 1, flags)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50): bie.dlp_apply(g, s, o, 1, flags)
        e1.record(); torch.cuda.synchronize()
        res[flags] = e0.elapsed_time(e1) / 50 * 1e3
    print(json.dumps(dict(cfg=cid, N=p.N, sym_us=res[0], onesided_us=res[2])), flush=True)
