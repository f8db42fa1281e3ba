"""Matvec times (bie_dlp_apply, BIE_FULL) for nvec 1 (one-sided and symmetric), 4, 16."""
import json, sys
import torch
sys.path.insert(0, '.')
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem, density
for cid in [int(c) for c in sys.argv[1:]] or [4]:
    p = make_problem(cid); g = bie.Geometry.from_problem(p)
    for nvec, flags in ((1, 0), (1, 2), (4, 0), (16, 0)):
        s = torch.from_numpy(density(p, nvec=nvec).reshape(-1)).cuda(); o = torch.zeros_like(s)
        for _ in range(2): bie.dlp_apply(g, s, o, nvec, flags)
        torch.cuda.synchronize()
        reps = 3 if cid < 5 else 1
        bie.profile_begin(g)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps): bie.dlp_apply(g, s, o, nvec, flags)
        e1.record(); torch.cuda.synchronize()
        pr = bie.profile_end(g)
        ms = e0.elapsed_time(e1) / reps
        print(json.dumps(dict(cfg=cid, nvec=nvec, flags=flags, ms=round(ms, 3), kernel_ms=round(pr['pairs_ms'] / reps, 3),
                              gpairs=round(nvec * p.N * p.N / ms / 1e6, 1))), flush=True)
        del s, o
