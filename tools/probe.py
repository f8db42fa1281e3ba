"""Quick timing probe of the DLP matvec (not the bench contract)."""
import sys, time, json
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem, density

def time_apply(g, nvec, flags, reps=5):
    s = torch.from_numpy(density(g._p, nvec=nvec).reshape(-1)).cuda()
    o = torch.zeros_like(s)
    for _ in range(2):
        bie.dlp_apply(g, s, o, nvec, flags)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        bie.dlp_apply(g, s, o, nvec, flags)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3

for cid in [int(c) for c in sys.argv[1:]] or [3, 4]:
    p = make_problem(cid)
    g = bie.Geometry.from_problem(p); g._p = p
    for nvec in (1, 4, 16):
        for flags in ((1, 0, 2) if nvec == 1 else (1, 0)):
            t = time_apply(g, nvec, flags, reps=3 if cid == 5 else 5)
            pairs = p.N * p.N * nvec
            print(json.dumps(dict(cfg=cid, N=p.N, nvec=nvec, flags=flags, ms=t*1e3, gpairs_s=pairs/t/1e9,
                                  alg_tflops=(11+8*nvec)*p.N*p.N/t/1e12)), flush=True)

if len(sys.argv) > 1 and sys.argv[1] == 'bd':
    pass
