"""Time the nvec=1 matvec paths (symmetric vs one-sided) at configs given on argv."""
import json, os, sys
import torch
sys.path.insert(0, '.')
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem, density
for cid in [int(c) for c in sys.argv[1:]] or [4]:
    p = make_problem(cid); g = bie.Geometry.from_problem(p)
    s = torch.from_numpy(density(p)[0]).cuda(); o = torch.zeros_like(s)
    for flags in (1, 0, 2):
        for _ in range(2): bie.dlp_apply(g, s, o, 1, flags)
        torch.cuda.synchronize()
        bie.profile_begin(g)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): bie.dlp_apply(g, s, o, 1, flags)
        e1.record(); torch.cuda.synchronize()
        pr = bie.profile_end(g)
        ms = e0.elapsed_time(e1) / 5
        print(json.dumps(dict(variant=os.environ.get('BIE_SYM_VARIANT', '0'), cfg=cid, flags=flags, ms=ms,
                              gpairs=p.N * p.N / ms / 1e6, pairs_ms=pr['pairs_ms'] / 5, epi_ms=pr['epilogue_ms'] / 5,
                              mom_ms=pr['moments_ms'] / 5)), flush=True)
