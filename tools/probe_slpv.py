"""Time SLP symmetric-kernel variants (BIE_SLP_SYM_VARIANT) at config 4 and check
them against the one-sided SLP path."""
import json, os, sys
import torch
sys.path.insert(0, '.')
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem, density
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
p = make_problem(cid); g = bie.Geometry.from_problem(p)
s = torch.from_numpy(density(p)[0]).cuda(); o = torch.zeros_like(s); r = torch.zeros_like(s)
bie.slp_apply(g, s, r, 1, 2)
for _ in range(2): bie.slp_apply(g, s, o, 1, 0)
torch.cuda.synchronize()
bie.profile_begin(g)
for _ in range(3): bie.slp_apply(g, s, o, 1, 0)
torch.cuda.synchronize()
pr = bie.profile_end(g)
err = ((o - r).abs().max() / r.abs().max()).item()
print(json.dumps(dict(slp_variant=os.environ.get('BIE_SLP_SYM_VARIANT', '0'), cfg=cid, pairs_ms=pr['pairs_ms'] / 3,
                      gpairs=p.N * p.N / (pr['pairs_ms'] / 3) / 1e6, err=err)), flush=True)
