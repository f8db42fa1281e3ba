"""Which phase grows in the slow bench steps?  Per step: device time, summed
all-pairs/epilogue phase times (bie_profile_*), and the k_dlp_sym CTA trace."""
import json, os, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem, rhs_pipe
p = make_problem(4); g = bie.Geometry.from_problem(p); bd = bie.BlockDiag(g, structured=True)
f = torch.from_numpy(rhs_pipe(p)).cuda(); x = torch.zeros_like(f)
for _ in range(3): bie.gmres_solve(g, bd, f, x, tol=1e-30, max_iter=50)
for k in range(14):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    bie.profile_begin(g)
    a.record(); bie.gmres_solve(g, bd, f, x, tol=1e-30, max_iter=50); b.record(); torch.cuda.synchronize()
    pr = bie.profile_end(g)
    print(json.dumps(dict(step_ms=round(a.elapsed_time(b), 1), pairs_ms=round(pr['pairs_ms'], 1),
                          epi_ms=round(pr['epilogue_ms'], 1), mom_ms=round(pr['moments_ms'], 1), n=pr['applies'])), flush=True)
