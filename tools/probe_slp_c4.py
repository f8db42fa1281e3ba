"""Full config-4 single-layer (NEXT-1) BD-GMRES solve to 1e-8 (iterations, time, history samples)."""
import json, sys, time
import torch
sys.path.insert(0, '.')
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem, rhs_pipe
p = make_problem(4); g = bie.Geometry.from_problem(p)
bd = bie.BlockDiag(g, op="slp"); torch.cuda.synchronize()
f = torch.from_numpy(rhs_pipe(p)).cuda(); x = torch.zeros_like(f)
t = time.time(); r = bie.gmres_solve_slp(g, bd, f, x, 1e-8, 2000); torch.cuda.synchronize(); tg = time.time() - t
h = r['hist']
print(json.dumps(dict(iters=r['iters'], conv=r['converged'], res_true=r['res_true'], res_pc=r['res_pc'], s=tg,
                      hist_at=[float(h[k]) for k in (0, 100, 200, 300, 500, 1000, 1500) if k < len(h)] + [float(h[-1])])))
