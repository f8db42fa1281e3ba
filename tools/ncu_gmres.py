"""Short command for ncu captures of the GMRES vector kernels and the BD apply
at config 4 (300 iterations, profiled range only)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem, rhs_pipe
p = make_problem(4)
g = bie.Geometry.from_problem(p)
bd = bie.BlockDiag(g)
f = torch.from_numpy(rhs_pipe(p)).cuda()
x = torch.zeros_like(f)
torch.cuda.synchronize()
torch.cuda.profiler.start()
r = bie.gmres_solve(g, bd, f, x, tol=1e-30, max_iter=int(sys.argv[1]) if len(sys.argv) > 1 else 300)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok", r["iters"])
