"""One BD-GMRES solve (graph loop) at config CID after warm-up, bracketed by
cudaProfilerStart/Stop for `ncu --profile-from-start off` launch lists."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem, rhs_pipe

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
it = int(sys.argv[2]) if len(sys.argv) > 2 else 3
p = make_problem(cid); g = bie.Geometry.from_problem(p); bd = bie.BlockDiag(g, structured=True)
f = torch.from_numpy(rhs_pipe(p)).cuda(); x = torch.zeros_like(f)
for _ in range(2): bie.gmres_solve(g, bd, f, x, tol=1e-30, max_iter=it)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
r = bie.gmres_solve(g, bd, f, x, tol=1e-30, max_iter=it)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("iters", r["iters"])
