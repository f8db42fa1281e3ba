"""dist_gmres (GpuBackend, world 1) vs bie_gmres_solve on config 4, 50 iterations:
the Python driver's per-iteration overhead."""
import json, sys, time
import torch
sys.path.insert(0, '.')
import paper_1609_04484_b200 as bie
from paper_1609_04484_b200.dist import GpuBackend, dist_gmres
from bie_inputs import make_problem, rhs_pipe
p = make_problem(4); g = bie.Geometry.from_problem(p)
f = torch.from_numpy(rhs_pipe(p)).cuda(); x = torch.zeros_like(f)
bd = bie.BlockDiag(g, structured=True)
for mode in ("sym",):
    be = GpuBackend(g, 0, 1, mode=mode)
    for _ in range(2): dist_gmres(be, f, tol=1e-30, max_iter=50)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(3): dist_gmres(be, f, tol=1e-30, max_iter=50)
    torch.cuda.synchronize(); td = (time.perf_counter() - t) / 3
for _ in range(2): bie.gmres_solve(g, bd, f, x, tol=1e-30, max_iter=50)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(3): bie.gmres_solve(g, bd, f, x, tol=1e-30, max_iter=50)
torch.cuda.synchronize(); tc = (time.perf_counter() - t) / 3
print(json.dumps(dict(dist_ms=td * 1e3, native_ms=tc * 1e3)))
