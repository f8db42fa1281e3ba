"""Batched multi-RHS GMRES (config 3, 16 RHS) vs 16 single solves."""
import json, sys, time
import torch
sys.path.insert(0, '.')
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem, density
p = make_problem(3); g = bie.Geometry.from_problem(p); bd = bie.BlockDiag(g, structured=True)
F = torch.from_numpy(density(p, nvec=16, vec_id=100).reshape(-1)).cuda(); X = torch.zeros_like(F)
bie.gmres_solve_batch(g, bd, F, X, nrhs=16, tol=1e-8, max_iter=1000)
torch.cuda.synchronize(); t = time.perf_counter()
rb = bie.gmres_solve_batch(g, bd, F, X, nrhs=16, tol=1e-8, max_iter=1000)
torch.cuda.synchronize(); tb = time.perf_counter() - t
n2 = 2 * p.N; t = time.perf_counter(); its = []
for r in range(16):
    rr = bie.gmres_solve(g, bd, F[r * n2:(r + 1) * n2], X[r * n2:(r + 1) * n2], tol=1e-8, max_iter=1000); its.append(rr['iters'])
torch.cuda.synchronize(); ts = time.perf_counter() - t
print(json.dumps(dict(batched_s=tb, sequential_s=ts, iters_b=[r['iters'] for r in rb], iters_s=its)))
