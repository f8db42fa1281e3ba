"""GMRES solve times for the small configs (launch-bound regime)."""
import json, sys, time
import torch
sys.path.insert(0, '.')
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem, rhs_pipe, rhs_rotation_outer
for cid in (1, 2, 3):
    p = make_problem(cid); g = bie.Geometry.from_problem(p); bd = bie.BlockDiag(g, structured=True)
    f = torch.from_numpy(rhs_pipe(p) if cid > 1 else rhs_rotation_outer(p)).cuda(); x = torch.zeros_like(f)
    for _ in range(3): r = bie.gmres_solve(g, bd, f, x, tol=1e-8, max_iter=1000)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(5): r = bie.gmres_solve(g, bd, f, x, tol=1e-8, max_iter=1000)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 5
    s = torch.randn(2 * p.N, dtype=torch.float64, device="cuda"); o = torch.zeros_like(s)
    for _ in range(3): bie.dlp_apply(g, s, o)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(50): bie.dlp_apply(g, s, o)
    torch.cuda.synchronize(); dm = (time.perf_counter() - t) / 50
    print(json.dumps(dict(cfg=cid, N=p.N, iters=r['iters'], gmres_ms=dt * 1e3, per_iter_us=dt * 1e6 / max(1, r['iters']),
                          matvec_us=dm * 1e6)), flush=True)
