"""Timing probe for BD factor/apply and GMRES (not the bench contract)."""
import sys, time, json
import numpy as np, torch
sys.path.insert(0, '.')
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem, density, rhs_pipe
for cid in [int(c) for c in sys.argv[1:]] or [3]:
    p = make_problem(cid); g = bie.Geometry.from_problem(p)
    torch.cuda.synchronize(); t = time.time(); bd = bie.BlockDiag(g); torch.cuda.synchronize(); tf = time.time() - t
    v = torch.from_numpy(density(p)[0]).cuda(); o = torch.zeros_like(v)
    for _ in range(3): bie.blockdiag_apply(bd, v, o)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): bie.blockdiag_apply(bd, v, o)
    e1.record(); torch.cuda.synchronize(); ta = e0.elapsed_time(e1) / 10
    nbytes = 8 * (p.M * (2 * p.n_pore) ** 2 + (2 * p.n_outer) ** 2)
    print(json.dumps(dict(cfg=cid, bd_factor_s=tf, bd_apply_ms=ta, bd_apply_GBps=nbytes / ta / 1e6)), flush=True)
    f = torch.from_numpy(rhs_pipe(p)).cuda(); x = torch.zeros_like(f)
    mi = 300 if cid >= 4 else 1000
    t = time.time(); r = bie.gmres_solve(g, bd, f, x, 1e-8, mi); tg = time.time() - t
    print(json.dumps(dict(cfg=cid, gmres_s=tg, iters=r['iters'], res_pc=r['res_pc'], res_true=r['res_true'],
                          conv=r['converged'], last=r['hist'][-1])), flush=True)
