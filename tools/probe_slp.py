"""Time the single-layer matvec (NEXT-1) at the configs on argv: symmetric nvec=1,
one-sided nvec=1, nvec=4/16; and the SLP BD factor + BD-GMRES solve."""
import json, sys, time
import torch
sys.path.insert(0, '.')
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem, density, rhs_pipe
for cid in [int(c) for c in sys.argv[1:]] or [4]:
    p = make_problem(cid); g = bie.Geometry.from_problem(p)
    for nvec, flags in ((1, 0), (1, 2), (4, 0), (16, 0)):
        s = torch.from_numpy(density(p, nvec=nvec).reshape(-1)).cuda(); o = torch.zeros_like(s)
        for _ in range(2): bie.slp_apply(g, s, o, nvec, flags)
        torch.cuda.synchronize()
        bie.profile_begin(g)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3): bie.slp_apply(g, s, o, nvec, flags)
        e1.record(); torch.cuda.synchronize()
        pr = bie.profile_end(g)
        ms = e0.elapsed_time(e1) / 3
        print(json.dumps(dict(cfg=cid, nvec=nvec, flags=flags, ms=ms, gpairs=nvec * p.N * p.N / ms / 1e6,
                              pairs_ms=pr['pairs_ms'] / 3, epi_ms=pr['epilogue_ms'] / 3)), flush=True)
    torch.cuda.synchronize(); t = time.time(); bd = bie.BlockDiag(g, op="slp"); torch.cuda.synchronize()
    tf = time.time() - t
    f = torch.from_numpy(rhs_pipe(p)).cuda(); x = torch.zeros_like(f)
    t = time.time(); r = bie.gmres_solve_slp(g, bd, f, x, 1e-8, 300 if cid >= 4 else 1000); tg = time.time() - t
    print(json.dumps(dict(cfg=cid, slp_bd_factor_s=tf, slp_gmres_s=tg, iters=r['iters'], res_true=r['res_true'],
                          conv=r['converged'])), flush=True)
