"""Short command for ncu captures: setup + warm-up outside the profiled range,
then exactly one bench step (or one matvec) inside cudaProfilerStart/Stop.

ncu --profile-from-start off ... python tools/ncu_step.py [step|matvec] [config]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1609_04484_b200 as bie  # noqa: E402
from bie_inputs import density, make_problem, rhs_pipe  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "step"
cid = int(sys.argv[2]) if len(sys.argv) > 2 else 4
p = make_problem(cid)
g = bie.Geometry.from_problem(p)
dev = torch.device("cuda", 0)
if mode == "step":
    bd = bie.BlockDiag(g, structured=True)
    f = torch.from_numpy(rhs_pipe(p)).to(dev)
    x = torch.zeros_like(f)
    bie.gmres_solve(g, bd, f, x, tol=1e-30, max_iter=50)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    bie.gmres_solve(g, bd, f, x, tol=1e-30, max_iter=50)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
else:
    nvec = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    s = torch.from_numpy(density(p, nvec=nvec).reshape(-1)).to(dev)
    o = torch.zeros_like(s)
    bie.dlp_apply(g, s, o, nvec)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    bie.dlp_apply(g, s, o, nvec)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
print("ok")
