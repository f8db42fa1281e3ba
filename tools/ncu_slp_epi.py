"""One config-4 SLP apply and one DLP apply inside cudaProfilerStart/Stop (for
ncu captures of the SLP symmetric kernel and the DLP epilogue)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1609_04484_b200 as bie
from bie_inputs import density, make_problem
p = make_problem(4); g = bie.Geometry.from_problem(p)
s = torch.from_numpy(density(p, nvec=1).reshape(-1)).cuda(); o = torch.zeros_like(s)
bie.slp_apply(g, s, o); bie.dlp_apply(g, s, o); torch.cuda.synchronize()
torch.cuda.profiler.start()
bie.slp_apply(g, s, o); bie.dlp_apply(g, s, o)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
