"""ncu helper: one SLP matvec (config 4, nvec = 1) inside cudaProfilerStart/Stop."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1609_04484_b200 as bie  # noqa: E402
from bie_inputs import density, make_problem  # noqa: E402
p = make_problem(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
g = bie.Geometry.from_problem(p)
s = torch.from_numpy(density(p)[0]).cuda(); o = torch.zeros_like(s)
bie.slp_apply(g, s, o); torch.cuda.synchronize()
torch.cuda.profiler.start()
bie.slp_apply(g, s, o); torch.cuda.synchronize()
torch.cuda.profiler.stop()
