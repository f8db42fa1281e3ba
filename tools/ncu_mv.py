"""ncu helper: one DLP matvec at config argv[1] with nvec argv[2] inside cudaProfilerStart/Stop."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1609_04484_b200 as bie  # noqa: E402
from bie_inputs import density, make_problem  # noqa: E402
cid, nvec = int(sys.argv[1]), int(sys.argv[2])
p = make_problem(cid)
g = bie.Geometry.from_problem(p)
s = torch.from_numpy(density(p, nvec=nvec).reshape(-1)).cuda(); o = torch.zeros_like(s)
bie.dlp_apply(g, s, o, nvec); torch.cuda.synchronize()
torch.cuda.profiler.start()
bie.dlp_apply(g, s, o, nvec); torch.cuda.synchronize()
torch.cuda.profiler.stop()
