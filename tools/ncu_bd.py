"""Short command for an ncu launch list of the BD factor (profiled range only)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem
p = make_problem(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
g = bie.Geometry.from_problem(p)
torch.cuda.synchronize()
torch.cuda.profiler.start()
bd = bie.BlockDiag(g)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
