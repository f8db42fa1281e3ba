"""Per-step device times of the bench step (50-iteration BD-GMRES, config 4) to
study step-time jitter: BIE_GMRES_LOOKAHEAD, clock sampler on/off."""
import json, os, subprocess, sys, time
import torch
sys.path.insert(0, '.')
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem, rhs_pipe
p = make_problem(4); g = bie.Geometry.from_problem(p); bd = bie.BlockDiag(g, structured=True)
f = torch.from_numpy(rhs_pipe(p)).cuda(); x = torch.zeros_like(f)
for _ in range(3): bie.gmres_solve(g, bd, f, x, tol=1e-30, max_iter=50)
smi = None
if len(sys.argv) > 1 and sys.argv[1] == "smi":
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "200"],
                           stdout=subprocess.DEVNULL)
    time.sleep(2)
ms, wall = [], []
for k in range(12):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record(); bie.gmres_solve(g, bd, f, x, tol=1e-30, max_iter=50); b.record(); torch.cuda.synchronize()
    wall.append((time.perf_counter() - t0) * 1e3); ms.append(a.elapsed_time(b))
if smi: smi.terminate()
print(json.dumps(dict(look=os.environ.get("BIE_GMRES_LOOKAHEAD", "3"), smi=smi is not None,
                      ms=[round(v, 1) for v in ms], wall=[round(v, 1) for v in wall])), flush=True)
