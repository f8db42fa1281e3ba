"""Where do the bench step's extra ~35 ms go (735 ms/step vs 700 ms of kernels in
the ncu launch list)?  Times the 50-iteration config-4 BD-GMRES step with CUDA
events under several conditions."""
import json, os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem, rhs_pipe

p = make_problem(4)
g = bie.Geometry.from_problem(p)
bd = bie.BlockDiag(g, structured=True)
f = torch.from_numpy(rhs_pipe(p)).cuda()
x = torch.zeros_like(f)
flush = torch.empty((256 << 20) // 8, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()


def steps(k=3, prof=False, flush_l2=True):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
    torch.cuda.synchronize()
    if prof:
        bie.profile_begin(g)
    for i in range(k):
        if flush_l2:
            flush.fill_(float(i))
        ev[i][0].record(st)
        bie.gmres_solve(g, bd, f, x, tol=1e-30, max_iter=50)
        ev[i][1].record(st)
    torch.cuda.synchronize()
    out = {"ms": [round(a.elapsed_time(b), 2) for a, b in ev]}
    if prof:
        pr = bie.profile_end(g)
        out["pairs_ms_per_apply"] = pr["pairs_ms"] / max(1, pr["applies"])
        out["epi_ms_per_apply"] = pr["epilogue_ms"] / max(1, pr["applies"])
    return out


for _ in range(3):
    bie.gmres_solve(g, bd, f, x, tol=1e-30, max_iter=50)
res = {}
res["plain"] = steps()
res["prof"] = steps(prof=True)
res["noflush"] = steps(flush_l2=False)
sm = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader", "-lms", "200"],
                      stdout=subprocess.DEVNULL)
time.sleep(1.0)
res["with_smi"] = steps(prof=True)
sm.terminate()
bie.fp64_peak(200000)
res["after_fp64_peak"] = steps(prof=True)
# standalone matvec loop
s = torch.randn(2 * p.N, dtype=torch.float64, device="cuda")
o = torch.zeros_like(s)
for _ in range(3):
    bie.dlp_apply(g, s, o, 1)
torch.cuda.synchronize()
bie.profile_begin(g)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(10):
    bie.dlp_apply(g, s, o, 1)
e1.record(st)
torch.cuda.synchronize()
pr = bie.profile_end(g)
res["matvec_loop"] = {"ms_per": e0.elapsed_time(e1) / 10, "pairs_ms_per_apply": pr["pairs_ms"] / pr["applies"],
                      "epi_ms_per_apply": pr["epilogue_ms"] / pr["applies"]}
print(json.dumps(res, indent=1))
