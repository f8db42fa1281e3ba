"""Per-CTA start/end times of the symmetric DLP kernel (BIE_SYM_TRACE diagnostics)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, '.')
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem, density
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
out = os.environ["BIE_SYM_TRACE"]
p = make_problem(cid); g = bie.Geometry.from_problem(p)
s = torch.from_numpy(density(p)[0]).cuda(); o = torch.zeros_like(s)
for _ in range(3): bie.dlp_apply(g, s, o, 1, 1)
torch.cuda.synchronize()
g.close()
t = np.loadtxt(out, dtype=np.float64)
t0 = t[:, 0].min()
st, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
dur = en - st
P = len(t)
print(f"P={P} kernel span {en.max():.1f} us; start max {st.max():.1f} us; duration min/med/max {dur.min():.1f}/{np.median(dur):.1f}/{dur.max():.1f} us")
q = np.array_split(np.arange(P), 8)
print("mean duration by CTA octile:", [round(float(dur[i].mean()), 1) for i in q])
print("mean warps-active fraction:", dur.sum() / (P * en.max()))
