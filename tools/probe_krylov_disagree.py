"""GPU-vs-oracle matvec disagreement on Krylov-like vectors (A^k f normalised)
of the no-PC config-2 systems, against the random-density level in
profiles/round2/disagreement.json (reading C23)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import oracle
import paper_1609_04484_b200 as bie
from bie_inputs import make_problem, rhs_pipe, rhs_shear_all

p = make_problem(2)
g = bie.Geometry.from_problem(p)
og = oracle.OracleGeometry(p)
for name, f in (("pipe", rhs_pipe(p)), ("shear_all", rhs_shear_all(p))):
    v = f / np.linalg.norm(f)
    out = []
    for k in range(30):
        y = torch.zeros(v.size, dtype=torch.float64, device="cuda")
        bie.dlp_apply(g, torch.from_numpy(v.copy()).cuda(), y, 1)
        torch.cuda.synchronize()
        yg = y.cpu().numpy()
        yo = og.apply(v)
        d = (yg - yo) / np.abs(yo).max()
        out.append((float(np.sqrt(np.mean(d * d))), float(np.abs(d).max())))
        v = yo / np.linalg.norm(yo)
    print(name, json.dumps({"rms_max": max(o[0] for o in out), "rms_med": float(np.median([o[0] for o in out])),
                            "max": max(o[1] for o in out)}), flush=True)
