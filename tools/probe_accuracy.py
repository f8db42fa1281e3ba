"""Save GPU matvec outputs (configs 3-4, density vec 70) for an accuracy study
against the oracle and a long-double reference (reading C15).

usage: python tools/probe_accuracy.py  -> gpurun_out/acc_config{3,4}.npz
Paths: symmetric (default), one-sided (BIE_ONE_SIDED), BIE_FULL and BIE_D_ONLY.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1609_04484_b200 as bie
from bie_inputs import density, make_problem

BIE_ONE_SIDED = 2


def main():
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    for cid in [int(c) for c in sys.argv[1:]] or [3, 4]:
        p = make_problem(cid)
        g = bie.Geometry.from_problem(p)
        s = density(p, nvec=4, vec_id=70)[0]
        sig = torch.from_numpy(s.copy()).cuda()
        res = {}
        for name, fl in (("sym_full", 0), ("sym_donly", 1), ("one_full", BIE_ONE_SIDED), ("one_donly", 1 | BIE_ONE_SIDED)):
            o = torch.zeros_like(sig)
            bie.dlp_apply(g, sig, o, 1, fl)
            torch.cuda.synchronize()
            res[name] = o.cpu().numpy()
        np.savez(os.path.join(ROOT, "gpurun_out", f"acc_config{cid}.npz"), s=s, **res)
        print(cid, "saved", flush=True)
        g.close()


if __name__ == "__main__":
    main()
