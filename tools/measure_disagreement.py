"""Measure the GPU-vs-oracle disagreement of the two operators GMRES applies
(A v and P^-1 v), per config -- the perturbation amplitude of the GMRES
envelope runs (reading C23, tools/make_golden.py).

For each config: several seeded N(0,1) densities (bie_inputs.density), the
completed DLP matvec (BIE_FULL) and the BD apply (explicit and structured
pore blocks) on the GPU against the oracle on the same inputs.  Reported per
vector: max |gpu - ora| / max |ora| (the C15 norm) and the rms of
(gpu - ora) / max |ora|.  Config 4's oracle BD is the LU form (plain-C
inversion of the 16384^2 wall block takes hours); its GPU applies are saved to
gpurun_out/ so the comparison can be finished on any host.

usage: python tools/measure_disagreement.py [configs...] > gpurun_out/disagree.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import oracle
import paper_1609_04484_b200 as bie
from bie_inputs import density, make_problem, rhs_pipe

OUT = os.path.join(ROOT, "gpurun_out")


def stats(y, r):
    d = (y - r) / np.abs(r).max()
    return {"max": float(np.abs(d).max()), "rms": float(np.sqrt(np.mean(d * d)))}


def main():
    cfgs = [int(c) for c in sys.argv[1:]] or [1, 2, 3, 4]
    res = {}
    os.makedirs(OUT, exist_ok=True)
    for cid in cfgs:
        p = make_problem(cid)
        g = bie.Geometry.from_problem(p)
        og = oracle.OracleGeometry(p)
        nv = 4
        s = density(p, nvec=nv, vec_id=70)
        sig = torch.from_numpy(s.reshape(-1).copy()).cuda()
        rec = {"N": p.N, "matvec": [], "bd_explicit": [], "bd_structured": []}
        t0 = time.time()
        ref = og.apply(s)
        rec["oracle_matvec_s"] = (time.time() - t0) / nv
        for v in range(nv):
            o = torch.zeros(2 * p.N, dtype=torch.float64, device="cuda")
            bie.dlp_apply(g, sig[v * 2 * p.N:(v + 1) * 2 * p.N], o, 1)  # nvec = 1: the symmetric path GMRES uses
            torch.cuda.synchronize()
            rec["matvec"].append(stats(o.cpu().numpy(), ref[v]))
        bde = bie.BlockDiag(g)
        bds = bie.BlockDiag(g, structured=True)
        # Krylov-like vectors -- what GMRES actually applies the operators to:
        # no PC: v <- A v / |A v| from f; BD: v <- P^-1 A v / |.| from P^-1 f
        # (generated on the GPU; they are probe inputs, not expected values)
        f = rhs_pipe(p)
        kry = {"nopc": [], "bd": []}
        for kind in kry:
            v = torch.from_numpy(f.copy()).cuda()
            if kind == "bd":
                t = torch.zeros_like(v)
                bie.blockdiag_apply(bde, v, t)
                v = t
            for _ in range(12):
                v = v / torch.linalg.norm(v)
                kry[kind].append(v.cpu().numpy())
                t = torch.zeros_like(v)
                bie.dlp_apply(g, v, t, 1)
                if kind == "bd":
                    z = torch.zeros_like(v)
                    bie.blockdiag_apply(bde, t, z)
                    t = z
                v = t
        K = np.array(kry["nopc"] + kry["bd"])
        KA = []
        for v in K:
            o = torch.zeros(v.size, dtype=torch.float64, device="cuda")
            bie.dlp_apply(g, torch.from_numpy(v.copy()).cuda(), o, 1)
            torch.cuda.synchronize()
            KA.append(o.cpu().numpy())
        ro = og.apply(K)
        rec["matvec_krylov_nopc"] = [stats(KA[q], ro[q]) for q in range(12)]
        rec["matvec_krylov_bd"] = [stats(KA[q], ro[q]) for q in range(12, 24)]
        KB = np.array(kry["bd"])
        KBe, KBs = [], []
        for v in KB:
            vv = torch.from_numpy(v.copy()).cuda()
            oe, os_ = torch.zeros_like(vv), torch.zeros_like(vv)
            bie.blockdiag_apply(bde, vv, oe)
            bie.blockdiag_apply(bds, vv, os_)
            torch.cuda.synchronize()
            KBe.append(oe.cpu().numpy())
            KBs.append(os_.cpu().numpy())
        ye, ys = [], []
        for v in range(nv):
            x = sig[v * 2 * p.N:(v + 1) * 2 * p.N]
            oe = torch.zeros_like(x)
            os_ = torch.zeros_like(x)
            bie.blockdiag_apply(bde, x, oe)
            bie.blockdiag_apply(bds, x, os_)
            torch.cuda.synchronize()
            ye.append(oe.cpu().numpy())
            ys.append(os_.cpu().numpy())
        bde.close()
        bds.close()
        if cid <= 3:
            obd = oracle.OracleBD(og)
            for v in range(nv):
                r = obd.apply(s[v])
                rec["bd_explicit"].append(stats(ye[v], r))
                rec["bd_structured"].append(stats(ys[v], r))
            rec["bd_krylov"] = []
            for q in range(KB.shape[0]):
                r = obd.apply(KB[q])
                rec["bd_krylov"].append(stats(KBe[q], r))
                rec["bd_krylov"].append(stats(KBs[q], r))
        else:
            # gpurun copies back <= 64 MiB: the random-density applies (already
            # measured) stay out; 6 of the Krylov-like vectors go in
            np.savez(os.path.join(OUT, f"bd_apply_config{cid}.npz"), kry=KB[:6], kry_explicit=np.array(KBe[:6]),
                     kry_structured=np.array(KBs[:6]))
            rec["bd_note"] = f"GPU BD applies saved to gpurun_out/bd_apply_config{cid}.npz (oracle LU form offline)"
        # Krylov primitives (bie_krylov_dots / _axpy vs the oracle GMRES's own loops) on
        # an orthonormal-like basis of 32 normalised Gaussian vectors and a unit w
        n = 2 * p.N
        rng = np.random.default_rng(900 + cid)
        Vh = rng.standard_normal((32, n))
        Vh /= np.linalg.norm(Vh, axis=1, keepdims=True)
        wh = rng.standard_normal(n)
        wh /= np.linalg.norm(wh)
        V = torch.from_numpy(Vh).cuda()
        w = torch.from_numpy(wh).cuda()
        out = torch.zeros(64, dtype=torch.float64, device="cuda")
        bie.Krylov.dots(V, n, 32, w, n, out)
        for j in range(32):  # ||V_j||^2 with the norm kernel path (a 1-vector multidot)
            bie.Krylov.dots(V[j], n, 1, V[j], n, out[32 + j:33 + j])
        torch.cuda.synchronize()
        od = out.cpu().numpy()
        rd = oracle.cgs_dots(Vh, wh)
        rn = np.sqrt(np.array([oracle.cgs_dots(Vh[j][None, :], Vh[j])[0] for j in range(32)]))
        gn = np.sqrt(od[32:])
        rec["dot"] = {"max": float(np.abs(od[:32] - rd).max()), "rms": float(np.sqrt(np.mean((od[:32] - rd) ** 2)))}
        rec["norm"] = {"max": float(np.abs(gn / rn - 1).max()), "rms": float(np.sqrt(np.mean((gn / rn - 1) ** 2)))}
        h = torch.from_numpy(rd.copy()).cuda()
        y = w.clone()
        bie.Krylov.axpy(V, n, 32, h, -1.0, 1.0, y, n)
        torch.cuda.synchronize()
        ys = oracle.cgs_sub(Vh, rd, wh)
        rec["sub"] = stats(y.cpu().numpy(), ys)
        if cid <= 2:  # NEXT-1 single-layer operator and its BD (configs 1-2, C26)
            rs = og.slp_apply(s)
            rec["slp_matvec"], rec["slp_bd"] = [], []
            bds = bie.BlockDiag(g, op="slp")
            obs = oracle.OracleSLPBD(og)
            for v in range(nv):
                x = sig[v * 2 * p.N:(v + 1) * 2 * p.N]
                o = torch.zeros_like(x)
                bie.slp_apply(g, x, o)
                ob = torch.zeros_like(x)
                bie.blockdiag_apply(bds, x, ob)
                torch.cuda.synchronize()
                rec["slp_matvec"].append(stats(o.cpu().numpy(), rs[v]))
                rec["slp_bd"].append(stats(ob.cpu().numpy(), obs.apply(s[v])))
            bds.close()
        res[f"config{cid}"] = rec
        print(json.dumps({f"config{cid}": rec}), flush=True)
        g.close()
    json.dump(res, open(os.path.join(OUT, "disagree.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
