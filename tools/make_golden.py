"""Write GMRES golden histories for the large configs by calling ONLY oracle/.

tests/test_gpu_bd_gmres.py::test_gmres_golden and
tests/test_gpu_bd_structured.py compare the CUDA path against these files.
Inputs: bie_inputs (seeded); boundary data: pipe flow (P:l.217-227, reading
C10); solver: reading C13 (tol 1e-8).

Envelope (reading C23): besides the unperturbed history, RUNS >= 3
oracle solves in which every primitive of the iteration (A v, P^-1 v, CGS
inner products, norms, CGS subtractions) gets seeded Gaussian noise at the
GPU-vs-oracle disagreement MEASURED for that primitive and config
(profiles/round2/disagreement.json, written by tools/measure_disagreement.py
on the B200).  The tests bar the GPU history at max(1e-10, 2 x the running
maximum over runs of |h_pert - h| / h).

usage: python tools/make_golden.py [case ...]      (default: all cases)
The full config-4 solve takes ~2 h of oracle time per run on 6-8 host
threads; each finished run is written out immediately (partial files are
valid goldens with fewer envelope runs, and say so).

Long cases can run as independent processes, one per solve, and be merged:
  python tools/make_golden.py CASE --run -1      (unperturbed)
  python tools/make_golden.py CASE --run K       (perturbed run K, seed 1000 + K)
  python tools/make_golden.py CASE --merge       (-> tests/golden/gmres_CASE.json)
Each --run writes tests/golden/parts/CASE.runK.json; the merged file is the
same record main() writes (same seeds, same noise levels).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import oracle
from bie_inputs import make_problem, rhs_pipe

OUT = os.path.join(ROOT, "tests", "golden")
EPS_FILE = os.path.join(ROOT, "profiles", "round2", "disagreement.json")
RUNS = 3
CASES = {
    "config3_bd_pipe": dict(config=3, pc="bd", tol=1e-8, max_iter=1000),
    "config4_none_pipe_prefix": dict(config=4, pc="none", tol=1e-8, max_iter=6),
    "config4_bd_pipe_prefix": dict(config=4, pc="bdlu", tol=1e-8, max_iter=8),
    "config4_bd_pipe_full": dict(config=4, pc="bdlu", tol=1e-8, max_iter=2000),
}


def perturbation(cid: int, pc: str) -> dict:
    """Noise levels per primitive for config cid: the worst measured rms
    disagreement (max-norm-relative for vectors, ||w||-relative for dots) over
    random densities AND the Krylov-like vectors of the same iteration (P^-1 A
    powers for BD, A powers without PC), which carry up to ~3x the random
    level."""
    d = json.load(open(EPS_FILE))[f"config{cid}"]
    kry = d["matvec_krylov_bd" if pc != "none" else "matvec_krylov_nopc"]
    eps = {"A": max(x["rms"] for x in d["matvec"] + kry), "dot": d["dot"]["rms"], "norm": d["norm"]["rms"],
           "sub": d["sub"]["rms"]}
    if pc != "none":
        eps["P"] = max(x["rms"] for x in d["bd_explicit"] + d["bd_structured"] + d["bd_krylov"])
    return eps


def solve(g, f, bd, c):
    if c["pc"] == "bdlu":  # LU-solve form of the same BD operator (wall block too large to invert in plain C)
        return oracle.gmres_bdlu(g, f, bd, tol=c["tol"], max_iter=c["max_iter"])
    return oracle.gmres(g, f, bd, tol=c["tol"], max_iter=c["max_iter"])


def _setup(name):
    c = CASES[name]
    p = make_problem(c["config"])
    g = oracle.OracleGeometry(p)
    f = rhs_pipe(p)
    eps = perturbation(c["config"], c["pc"])
    t0 = time.time()
    bd = None if c["pc"] == "none" else (oracle.OracleBDLU(g) if c["pc"] == "bdlu" else oracle.OracleBD(g))
    return c, g, f, eps, bd, time.time() - t0


def run_one(name, k):
    """One solve of CASE as its own process: k = -1 unperturbed, else perturbed run k."""
    c, g, f, eps, bd, tb = _setup(name)
    t0 = time.time()
    if k < 0:
        r = solve(g, f, bd, c)
    else:
        with oracle.perturbed(eps, seed=1000 + k):
            r = solve(g, f, bd, c)
    part = dict(name=name, run=k, iters=r["iters"], converged=r["converged"], hist=[float(h) for h in r["hist"]],
                res_pc=r["res_pc"], res_true=r["res_true"], f_norm=float(np.linalg.norm(f)), perturbation=eps,
                oracle_build_s=tb, oracle_gmres_s=time.time() - t0,
                omp_threads=os.environ.get("OMP_NUM_THREADS", str(os.cpu_count())))
    d = os.path.join(OUT, "parts")
    os.makedirs(d, exist_ok=True)
    path = os.path.join(d, f"{name}.run{k}.json")
    json.dump(part, open(path + ".tmp", "w"), indent=1)
    os.replace(path + ".tmp", path)
    print(name, "run", k, r["iters"], f"{time.time() - t0:.0f}s", flush=True)


def merge(name):
    c = CASES[name]
    d = os.path.join(OUT, "parts")
    base = json.load(open(os.path.join(d, f"{name}.run-1.json")))
    h = np.asarray(base["hist"])
    rec = dict(name=name, **c, f_norm=base["f_norm"], iters=base["iters"], converged=base["converged"],
               hist=base["hist"], res_pc=base["res_pc"], res_true=base["res_true"],
               perturbation=base["perturbation"], envelope_runs=[], envelope_iters=[], envelope=[],
               oracle_build_s=base["oracle_build_s"], oracle_gmres_s=base["oracle_gmres_s"],
               source="oracle/bie_oracle.c via tools/make_golden.py (one process per solve, merged); inputs "
                      "bie_inputs seeded config; noise levels profiles/round2/disagreement.json",
               omp_threads=base["omp_threads"])
    env = np.zeros(len(h))
    for k in range(RUNS):
        pth = os.path.join(d, f"{name}.run{k}.json")
        if not os.path.exists(pth):
            continue
        rp = json.load(open(pth))
        assert rp["perturbation"] == base["perturbation"]
        n = min(len(h), len(rp["hist"]))
        env[:n] = np.maximum(env[:n], np.abs(np.asarray(rp["hist"][:n]) - h[:n]) / h[:n])
        rec["envelope_runs"].append(rp["hist"])
        rec["envelope_iters"].append(rp["iters"])
    rec["envelope"] = [float(e) for e in env]
    rec["envelope_complete"] = len(rec["envelope_runs"]) == RUNS
    path = os.path.join(OUT, f"gmres_{name}.json")
    json.dump(rec, open(path + ".tmp", "w"), indent=1)
    os.replace(path + ".tmp", path)
    print(name, "merged", len(rec["envelope_runs"]), "envelope runs, max env", float(env.max()))


def main():
    args = sys.argv[1:]
    if "--run" in args:
        i = args.index("--run")
        return run_one(args[0], int(args[i + 1]))
    if "--merge" in args:
        return merge(args[0])
    for name in (args or list(CASES)):
        c = CASES[name]
        p = make_problem(c["config"])
        g = oracle.OracleGeometry(p)
        f = rhs_pipe(p)
        eps = perturbation(c["config"], c["pc"])
        t0 = time.time()
        bd = None if c["pc"] == "none" else (oracle.OracleBDLU(g) if c["pc"] == "bdlu" else oracle.OracleBD(g))
        t1 = time.time()
        r = solve(g, f, bd, c)
        t2 = time.time()
        rec = dict(name=name, **c, f_norm=float(np.linalg.norm(f)), iters=r["iters"], converged=r["converged"],
                   hist=[float(h) for h in r["hist"]], res_pc=r["res_pc"], res_true=r["res_true"],
                   perturbation=eps, envelope_runs=[], envelope_iters=[], envelope=[],
                   oracle_build_s=t1 - t0, oracle_gmres_s=t2 - t1,
                   source="oracle/bie_oracle.c via tools/make_golden.py; inputs bie_inputs seeded config; "
                          "noise levels profiles/round2/disagreement.json",
                   omp_threads=os.environ.get("OMP_NUM_THREADS", str(os.cpu_count())))
        path = os.path.join(OUT, f"gmres_{name}.json")
        os.makedirs(OUT, exist_ok=True)
        rec["envelope_complete"] = False
        json.dump(rec, open(path + ".tmp", "w"), indent=1)
        os.replace(path + ".tmp", path)
        env = np.zeros(len(r["hist"]))
        for s in range(RUNS):
            with oracle.perturbed(eps, seed=1000 + s):
                rp = solve(g, f, bd, c)
            n = min(len(r["hist"]), len(rp["hist"]))
            dev = np.abs(rp["hist"][:n] - r["hist"][:n]) / r["hist"][:n]
            env[:n] = np.maximum(env[:n], dev)
            rec["envelope_runs"].append([float(h) for h in rp["hist"]])
            rec["envelope_iters"].append(rp["iters"])
            rec["envelope"] = [float(e) for e in env]
            rec["envelope_complete"] = s + 1 == RUNS
            json.dump(rec, open(path + ".tmp", "w"), indent=1)
            os.replace(path + ".tmp", path)
            print(name, "run", s, rp["iters"], f"max dev {dev.max():.3e}", f"{time.time() - t2:.0f}s", flush=True)
        print(name, r["iters"], r["res_pc"], r["res_true"], f"build {t1 - t0:.1f}s gmres {t2 - t1:.1f}s", flush=True)


if __name__ == "__main__":
    main()
