"""Write GMRES golden histories for the large configs by calling ONLY oracle/.

tests/test_gpu_bd_gmres.py::test_gmres_golden compares the CUDA path against
these files.  Inputs: bie_inputs (seeded); boundary data: pipe flow
(P:l.217-227, reading C10); solver: reading C13 (tol 1e-8).
usage: python tools/make_golden.py [config3_bd_pipe] [config4_none_pipe_prefix] [config4_bd_pipe_full]
"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from bie_inputs import make_problem, rhs_pipe

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
CASES = {
    "config3_bd_pipe": dict(config=3, pc="bd", tol=1e-8, max_iter=1000, env_runs=2),
    "config4_none_pipe_prefix": dict(config=4, pc="none", tol=1e-8, max_iter=6),
    "config4_bd_pipe_prefix": dict(config=4, pc="bdlu", tol=1e-8, max_iter=8, env_runs=2),
    # the full config-4 BD solve (579 iterations on the GPU): ~1 h of oracle time per run
    "config4_bd_pipe_full": dict(config=4, pc="bdlu", tol=1e-8, max_iter=2000, env_runs=1),
}
for name in (sys.argv[1:] or list(CASES)):
    c = CASES[name]
    p = make_problem(c["config"]); g = oracle.OracleGeometry(p)
    f = rhs_pipe(p)
    t0 = time.time()
    if c["pc"] == "bdlu":  # LU-solve form of the same BD operator (wall block too large to invert in plain C)
        bd = oracle.OracleBDLU(g)
        t1 = time.time()
        r = oracle.gmres_bdlu(g, f, bd, tol=c["tol"], max_iter=c["max_iter"])
    else:
        bd = oracle.OracleBD(g) if c["pc"] == "bd" else None
        t1 = time.time()
        r = oracle.gmres(g, f, bd, tol=c["tol"], max_iter=c["max_iter"])
    t2 = time.time()
    # self-sensitivity envelope (reading C23): the oracle's own history
    # under 1e-13 relative perturbations of f, at the GPU/oracle matvec agreement level
    env = np.zeros(len(r["hist"]))
    env_iters = []
    for s in range(c.get("env_runs", 0)):
        rng = np.random.default_rng(300 + s)
        fp = f * (1 + 1e-13 * rng.standard_normal(f.size))
        if c["pc"] == "bdlu":
            rp = oracle.gmres_bdlu(g, fp, bd, tol=c["tol"], max_iter=c["max_iter"])
        else:
            rp = oracle.gmres(g, fp, bd, tol=c["tol"], max_iter=c["max_iter"])
        n = min(len(r["hist"]), len(rp["hist"]))
        env[:n] = np.maximum(env[:n], np.abs(rp["hist"][:n] - r["hist"][:n]) / r["hist"][:n])
        env_iters.append(rp["iters"])
    rec = dict(name=name, **c, f_norm=float(np.linalg.norm(f)), iters=r["iters"], converged=r["converged"],
               hist=[float(h) for h in r["hist"]], res_pc=r["res_pc"], res_true=r["res_true"],
               envelope=[float(e) for e in env], envelope_iters=env_iters, envelope_eps=1e-13,
               oracle_build_s=t1 - t0, oracle_gmres_s=t2 - t1,
               source="oracle/bie_oracle.c via tools/make_golden.py; inputs bie_inputs seeded config",
               omp_threads=os.environ.get("OMP_NUM_THREADS", str(os.cpu_count())))
    os.makedirs(OUT, exist_ok=True)
    json.dump(rec, open(os.path.join(OUT, f"gmres_{name}.json"), "w"), indent=1)
    print(name, r["iters"], r["res_pc"], r["res_true"], f"build {t1-t0:.1f}s gmres {t2-t1:.1f}s", flush=True)
