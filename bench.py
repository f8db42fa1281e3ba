#!/usr/bin/env python
"""Benchmark of the B200 hot path (see DESIGN.md s5 for every definition).

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Workload (BASELINE.json configs[3]): pipe L=100,
1000 pores, N = 136,192 boundary nodes (272,384 FP64 unknowns), pipe-flow
boundary data.  One STEP = one left-preconditioned BD-GMRES solve with a fixed
budget of 50 iterations (tol below reach) through bie_gmres_solve: 51 completed
DLP matvecs (A2-A5: 50 Arnoldi + 1 residual), 52 BD applies (A7), CGS2 +
Givens (A8) and the finish (A9).  Setup (A1 geometry, A6 BD factor) happens
once before timing and is reported separately ("build PC", P:l.720).

metric = DLP matvec pair-interactions/s (N^2 per matvec, self pairs included
since the kernel evaluates them branch-free).

N > 1 (torchrun): the SAME solve is row-sharded over the ranks
(paper_1609_04484_b200.dist: body-range BD, all-gather of the density per
matvec, all-reduced inner products over NCCL) -> strong scaling; value is the
whole job's pair interactions over the max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG_ID = 4
GMRES_ITERS = 50
FLOP_PER_PAIR = 19  # algorithmic, nvec = 1 (11 geometry + 8 per vector)
# FP64 CUDA-core peak derived from unit counts and clocks:
# 148 SMs x 64 FP64 FMA/clk x 2 flop x 1.965 GHz (MEASURED_PEAKS.json sm_max_mhz)
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2


def _ncu_traffic(key="traffic_bytes_per_launch"):
    """DRAM bytes per launch (or another field) of the dominant kernel from the committed
    ncu --set full capture of the current kernel (profiles/round2/k_dlp_sym_traffic.json)."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "round2", "k_dlp_sym_traffic.json")))[key]
    except Exception:
        return None


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's start-up (NVML init, device enumeration) holds driver
            # locks for ~100 ms; wait for its first sample so that cost lands
            # before the timed region, not inside its first steps
            t0 = time.time()
            while not self.lines and time.time() - t0 < 10 and self.proc.poll() is None:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax = float(f[1])
            except ValueError:
                continue
            try:
                pw.append(float(f[2]))
            except ValueError:
                pass
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "sm_mhz_min": min(sm) if sm else None, "power_w_max": max(pw) if pw else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_baseline_sample(problem, seconds=12.0, max_rows=None):
    """Oracle completed matvec on a bounded strided row sample (TEST INFRA: oracle/)."""
    import numpy as np

    import oracle
    from bie_inputs import density

    og = oracle.OracleGeometry(problem)
    s = density(problem)[0]
    N = problem.N
    rows_per_batch = 256
    done_pairs, t_used, batch = 0, 0.0, 0
    stride = 97  # co-prime walk over targets
    while t_used < seconds and (max_rows is None or batch * rows_per_batch < max_rows):
        rows = ((np.arange(rows_per_batch) + batch * rows_per_batch) * stride % N).astype(np.int32)
        t0 = time.perf_counter()
        og.apply(s, rows=rows)
        t_used += time.perf_counter() - t0
        done_pairs += rows_per_batch * N
        batch += 1
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            model = next((ln.split(":", 1)[1].strip() for ln in fh if ln.startswith("model name")), None)
    except OSError:
        pass
    return {"value": done_pairs / t_used, "unit": "pair-interactions/s", "cores": cores, "kind": "oracle",
            "cpu_model": model, "omp_num_threads": os.environ.get("OMP_NUM_THREADS"),
            "sample": f"{batch * rows_per_batch} strided target rows x all {N} sources of the config-{problem.config_id} "
                      f"completed DLP matvec (oracle/bie_oracle.c, OpenMP over rows), {t_used:.1f} s",
            "seconds": t_used}


def cpu_gmres_baseline():
    """The oracle's BD-GMRES on the host cores (TEST INFRA: oracle/), next to the
    GPU solves (north_star; P:l.719-723 reports "Build PC" and "GMRES" per run):
      config 3 -- a full solve to 1e-8 (BD in the oracle's LU-solve form);
      config 4 -- bounded: LU of the 1000 pore blocks (timed), LU of the leading
        4096^2 block of the 16384^2 wall block (timed, extrapolated x 64 = O(n^3)),
        one oracle matvec (timed) as the cost of an iteration (BD apply and CGS2
        are < 5% of it), times the GPU solve's iteration count -- extrapolated,
        and labelled so."""
    import numpy as np

    import oracle
    from bie_inputs import make_problem, rhs_pipe

    out = {"cores": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)), "kind": "oracle"}
    p = make_problem(3)
    og = oracle.OracleGeometry(p)
    f = rhs_pipe(p)
    t0 = time.perf_counter()
    bd = oracle.OracleBDLU(og)
    t1 = time.perf_counter()
    r = oracle.gmres_bdlu(og, f, bd, tol=1e-8, max_iter=1000)
    t2 = time.perf_counter()
    out["config3"] = {"build_pc_s": t1 - t0, "gmres_s": t2 - t1, "iters": r["iters"], "converged": r["converged"],
                      "res_true": r["res_true"], "sample": "full oracle BD-GMRES solve (LU-form BD), measured"}
    del bd
    p = make_problem(4)
    og = oracle.OracleGeometry(p)
    nw = 2 * p.n_outer
    t0 = time.perf_counter()
    for b in range(p.M):  # the pore blocks, factored as the oracle's BD does
        oracle.lu(og.bd_block(b))
    t_pores = time.perf_counter() - t0
    W = og.bd_block(p.M)[:4096, :4096].copy()
    t0 = time.perf_counter()
    oracle.lu(W)
    t_w4096 = time.perf_counter() - t0
    s = rhs_pipe(p)
    t0 = time.perf_counter()
    og.apply(s)
    t_mv = time.perf_counter() - t0
    build = t_pores + t_w4096 * (nw / 4096) ** 3
    out["config4"] = {"build_pc_s_extrapolated": build, "pores_factor_s": t_pores,
                      "wall_lu_4096_s": t_w4096, "matvec_s": t_mv,
                      "gmres_s_per_iteration_extrapolated": t_mv,
                      "sample": f"extrapolated: pore factors timed; wall LU ({nw}^2) from a timed 4096^2 LU x "
                                f"{(nw / 4096) ** 3:.0f}; per iteration = one timed oracle matvec (BD apply and "
                                f"CGS2 excluded, < 5% of it)"}
    return out


def run_reference(args):
    """--impl reference: the CPU oracle as it stands, same metric/unit, rank 0 only."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    # torchrun sets OMP_NUM_THREADS=1 for multi-process launches; the reference arm
    # is the oracle on all of the box's host cores (set before liboracle loads OpenMP)
    if ws > 1 or "OMP_NUM_THREADS" not in os.environ:
        os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    from bie_inputs import make_problem

    p = make_problem(CONFIG_ID)
    per_step_s = max(2.0, min(15.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_baseline_sample(p, seconds=per_step_s / 4)
    vals, secs = [], 0.0
    last = None
    for _ in range(args.steps):
        last = cpu_baseline_sample(p, seconds=per_step_s)
        vals.append(last["value"])
        secs += last["seconds"]
    value = statistics.mean(vals)
    pairs_per_step = GMRES_ITERS + 1
    line = {
        "impl": "reference", "metric": "DLP matvec pair-interactions/s", "value": value,
        "unit": "pair-interactions/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * pairs_per_step * p.N * p.N / value, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config4 pipe L=100 M=1000 N={p.N}: oracle completed DLP matvec rows "
                               f"(bounded sample per step; ms_per_step extrapolated to {pairs_per_step} matvecs)",
                   "N": p.N, "unknowns": 2 * p.N},
        "cpu_baseline": {"value": value, "unit": "pair-interactions/s", "cores": last["cores"], "kind": "oracle",
                         "sample": last["sample"]},
        "e2e": {"value": value, "unit": "pair-interactions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config5_sweep(bie, dev, stream):
    """BASELINE.json configs[4]: N = 1,064,960 matvec sweep over nvec in {1, 4, 16}
    (bie_dlp_apply, BIE_FULL), plus the oracle on a 4096-row subsample
    extrapolated as O(N^2)."""
    import numpy as np
    import torch

    import oracle
    from bie_inputs import density, make_problem

    p = make_problem(5)
    g = bie.Geometry.from_problem(p)
    res = {"N": p.N}
    for nvec in (1, 4, 16):
        s = torch.from_numpy(density(p, nvec=nvec).reshape(-1)).to(dev)
        o = torch.zeros_like(s)
        bie.dlp_apply(g, s, o, nvec)
        times = []
        for _ in range(3):  # median of 3
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            bie.dlp_apply(g, s, o, nvec)
            b.record(stream)
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        ms = statistics.median(times)
        res[f"nvec{nvec}"] = {"ms": ms, "ms_each": times, "pairs_per_s": nvec * p.N * p.N / (ms * 1e-3),
                              "alg_tflops": (11 + 8 * nvec) * p.N * p.N / (ms * 1e-3) / 1e12}
        del s, o
    og = oracle.OracleGeometry(p)
    rows = np.linspace(0, p.N - 1, 4096).astype(np.int32)
    s0 = density(p)[0]
    t0 = time.perf_counter()
    og.apply(s0, rows=rows)
    t = time.perf_counter() - t0
    res["oracle_4096_rows"] = {"seconds": t, "pairs_per_s": 4096 * p.N / t,
                               "extrapolated_full_matvec_s": t * p.N / 4096,
                               "cores": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))}
    g.close()
    return res


def run_gpu(args):
    import numpy as np
    import torch

    import paper_1609_04484_b200 as bie
    from bie_inputs import density, make_problem, rhs_pipe

    ws, rank, local = _dist()
    # --dist-backend gloo: a correctness run of the multi-rank flow when there are
    # fewer GPUs than ranks (ranks share devices; never a timing run)
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()

    p = make_problem(CONFIG_ID)
    N = p.N
    t0 = time.perf_counter()
    g = bie.Geometry.from_problem(p)
    torch.cuda.synchronize()
    t_geom = time.perf_counter() - t0
    t0 = time.perf_counter()
    if ws == 1:
        bd = bie.BlockDiag(g, structured=True)  # pores: one inverse + rank-2 Woodbury terms (NEXT-4)
        rb, re_ = 0, N
    else:
        # row-sharded solve: body-range BD on each rank,
        # all-gather of the density per matvec, all-reduced inner products
        from paper_1609_04484_b200.dist import GpuBackend, dist_gmres

        be = GpuBackend(g, rank, ws)
        rb, re_ = be.rb, be.re
    torch.cuda.synchronize()
    t_bd = time.perf_counter() - t0

    f_full = rhs_pipe(p)
    f_host = torch.from_numpy(np.ascontiguousarray(f_full[2 * rb:2 * re_])).pin_memory()
    f = f_host.to(dev)
    x = torch.zeros_like(f)
    x_host = torch.zeros_like(f_host).pin_memory()
    flush = torch.empty(L2_FLUSH_BYTES // 8, dtype=torch.float64, device=dev)
    # whole-job pair interactions per step (all ranks together)
    pairs_per_step = (GMRES_ITERS + 1) * N * N

    def step():
        if ws == 1:
            return bie.gmres_solve(g, bd, f, x, tol=1e-30, max_iter=GMRES_ITERS)
        xx, rr = dist_gmres(be, f, tol=1e-30, max_iter=GMRES_ITERS)
        x.copy_(xx)
        return rr

    for _ in range(max(3, args.warmup)):
        r = step()
    assert r["iters"] == GMRES_ITERS
    # measured FP64 peak of this device (DFMA chains, libbie.so bie_fp64_peak), best of 3
    fp64_meas = max(bie.fp64_peak(200000)["tflops"] for _ in range(3))

    # ---- timed region: device-resident inputs, L2 flushed between steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = bie.launch_count()
    bie.profile_begin(g)
    with ClockSampler(local) as clk:
        torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include "timed/" selects this region
        for k in range(args.steps):
            flush.fill_(float(k))
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
    prof = bie.profile_end(g)
    launches = bie.launch_count() - launches0
    if dist:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t_total = sum(step_ms) / 1e3
    if dist:
        tt = torch.tensor([t_total], dtype=torch.float64, device=dev)
        tt = tt.cpu() if args.dist_backend != "nccl" else tt
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_total = tt.item()
    # N = 1: one solve; N > 1: ONE solve sharded over the ranks (strong scaling)
    value = args.steps * pairs_per_step / t_total

    # ---- dominant kernel roofline (all-pairs phase, CUDA events on the launch stream)
    pair_ms = prof["pairs_ms"] / max(1, prof["applies"])
    # the rank's share of the N^2 pair interactions (units and diagonal blocks split evenly)
    achieved_tflops = FLOP_PER_PAIR * N * N / ws / (pair_ms * 1e-3) / 1e12
    pairs_share = prof["pairs_ms"] / sum(step_ms)

    # ---- e2e: public API with host buffers, H2D + D2H inside the timed region
    # (N = 1: bie_gmres_solve_host, the C-ABI call with pinned HOST f and x)
    e2e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk_e2e:
        for k in range(args.steps):
            flush.fill_(float(k))
            e2e_ev[k][0].record(stream)
            if ws == 1:
                bie.gmres_solve_host(g, bd, f_host, x_host, tol=1e-30, max_iter=GMRES_ITERS)
            else:
                f.copy_(f_host, non_blocking=True)
                step()
                x_host.copy_(x, non_blocking=True)
            e2e_ev[k][1].record(stream)
        torch.cuda.synchronize()
    e2e_ms_each = [a.elapsed_time(b) for a, b in e2e_ev]
    e2e_s = sum(e2e_ms_each) / 1e3
    if dist:
        tt = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        tt = tt.cpu() if args.dist_backend != "nccl" else tt
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = tt.item()

    extra = {}
    if rank == 0 and ws == 1 and not args.quick:
        # matvec-only sweep (bie_dlp_apply, BIE_FULL) and full GMRES solves
        sweep = {}
        for nvec in (1, 4, 16):
            s = torch.from_numpy(density(p, nvec=nvec).reshape(-1)).to(dev)
            o = torch.zeros_like(s)
            for _ in range(2):
                bie.dlp_apply(g, s, o, nvec)
            reps = 5 if nvec < 16 else 2
            bie.profile_begin(g)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(reps):
                bie.dlp_apply(g, s, o, nvec)
            b.record(stream)
            torch.cuda.synchronize()
            pr = bie.profile_end(g)
            ms = a.elapsed_time(b) / reps
            kms = pr["pairs_ms"] / max(1, pr["applies"])
            sweep[f"nvec{nvec}"] = {
                "ms": ms, "pairs_per_s": nvec * N * N / (ms * 1e-3), "kernel_ms": kms,
                "kernel_alg_tflops": (11 + 8 * nvec) * N * N / (kms * 1e-3) / 1e12,
                "kernel_frac_of_fp64_peak": (11 + 8 * nvec) * N * N / (kms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS}
            del s, o
        extra["matvec_sweep"] = sweep
        sol = {}
        # configs 2-3: the first call captures the iteration graph (conditional WHILE
        # node, cached on the geometry); gmres_s is the median of 3 warm solves
        for cid, mi in ((2, 1000), (3, 1000), (CONFIG_ID, args.gmres_cap)):
            pp = make_problem(cid)
            gg = g if cid == CONFIG_ID else bie.Geometry.from_problem(pp)
            torch.cuda.synchronize()
            tb = time.perf_counter()
            bdd = bd if cid == CONFIG_ID else bie.BlockDiag(gg, structured=True)
            torch.cuda.synchronize()
            tb = time.perf_counter() - tb
            ff = torch.from_numpy(rhs_pipe(pp)).to(dev)
            xx = torch.zeros_like(ff)
            reps = 1 if cid == CONFIG_ID else 4
            tss = []
            for _ in range(reps):
                torch.cuda.synchronize()
                ts = time.perf_counter()
                rr = bie.gmres_solve(gg, bdd, ff, xx, tol=1e-8, max_iter=mi)
                tss.append(time.perf_counter() - ts)
            sol[f"config{cid}"] = {"N": pp.N, "build_pc_s": tb if cid != CONFIG_ID else t_bd,
                                   "gmres_s": tss[0] if reps == 1 else statistics.median(tss[1:]),
                                   "gmres_first_call_s": tss[0],
                                   "iters": rr["iters"], "converged": rr["converged"], "max_iter": mi,
                                   "res_pc": rr["res_pc"], "res_true": rr["res_true"], "tol": 1e-8}
        extra["gmres_solve"] = sol
        # NEXT-3: the paper's three scenarios on config 3 -- pipe flow (P:l.217-227),
        # shear on all curves (P:l.634-638) and the Stokeslet/rotlet exact solution
        # (P:l.933-958) -- batched solver vs single solves; NEXT-2: the represented
        # field on a reliable interior grid and the paper's eps(x) (P:l.752-757)
        from bie_inputs import (interior_grid, node_positions, rhs_shear_all, stokeslet_rotlet_field,
                                stokeslet_rotlet_params)

        pp = make_problem(3)
        gg = bie.Geometry.from_problem(pp)
        bdd = bie.BlockDiag(gg, structured=True)
        cs_, lam_, mu_ = stokeslet_rotlet_params(pp)
        Fs = np.stack([rhs_pipe(pp), rhs_shear_all(pp),
                       stokeslet_rotlet_field(node_positions(pp), cs_, lam_, mu_).reshape(-1)])
        F = torch.from_numpy(Fs.reshape(-1).copy()).to(dev)
        X = torch.zeros_like(F)
        bie.gmres_solve_batch(gg, bdd, F, X, nrhs=3, tol=1e-8, max_iter=1000)  # warm-up
        torch.cuda.synchronize()
        tb = time.perf_counter()
        rb_ = bie.gmres_solve_batch(gg, bdd, F, X, nrhs=3, tol=1e-8, max_iter=1000)
        torch.cuda.synchronize()
        tb = time.perf_counter() - tb
        n2 = 2 * pp.N
        Xs = torch.zeros_like(F)
        ts = time.perf_counter()
        for r in range(3):
            bie.gmres_solve(gg, bdd, F[r * n2:(r + 1) * n2], Xs[r * n2:(r + 1) * n2], tol=1e-8, max_iter=1000)
        torch.cuda.synchronize()
        ts = time.perf_counter() - ts
        xs = X.cpu().numpy().reshape(3, -1, 2)
        wl = pp.M * pp.n_pore
        pts = interior_grid(pp, 400, 24)
        u = torch.zeros(pts.size, dtype=torch.float64, device=dev)
        bie.field_eval(gg, X[2 * n2:3 * n2], torch.from_numpy(pts.reshape(-1).copy()).to(dev), u)
        uu = u.cpu().numpy().reshape(-1, 2)
        uref = stokeslet_rotlet_field(pts, cs_, lam_, mu_)
        nu_, nr_ = np.linalg.norm(uu, axis=1), np.linalg.norm(uref, axis=1)
        eps_x = np.abs(nu_ - nr_) / nr_
        extra["multi_rhs"] = {
            "config": 3, "scenarios": ["pipe", "shear_all", "stokeslet_rotlet"], "nrhs": 3, "batched_s": tb,
            "sequential_s": ts, "iters": [r["iters"] for r in rb_], "all_converged": all(r["converged"] for r in rb_),
            "shear_pore_over_wall_density": float(np.abs(xs[1, :wl]).max() / np.abs(xs[1, wl:]).max()),
            "stokeslet_eps_x": {"max": float(eps_x.max()), "median": float(np.median(eps_x)), "points": int(pts.shape[0]),
                                "definition": "| |u| - |u_ref| | / |u_ref| on grid points with d(x, Gamma) > sqrt(ds) "
                                              "(P:l.752-757, P:l.355-358), tol 1e-8 solve"}}
        # NEXT-1: the paper's own single-layer operator (KR-6 corrected) on the same
        # geometry, and an SLP BD-GMRES solve on config 3
        slp = {}
        for nvec in (1, 16):
            s = torch.from_numpy(density(p, nvec=nvec).reshape(-1)).to(dev)
            o = torch.zeros_like(s)
            for _ in range(2):
                bie.slp_apply(g, s, o, nvec)
            reps = 3 if nvec == 1 else 1
            bie.profile_begin(g)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(reps):
                bie.slp_apply(g, s, o, nvec)
            b.record(stream)
            torch.cuda.synchronize()
            pr = bie.profile_end(g)
            ms = a.elapsed_time(b) / reps
            slp[f"matvec_config{CONFIG_ID}_nvec{nvec}"] = {
                "ms": ms, "pairs_per_s": nvec * N * N / (ms * 1e-3),
                "kernel_ms": pr["pairs_ms"] / max(1, pr["applies"])}
            del s, o
        pp = make_problem(3)
        gg = bie.Geometry.from_problem(pp)
        torch.cuda.synchronize()
        tb = time.perf_counter()
        bdd = bie.BlockDiag(gg, op="slp")
        torch.cuda.synchronize()
        tb = time.perf_counter() - tb
        ff = torch.from_numpy(rhs_pipe(pp)).to(dev)
        xx = torch.zeros_like(ff)
        ts = time.perf_counter()
        rr = bie.gmres_solve_slp(gg, bdd, ff, xx, tol=1e-8, max_iter=1000)
        ts = time.perf_counter() - ts
        slp["gmres_config3"] = {"build_pc_s": tb, "gmres_s": ts, "iters": rr["iters"], "converged": rr["converged"],
                                "res_true": rr["res_true"], "tol": 1e-8}
        # the structured SLP BD: pore blocks as rotating-frame circulant inverses
        torch.cuda.synchronize()
        tb = time.perf_counter()
        bds = bie.BlockDiag(gg, op="slp", structured=True)
        torch.cuda.synchronize()
        tb = time.perf_counter() - tb
        xx.zero_()
        ts = time.perf_counter()
        rr = bie.gmres_solve_slp(gg, bds, ff, xx, tol=1e-8, max_iter=1000)
        ts = time.perf_counter() - ts
        slp["gmres_config3_structured_bd"] = {"build_pc_s": tb, "gmres_s": ts, "iters": rr["iters"],
                                              "converged": rr["converged"], "res_true": rr["res_true"], "tol": 1e-8}
        extra["slp"] = slp
        if not args.no_config5:
            extra["config5_sweep"] = config5_sweep(bie, dev, stream)

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    peaks = _peaks()
    clocks = clk.summary()
    line = {
        "metric": "DLP matvec pair-interactions/s", "value": value, "unit": "pair-interactions/s", "n_gpus": ws,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": statistics.mean(step_ms),
        "step_ms_each": [round(t, 3) for t in step_ms],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config4 pipe L=100 M=1000 N={N} (2N={2 * N} unknowns), pipe BC; step = "
                               f"BD-preconditioned GMRES solve, fixed {GMRES_ITERS} iterations "
                               f"({GMRES_ITERS + 1} completed DLP matvecs + BD applies + CGS2)",
                   "N": N, "unknowns": 2 * N, "gmres_iters_per_step": GMRES_ITERS,
                   "matvecs_per_step": GMRES_ITERS + 1,
                   "parallelism": f"rows{ws} (row-sharded solve, all-gather + all-reduce over NCCL)" if ws > 1
                   else "single",
                   "l2": "flushed between timed steps (256 MiB write); BD inverses (2.67 GB) exceed L2 each step",
                   "gmres_loop": "timed steps: host-enqueued iterations (bie_profile_* per-apply events on, "
                                 "which a CUDA graph body cannot hold); e2e: the CUDA-graph conditional WHILE loop "
                                 "(one graph launch per solve)"},
        "roofline": {"kernel": ("all-pairs phase: k_dlp_sym<8,2> dual-source + k_dlp_diag (nvec=1 symmetric path)" if ws == 1
                                else "all-pairs phase on this rank's slice of the symmetric work list"),
                     "bound": "alu", "achieved": achieved_tflops,
                     "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": achieved_tflops / FP64_PEAK_TFLOPS,
                     "traffic": _ncu_traffic(), "traffic_source": "profiles/round2/k_dlp_sym_traffic.json "
                     "(dram__bytes_read.sum + dram__bytes_write.sum, ncu --set full, one launch)",
                     "peak_measured": fp64_meas, "frac_of_measured": achieved_tflops / fp64_meas,
                     "peak_measured_source": "bie_fp64_peak in this run: DFMA chains, 8 x 256-thread CTAs/SM",
                     "flop_per_pair": FLOP_PER_PAIR, "kernel_ms": pair_ms,
                     "kernel_share_of_step": pairs_share,
                     "executed_flop_per_pair": 17,
                     "ncu_fp64_pipe_active_pct": _ncu_traffic("fp64_pipe_active_pct"),
                     "ncu_fp64_pipe_source": "profiles/round2/k_dlp_sym_traffic.json (ncu capture of this kernel)",
                     "peak_source": "derived: 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz (DESIGN.md s5)"},
        "e2e": {"value": args.steps * pairs_per_step / e2e_s, "unit": "pair-interactions/s",
                "h2d_bytes_per_step": int(f_host.numel() * 8), "d2h_bytes_per_step": int(x_host.numel() * 8),
                "step_ms_each": [round(t, 3) for t in e2e_ms_each], "clocks": clk_e2e.summary()},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "setup": {"geometry_s": t_geom, "build_pc_s": t_bd},
        "hbm_peak_gbs": peaks.get("hbm_gbs"),
    }
    line.update(extra)
    if not args.no_cpu_baseline and ws == 1:
        line["cpu_baseline"] = {k: v for k, v in cpu_baseline_sample(p, seconds=args.cpu_seconds).items()
                                if k != "seconds"}
        if not args.quick:
            cg = cpu_gmres_baseline()
            it4 = extra.get("gmres_solve", {}).get(f"config{CONFIG_ID}", {}).get("iters")
            if it4:
                cg["config4"]["iters_of_gpu_solve"] = it4
                cg["config4"]["gmres_s_extrapolated"] = it4 * cg["config4"]["gmres_s_per_iteration_extrapolated"]
            line["cpu_baseline"]["gmres"] = cg
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--quick", action="store_true", help="skip the matvec sweep and full GMRES solves")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--gmres-cap", type=int, default=2000)
    ap.add_argument("--no-config5", action="store_true", help="skip the config-5 (N = 1.06M) nvec sweep")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: check the multi-rank flow with ranks sharing a GPU (not a measurement)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
