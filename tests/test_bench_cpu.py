"""CPU checks of bench.py's command-line contract (no GPU needed):
the reference arm (the CPU oracle, `--impl reference`) prints one JSON line with
the keys the driver reads; non-zero ranks of a multi-rank reference run print
nothing and exit 0; our arm fails loudly without a GPU (no CPU fallback)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra, timeout):
    env = dict(os.environ)
    env.update(env_extra)
    env.setdefault("OMP_NUM_THREADS", "4")
    return subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, env=env, capture_output=True, text=True,
                          timeout=timeout)


def test_reference_arm_json_line():
    r = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"], {}, 600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"] == "DLP matvec pair-interactions/s" and d["unit"] == "pair-interactions/s"
    assert d["value"] > 0 and d["higher_is_better"] is True and d["dtype"] == "f64"
    assert d["steps"] == 1 and d["n_gpus"] == 1 and d["vs_baseline"] is None
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] == d["value"] and cb["cores"] >= 1 and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["N"] == 136192  # BASELINE.json configs[3]: the bench workload


def test_reference_arm_nonzero_rank_is_silent():
    r = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"], {"WORLD_SIZE": "2", "RANK": "1"}, 120)
    assert r.returncode == 0 and r.stdout.strip() == ""


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="a GPU is present")
def test_our_arm_fails_loudly_without_gpu():
    r = _run(["--steps", "1", "--warmup", "3"], {}, 300)
    assert r.returncode != 0
    assert not any(ln.startswith("{") for ln in r.stdout.splitlines())
