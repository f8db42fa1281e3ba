for i in 1 2; do timeout 600 python bench.py --quick --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['step_ms_each'], d['roofline']['kernel_ms'], d['clocks'])"; done
python tools/probe_step_gap.py 2>&1 | head -8
