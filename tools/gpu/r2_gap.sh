python tools/probe_step_gap.py > gpurun_out/step_gap.json 2>&1; cat gpurun_out/step_gap.json
