mkdir -p gpurun_out/parts
(OMP_NUM_THREADS=14 nice -n 15 python tools/make_golden.py config4_bd_pipe_full --run 1 > gpurun_out/parts/run1.log 2>&1; cp tests/golden/parts/config4_bd_pipe_full.run1.json gpurun_out/parts/) &
GP=$!
{
python tools/probe_bd4.py 4
BIE_BD_LOOKAHEAD=0 python tools/probe_bd4.py 4
BIE_BD_LOOKAHEAD=0 BIE_BD_AGGK=0 python tools/probe_bd4.py 4
BIE_BD_AGG=0 python tools/probe_bd4.py 4
python tools/probe_bd4.py 3
} > gpurun_out/bd_probe_s6.log 2>&1
timeout 900 python -m pytest tests/test_gpu_bd_gmres.py tests/test_gpu_bd_structured.py -m gpu -x -q > gpurun_out/bd_tests_s6.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bd_factor_s6.csv python tools/probe_bd4.py 4 --once > gpurun_out/ncu_bd_s6.log 2>&1
cat gpurun_out/bd_probe_s6.log; tail -3 gpurun_out/bd_tests_s6.log
wait $GP
tail -2 gpurun_out/parts/run1.log
