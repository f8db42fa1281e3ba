# FP64 mix microbenchmark + symmetric-kernel variant timings (config 4)
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/fp64_mix2.cu -o /tmp/fp64_mix2 && /tmp/fp64_mix2 > gpurun_out/fp64_mix2.txt 2>&1
cat gpurun_out/fp64_mix2.txt
for v in 0 3 4 5 8 9 1 6 7; do BIE_SYM_VARIANT=$v timeout 120 python tools/probe_symv.py 4; done > gpurun_out/symv_r2.txt 2>&1
cat gpurun_out/symv_r2.txt
