nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/fp64_mix2.cu -o /tmp/fp64_mix2 && MIX2_CHAINS_ONLY=1 /tmp/fp64_mix2 > gpurun_out/fp64_mix2_chains.txt 2>&1
cat gpurun_out/fp64_mix2_chains.txt
