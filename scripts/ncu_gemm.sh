#!/bin/bash
# ncu --set full of the GEMM on a bench config: scripts/ncu_gemm.sh <config> <tag>
cfg=${1:-c1}; tag=${2:-k2}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 3 -c 1 -f -o gpurun_out/prof_${tag}_${cfg} \
  python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-sustained --no-comparators > gpurun_out/ncu_${tag}_${cfg}.log 2>&1
ncu -i gpurun_out/prof_${tag}_${cfg}.ncu-rep --page details --csv > gpurun_out/prof_${tag}_${cfg}_details.csv 2>/dev/null
ncu -i gpurun_out/prof_${tag}_${cfg}.ncu-rep --page source --csv > gpurun_out/prof_${tag}_${cfg}_source.csv 2>/dev/null
ncu -i gpurun_out/prof_${tag}_${cfg}.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_${cfg}_raw.csv 2>/dev/null
