#!/bin/bash
# ncu launch list (c1) + --set full of K1 and K2 at c1; CSV only.
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/launches_c1.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-sustained --no-comparators > gpurun_out/ncu_launch.log 2>&1
for kk in k_gemm k_act_quant; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kk -s 3 -c 1 -f -o gpurun_out/prof_${kk}_c1 \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-sustained --no-comparators > gpurun_out/ncu_${kk}_c1.log 2>&1
  ncu -i gpurun_out/prof_${kk}_c1.ncu-rep --page details --csv > gpurun_out/prof_${kk}_c1_details.csv 2>/dev/null
  ncu -i gpurun_out/prof_${kk}_c1.ncu-rep --page raw --csv > gpurun_out/prof_${kk}_c1_raw.csv 2>/dev/null
  rm -f gpurun_out/prof_${kk}_c1.ncu-rep
done
