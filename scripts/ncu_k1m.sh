#!/bin/bash
# ncu --set full of K1m (c1 MXFP4, c2-up NVFP4) + per-warp traces; large files removed.
mkdir -p gpurun_out
for cfg in c1 c2-up-nv; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_act_quant -s 3 -c 1 -f -o gpurun_out/prof_k1m_$cfg \
    python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-sustained --no-comparators > /dev/null 2>&1
  ncu -i gpurun_out/prof_k1m_$cfg.ncu-rep --page details --csv > gpurun_out/prof_k1m_${cfg}_details.csv 2>/dev/null
  ncu -i gpurun_out/prof_k1m_$cfg.ncu-rep --page source --csv > gpurun_out/prof_k1m_${cfg}_source.csv 2>/dev/null
  rm -f gpurun_out/prof_k1m_$cfg.ncu-rep
done
WARPS=8 python scripts/k1_trace_nv.py 2048 8192 16
WARPS=8 python scripts/k1_trace.py 2048 14336 0 32
