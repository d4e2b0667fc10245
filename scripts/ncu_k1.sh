#!/bin/bash
# ncu --set full of K1 at the bench configs: scripts/ncu_k1.sh <tag> [configs...]
tag=${1:-k1}; shift
cfgs=${@:-c1 c2-up-nv c0}
mkdir -p gpurun_out
for cfg in $cfgs; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_act_quant -s 3 -c 1 -f -o gpurun_out/prof_${tag}_$cfg \
    python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-sustained --no-comparators > /dev/null 2>&1
  ncu -i gpurun_out/prof_${tag}_$cfg.ncu-rep --page details --csv > gpurun_out/prof_${tag}_${cfg}_details.csv 2>/dev/null
  ncu -i gpurun_out/prof_${tag}_$cfg.ncu-rep --page source --csv > gpurun_out/prof_${tag}_${cfg}_source.csv 2>/dev/null
  ncu -i gpurun_out/prof_${tag}_$cfg.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_${cfg}_raw.csv 2>/dev/null
  [ "${KEEP_REP:-0}" = 1 ] || rm -f gpurun_out/prof_${tag}_$cfg.ncu-rep
done
