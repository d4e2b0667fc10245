#!/bin/bash
# Round-2 decode evidence: ncu launch lists (c1, c0), one --set full capture of k_linear_decode at
# c0 (reduced to CSV), the sanitizer pass over every kernel family (incl. the decode kernel).
mkdir -p gpurun_out
NB="--no-cpu-baseline --no-e2e --no-sustained --no-comparators"
for cfg in c1 c0; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/r02_launches_$cfg.csv python bench.py --config $cfg --steps 5 --warmup 3 $NB > gpurun_out/r02_ncu_launch_$cfg.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_linear_decode -s 3 -c 1 -f -o gpurun_out/prof_kd_c0 \
  python bench.py --config c0 --steps 3 --warmup 3 $NB > gpurun_out/r02_ncu_kd_c0.log 2>&1
ncu -i gpurun_out/prof_kd_c0.ncu-rep --page details --csv > gpurun_out/r02_ncu_k_linear_decode_c0_details.csv 2>/dev/null
ncu -i gpurun_out/prof_kd_c0.ncu-rep --page raw --csv > gpurun_out/r02_ncu_k_linear_decode_c0_raw.csv 2>/dev/null
rm -f gpurun_out/prof_kd_c0.ncu-rep
bash scripts/sanitize.sh
