#!/bin/bash
# One GPU-box evidence pass: tests, smoke, bench (all configs + reference arm + 70B token sweep),
# ncu launch list + full captures of K1 and K2 (reports reduced to CSV; .ncu-rep removed).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
for c in c0 c2-up-nv c2-down-mx c3-gateup; do
  timeout 300 python bench.py --config $c --steps 200 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
rm -f gpurun_out/sweep.jsonl; timeout 900 bash scripts/sweep.sh > gpurun_out/sweep.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/launches_c1.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-sustained --no-comparators > gpurun_out/ncu_launch.log 2>&1
for cfg in c1 c2-up-nv; do
  for kk in k_gemm k_act_quant; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kk -s 3 -c 1 -f -o gpurun_out/prof_${kk}_$cfg \
      python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-sustained --no-comparators > gpurun_out/ncu_${kk}_$cfg.log 2>&1
    ncu -i gpurun_out/prof_${kk}_$cfg.ncu-rep --page details --csv > gpurun_out/prof_${kk}_${cfg}_details.csv 2>/dev/null
    ncu -i gpurun_out/prof_${kk}_$cfg.ncu-rep --page raw --csv > gpurun_out/prof_${kk}_${cfg}_raw.csv 2>/dev/null
    rm -f gpurun_out/prof_${kk}_$cfg.ncu-rep
  done
done
ls -la gpurun_out
