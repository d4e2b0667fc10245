#!/bin/bash
# Round-2 final evidence pass: tests, smoke, bench lines for every config (+ reference arm),
# the 70B token sweep, ncu launch list and full captures of K1 / K2 at c1 and c2-up-nv.
mkdir -p gpurun_out
NB="--no-cpu-baseline --no-e2e --no-sustained --no-comparators"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02f_gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02f_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02f_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02f_smoke.log
timeout 900 python bench.py > gpurun_out/r02f_bench_c1.json 2> gpurun_out/r02f_bench_c1.err
for c in c0 c2-up-nv c2-up-mx c2-down-nv c2-down-mx c3-gateup; do
  timeout 600 python bench.py --config $c --steps 200 --no-cpu-baseline --no-sustained > gpurun_out/r02f_bench_$c.json 2> gpurun_out/r02f_bench_$c.err
done
timeout 900 python bench.py --impl reference > gpurun_out/r02f_bench_ref.json 2> gpurun_out/r02f_bench_ref.err
timeout 1500 bash scripts/sweep70b.sh r02f > gpurun_out/r02f_sweep.txt 2>&1
for cfg in c1 c2-up-nv; do
  for kk in k_gemm k_act_quant; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kk -s 3 -c 1 -f -o gpurun_out/prof_${kk}_$cfg \
      python bench.py --config $cfg --steps 3 --warmup 3 $NB > gpurun_out/r02f_ncu_${kk}_$cfg.log 2>&1
    ncu -i gpurun_out/prof_${kk}_$cfg.ncu-rep --page details --csv > gpurun_out/r02f_ncu_${kk}_${cfg}_details.csv 2>/dev/null
    rm -f gpurun_out/prof_${kk}_$cfg.ncu-rep
  done
done
ls -la gpurun_out | tail -40
