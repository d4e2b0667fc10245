#!/bin/bash
# Evidence pass after the split-K / pre-wait weight-load changes to the 1-CTA GEMM: tests, smoke,
# bench (all configs + reference arm), ncu launch lists (c1, c0) and a full capture of K2 at c0.
# The 2-CTA GEMM and K1 are unchanged since r01l (their full captures stand).
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
for c in c0 c2-up-nv c2-down-mx c3-gateup; do
  timeout 300 python bench.py --config $c --steps 200 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 200 python scripts/decode_probe.py > gpurun_out/decode_probe.txt 2>&1
for cfg in c1 c0; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/launches_$cfg.csv python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-sustained --no-comparators > gpurun_out/ncu_launch_$cfg.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 3 -c 1 -f -o gpurun_out/prof_k_gemm_c0 \
  python bench.py --config c0 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-sustained --no-comparators > gpurun_out/ncu_k_gemm_c0.log 2>&1
ncu -i gpurun_out/prof_k_gemm_c0.ncu-rep --page details --csv > gpurun_out/prof_k_gemm_c0_details.csv 2>/dev/null
rm -f gpurun_out/prof_k_gemm_c0.ncu-rep
ls -la gpurun_out
