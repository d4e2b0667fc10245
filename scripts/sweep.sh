#!/bin/bash
# Token sweep at the Llama-3-70B shapes (BASELINE.json configs[2]): one bench line per (shape, M).
mkdir -p gpurun_out
for c in c2-up-nv c2-down-mx; do
  for M in ${MS:-1 16 128 512 1024 2048 4096 8192}; do
    timeout 300 python bench.py --config $c --M $M --steps 100 --no-cpu-baseline --no-e2e --no-sustained --no-comparators 2>/dev/null | tee -a gpurun_out/sweep.jsonl | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', $M, round(d['ms_per_step']*1e3,1), round(d['value']), round(d['speedup_vs_cublas_bf16'],3), round(d['k1_us'],1), round(d['k2_us'],1), round(d['bf16_cublas_us'],1), round(d['roofline']['frac'],3))"
  done
done
