#!/bin/bash
# Fused decode kernel (default) vs the two-kernel path (MRFP4_DECODE=0) at decode shapes
for d in 1 0; do
  for cm in "c0 16" "c0 1" "c2-up-nv 1" "c2-up-nv 16" "c2-down-mx 16" "c1 16" "c2-up-mx 32"; do
    set -- $cm
    MRFP4_DECODE=$d timeout 300 python bench.py --config $1 --M $2 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-sustained --no-comparators 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('decode=$d', '$1 M=$2'.ljust(16), 'step %.1f us bf16 %.1f spd %.2f roof %s %.3f' % (d['ms_per_step']*1e3, d['bf16_cublas_us'], d['speedup_vs_cublas_bf16'], d['roofline']['kernel'][:16], d['roofline']['frac']))"
  done
done
