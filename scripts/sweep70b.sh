#!/bin/bash
# Llama-3-70B shapes x {NVFP4, MXFP4} x token sweep (BASELINE.json configs[2]): one bench line each.
tag=${1:-sweep}
mkdir -p gpurun_out
out=gpurun_out/${tag}_sweep_70b.jsonl
: > $out
for c in c2-up-nv c2-up-mx c2-down-nv c2-down-mx; do
  for m in ${MS:-1 16 128 512 1024 2048 4096 8192}; do
    timeout 300 python bench.py --config $c --M $m --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-sustained --no-comparators >> $out 2>/dev/null
  done
done
python - $out <<'PY'
import json, sys
print(f"{'shape':10s} {'fmt':6s} {'M':>5s} {'K1 us':>7s} {'K2 us':>7s} {'step us':>8s} {'bf16 us':>8s} {'speedup':>7s} {'K2 frac':>7s}")
for l in open(sys.argv[1]):
    d = json.loads(l); c = d['config']
    shape = 'up' if c['K'] == 8192 else 'down'
    print(f"{shape:10s} {c['format']:6s} {c['M']:5d} {d['k1_us']:7.1f} {d['k2_us']:7.1f} {d['ms_per_step']*1e3:8.1f} "
          f"{d['bf16_cublas_us']:8.1f} {d['speedup_vs_cublas_bf16']:7.2f} {d['roofline']['frac']:7.3f}")
PY
