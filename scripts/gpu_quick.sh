#!/bin/bash
# Quick GPU pass: full GPU tests, smoke, bench lines for all configs (no ncu).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --steps 300 2>/dev/null | tee gpurun_out/bench_c1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', d['value'], d['ms_per_step'], d.get('speedup_vs_cublas_bf16'), d['roofline_k1']['frac'] if 'roofline_k1' in d else '', d['roofline']['frac'])"
for c in c0 c2-up-nv c2-down-mx c3-gateup; do
  timeout 300 python bench.py --config $c --steps 200 --no-cpu-baseline --no-e2e --no-sustained --no-comparators 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['ms_per_step'], d.get('speedup_vs_cublas_bf16'), d.get('roofline_k1',{}).get('frac'), d['roofline']['frac'])"
done
