#!/bin/bash
# K2 iteration check: GEMM parity tests, K2 timeline (trace build), bench lines for the 2-CTA configs.
tag=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_fullsize.py tests/test_gpu_configs.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/${tag}_pytest.log
for c in c2-up-nv c1 c2-down-mx; do MRFP4_LIB=build/trace/libmrfp4.so timeout 120 python scripts/k2_timeline.py $c; done > gpurun_out/${tag}_timeline.txt 2>&1
for c in c1 c2-up-nv c2-down-mx c3-gateup; do timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-sustained --no-comparators >> gpurun_out/${tag}_bench.jsonl 2>>gpurun_out/${tag}_bench.err; done
cat gpurun_out/${tag}_pytest.log gpurun_out/${tag}_timeline.txt
python - "$tag" <<'PY'
import json, sys
for l in open(f"gpurun_out/{sys.argv[1]}_bench.jsonl"):
    d = json.loads(l)
    print(d['config']['workload'][:40], round(d['value']), 'k1 %.1f k2 %.1f' % (d['k1_us'], d['k2_us']),
          'spd %.2f' % d['speedup_vs_cublas_bf16'], 'k2frac %.3f k1frac %.3f' % (d['roofline']['frac'], d['roofline_k1']['frac']),
          d['clocks']['sm_mhz'])
PY
