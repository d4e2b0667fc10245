# K1 warps-per-CTA variants (8 x 3 CTAs/SM vs 24 x 1 CTA/SM), env knobs read once per process.
timeout 300 python -m pytest tests/test_gpu_act_quant.py -q -x 2>&1 | tail -1
MRFP4_K1_NVWARPS=8 MRFP4_K1_MXWARPS=8 timeout 300 python -m pytest tests/test_gpu_act_quant.py -q -x 2>&1 | tail -1
for w in 24 8; do
  echo "== warps $w"
  MRFP4_K1_NVWARPS=$w MRFP4_K1_MXWARPS=$w python scripts/k1_probe.py 2>&1 | head -10
  MRFP4_K1_NVWARPS=$w WARPS=$w python scripts/k1_trace_nv.py 2048 8192 16
  MRFP4_K1_NVWARPS=$w WARPS=$w python scripts/k1_trace_nv.py 8192 8192 16
done
