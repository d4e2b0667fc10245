# K1 ring-depth sweep: rebuild act_quant.o with -DMRFP4_K1_STAGES=S on the box, then probe.
for st in ${STAGES:-2 4 3}; do
  rm -f build/obj/act_quant.o; make EXTRA=-DMRFP4_K1_STAGES=$st > /dev/null 2>&1
  echo "== stages $st"
  timeout 300 python -m pytest tests/test_gpu_act_quant.py -q -x 2>&1 | tail -1
  python scripts/k1_probe.py 2>&1 | head -8
  python scripts/k1_trace.py 2048 14336 0 32 2>/dev/null | head -6
done
