#!/bin/bash
# bench lines (K1/K2 us, speedup) for the default build and each build/var_*/libmrfp4.so
cfgs=${CFGS:-c1 c2-up-nv c2-down-mx}
for lib in "" build/var_*/libmrfp4.so; do
  for c in $cfgs; do
    MRFP4_LIB=$lib timeout 300 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-sustained --no-comparators 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-default}'.ljust(34), '$c'.ljust(11), 'K1 %.1f K2 %.1f step %.1f us spd %.2f k2frac %.3f' % (d['k1_us'], d['k2_us'], d['ms_per_step']*1e3, d['speedup_vs_cublas_bf16'], d['roofline']['frac']))"
  done
done
