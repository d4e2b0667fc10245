for coop in 1 0; do for pdl in 1 0; do
  MRFP4_COOP=$coop MRFP4_PDL=$pdl timeout 300 python bench.py --config c0 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-sustained --no-comparators 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('coop $coop pdl $pdl', 'K1 %.1f K2 %.1f step %.1f us spd %.2f' % (d['k1_us'], d['k2_us'], d['ms_per_step']*1e3, d['speedup_vs_cublas_bf16']))"
done; done
