#!/bin/bash
# per-launch durations + SM active cycles of one bench config: scripts/ncu_launches.sh <config>
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_active.max,gpc__cycles_elapsed.max --clock-control none -c 40 --csv --log-file gpurun_out/launches_$1.csv \
  python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-sustained --no-comparators > /dev/null 2>&1
