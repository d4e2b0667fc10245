#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_case.py (small shapes).
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
    python scripts/sanitize_case.py > gpurun_out/r02_sanitizer_$tool.log 2>&1
  echo "$tool exit $?"; tail -4 gpurun_out/r02_sanitizer_$tool.log
done
