timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_gemm.py tests/test_gpu_configs.py -q -x 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -7
timeout 200 bash scripts/decode_ab.sh 2>&1 | head -2
