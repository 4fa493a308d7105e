make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_fused_gpu.py tests/test_gpt_gpu.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -1
timeout 300 python scripts/bench_fused.py 2>&1
