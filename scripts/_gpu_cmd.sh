make -j8 >/dev/null 2>&1
timeout 600 python -m pytest tests/test_gemm_gpu.py -m gpu -q -k gemm_adam 2>&1 | tail -2
timeout 300 python scripts/bench_gemm_adam.py 2>&1 | tail -5
