make -j8 >/dev/null 2>&1
timeout 300 python scripts/diag_ac9.py 2>&1 | tail -6
CUBLAS_WORKSPACE_CONFIG=:4096:8 timeout 300 python scripts/diag_ac9.py 2>&1 | tail -5
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_harness_gpu.py tests/test_gpt_gpu.py tests/test_cli.py -m gpu -q 2>&1 | tail -4
timeout 900 python scripts/ab_config5.py 0:12 3:12 2:12 3:16 4:12 2>&1 | grep -v Warn | tail -8
