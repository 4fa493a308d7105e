make -j8 >/dev/null 2>&1
timeout 900 python -m pytest tests/test_fullsize_gpu.py -m gpu -q -k "config5" --durations=5 2>&1 | tail -12
