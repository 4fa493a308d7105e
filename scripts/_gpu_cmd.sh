make -j8 >/dev/null 2>&1
for i in 1 2; do timeout 900 python -m pytest tests/test_multiproc_gpu.py -m gpu -q 2>&1 | tail -1; done
timeout 900 python -m pytest tests/test_gpt_gpu.py -m gpu -q 2>&1 | tail -1
