make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 1200 python -m pytest tests/test_prefetch_gpu.py tests/test_multiproc_gpu.py tests/test_gpt_gpu.py -q -p no:cacheprovider -rf -x 2>&1 | tail -25
for i in 1 2 3 4 5 6; do timeout 300 python -m pytest tests/test_cli.py -m gpu -q -p no:cacheprovider 2>&1 | tail -1; done
