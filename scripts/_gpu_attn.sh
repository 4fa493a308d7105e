make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
ZI_ATTN_ALT=1 timeout 900 python -m pytest tests/test_attn_gpu.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -1
for r in 1 2; do for a in 0 1; do echo "ALT=$a"; ZI_ATTN_ALT=$a timeout 300 python scripts/bench_attn.py 2>&1 | tail -3 | head -2 | tail -1; done; done
ZI_ATTN_ALT=1 timeout 300 python scripts/bench_attn.py 8 16 1024 128 --trace2 2>&1 | head -16
