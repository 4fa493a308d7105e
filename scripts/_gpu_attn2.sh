make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_attn_gpu.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
for g in 0; do echo "G=$g"; ZI_ATTN_GROUP=$g timeout 300 python scripts/bench_attn.py 2>&1 | tail -2 | head -1; done
timeout 300 python scripts/bench_attn.py 8 16 1024 128 --trace 2>&1 | head -14
