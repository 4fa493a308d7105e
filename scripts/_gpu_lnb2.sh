make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
ZI_LNB_NT=256 timeout 900 python -m pytest tests/test_fused_gpu.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
for n in 512 256; do echo "NT=$n"; ZI_LNB_NT=$n timeout 300 python scripts/bench_fused.py 2>&1 | grep ln_; done
