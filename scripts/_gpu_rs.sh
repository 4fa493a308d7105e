make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
ZI_RS_ILP=1 timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_fullsize_gpu.py -m gpu -q -p no:cacheprovider -x -k "rs_adam or adam" 2>&1 | tail -1
for r in 1 2; do for v in 0 1; do echo "ILP=$v"; ZI_RS_ILP=$v timeout 300 python scripts/bench_rs_adam.py 2>&1 | head -1; done; done
