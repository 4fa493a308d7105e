make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 1200 python -m pytest tests/test_attn_gpu.py tests/test_gpt_gpu.py tests/test_fused_gpu.py tests/test_multiproc_gpu.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
ZI_LNB_NT=256 timeout 900 python -m pytest tests/test_fused_gpu.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -1
for n in 512 256; do echo "NT=$n"; ZI_LNB_NT=$n timeout 300 python scripts/bench_fused.py 2>&1 | grep ln_bwd; done
bash scripts/_gpu_ab.sh ZI_EPI_AUX "0 1" 2
