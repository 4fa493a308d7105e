make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests/test_gemm_sk_gpu.py tests/test_gpt_gpu.py tests/test_multiproc_gpu.py tests/test_prefetch_gpu.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
python scripts/epi_probe.py
bash scripts/_gpu_ab.sh ZI_EPI_AUX "0 1" 2
