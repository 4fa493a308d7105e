make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 300 python scripts/gemm_sustained.py 8192 8192 2048
timeout 300 python scripts/gemm_sustained.py 8192 2048 8192
