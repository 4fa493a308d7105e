# power-capped sustained TFLOPS of zi_gemm_sk: clusters of 2 (no multicast) vs 4 (A multicast)
make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
for cl in 2 4 2 4; do
  echo "CL=$cl"
  ZI_SK_CL=$cl timeout 120 python scripts/gemm_sustained.py 8192 8192 2048 2>/dev/null | head -1
  ZI_SK_CL=$cl timeout 120 python scripts/gemm_sustained.py 8192 2048 8192 2>/dev/null | head -1
done
