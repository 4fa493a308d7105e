make -j8 >/dev/null 2>&1
L=paper_2104_07857_b200/libzinf.so
cp $L /tmp/new.so
echo EW8; timeout 300 python scripts/bench_gemm_adam.py 2>&1 | tail -1
cp build_ab/lib_ew16.so $L
timeout 600 python -m pytest tests/test_gemm_gpu.py -m gpu -q -k gemm_adam 2>&1 | tail -1
echo EW16; timeout 300 python scripts/bench_gemm_adam.py 2>&1 | tail -5
cp /tmp/new.so $L
