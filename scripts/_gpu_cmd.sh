L=paper_2104_07857_b200/libzinf.so
cp $L /tmp/new.so
for rep in 1 2; do
cp build_ab/libzinf_old.so $L; echo old; timeout 300 python scripts/bench_fused.py 2>&1 | grep -i "ln_bwd"
cp /tmp/new.so $L; echo new; timeout 300 python scripts/bench_fused.py 2>&1 | grep -i "ln_bwd"
done
timeout 600 python -m pytest tests/test_fused_gpu.py tests/test_gpt_gpu.py -q -m gpu 2>&1 | tail -2
