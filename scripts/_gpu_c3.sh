# config-3 real 10B leg + test; step breakdown zi vs cublas; cluster-4 A/B in the full step
make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
free -g | tee gpurun_out/free.txt; nproc
timeout 900 python -m pytest tests/test_fullsize_gpu.py -m gpu -q -p no:cacheprovider -k "10b_offloaded or 1p3b_offloaded" 2>&1 | tail -5 | tee gpurun_out/t10b.log
timeout 1200 python bench.py --leg config3_real --steps 3 --warmup 3 > gpurun_out/c3.log 2>&1; tail -c 2500 gpurun_out/c3.log
timeout 300 python scripts/step_gaps.py > gpurun_out/gaps_zi.txt 2>&1; head -30 gpurun_out/gaps_zi.txt
ZI_GEMM_SELECT=cublas timeout 300 python scripts/step_gaps.py > gpurun_out/gaps_cublas.txt 2>&1; head -30 gpurun_out/gaps_cublas.txt
for v in 2 4; do ZI_SK_CL=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-offload --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('CL=$v', d['value'], d['ms_per_step'], d['clocks'])"; done
