# GEMM side outputs (fc1 bias colsum, attention delta): tests, step A/B; copy-size probe; ncu of LN kernels
make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 1200 python -m pytest tests/test_gemm_sk_gpu.py tests/test_attn_gpu.py tests/test_gpt_gpu.py tests/test_multiproc_gpu.py tests/test_fused_gpu.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -4
timeout 300 python scripts/copy_probe.py
for r in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 --no-offload --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('run', d['value'], d['ms_per_step'], d['clocks'], d['gpu_launches'])"; done
timeout 600 ncu --set full --clock-control none -k regex:"ln_bwd_split|ln_fwd_warp" -s 4 -c 2 -o gpurun_out/ln_ncu python scripts/bench_fused.py > /dev/null 2>&1; ls gpurun_out/ | grep ncu
