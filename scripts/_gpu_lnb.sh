# split LayerNorm backward: tests, kernel roofline A/B vs the legacy kernel, step A/B
make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_fused_gpu.py tests/test_gpt_gpu.py tests/test_gemm_sk_gpu.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -4
for L in 0 1; do echo "legacy=$L"; ZI_LN_BWD_LEGACY=$L timeout 300 python scripts/bench_fused.py 2>&1 | grep -i "ln_bwd\|ln_fwd"; done
for r in 1 2; do for L in 1 0; do ZI_LN_BWD_LEGACY=$L timeout 600 python bench.py --steps 20 --warmup 5 --no-offload --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('legacy=$L', d['value'], d['ms_per_step'], d['clocks'])"; done; done
