# preferred-cluster-4 stream-K GEMM: correctness under ZI_SK_CL=4, then full-step A/B (interleaved)
make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
ZI_SK_CL=4 timeout 900 python -m pytest tests/test_gemm_sk_gpu.py tests/test_gpt_gpu.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -4
for r in 1 2; do for v in 2 4; do ZI_SK_CL=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-offload --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('CL=$v', d['value'], d['ms_per_step'], d['clocks'])"; done; done
for v in 2 4; do ZI_SK_CL=$v timeout 600 python scripts/bench_gemm_sk.py 2>&1 | tail -3; done
