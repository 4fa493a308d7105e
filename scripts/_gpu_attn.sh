# attention: tests, kernel timing vs cuDNN, trace, step bench
make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_attn_gpu.py tests/test_gpt_gpu.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
timeout 300 python scripts/bench_attn.py 2>&1 | tail -3
timeout 300 python scripts/bench_attn.py 8 16 1024 128 --trace 2>&1 | head -14
for r in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 --no-offload --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"; done
