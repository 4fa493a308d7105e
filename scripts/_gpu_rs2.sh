make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
for v in 0 1; do echo "ILP=$v"; ZI_RS_ILP=$v timeout 300 python scripts/bench_rs_adam.py 2>&1 | head -1; done
for r in 1 2; do for v in 0 1; do ZI_RS_ILP=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-offload --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ILP=$v', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['roofline']['frac'], d['roofline']['avg_launch_ms'])"; done; done
