# round-2 re-entry check: full GPU suite, smoke, bench
make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider -rf 2>&1 | tail -40 > gpurun_out/gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
tail -12 gpurun_out/gputest.log; tail -2 gpurun_out/smoke.log
python - <<'P'
import json
d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1])
print({k: d.get(k) for k in ('value','ms_per_step','e2e','gpu_launches','clocks')})
print(d.get('roofline'))
print(json.dumps(d.get('offload'))[:1500])
P
