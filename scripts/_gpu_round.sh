# full GPU suite, smoke, bench, and the ncu launch list of the bench's step
make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x 2>&1 | tail -15 > gpurun_out/gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
tail -5 gpurun_out/gputest.log; tail -2 gpurun_out/smoke.log
python - <<'P'
import json
d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1])
print({k: d.get(k) for k in ('value','ms_per_step','e2e','gpu_launches','clocks')})
print(d.get('roofline'))
for k,v in d.get('gemm_sites',{}).items(): print(k, v)
P
