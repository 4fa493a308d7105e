# full GPU suite + smoke + full default bench + launch list + the N=2 (same-GPU) path
make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
T0=$(date +%s); timeout 2400 python bench.py > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err; echo "bench wall $(( $(date +%s) - T0 )) s"
python - <<'P'
import json
d=json.loads(open('gpurun_out/bench_full.log').read().strip().splitlines()[-1])
print({k: d.get(k) for k in ('value','ms_per_step','e2e','gpu_launches','clocks')})
print(d.get('roofline'))
o=d.get('offload') or {}
for k in ('config3_real','nvme_params','config3_equiv','config5_equiv'):
    v=o.get(k) or {}
    print(k, {x: v.get(x) for x in ('ms_per_step_offload','ms_per_step_nvme','hidden_fraction','tflops_offload','skipped','error')})
P
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv python scripts/profile_step.py --graph > gpurun_out/launches_final.csv 2>/dev/null; wc -l gpurun_out/launches_final.csv
timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-offload --no-nvme --no-cpu --no-config3 > gpurun_out/bench_2rank.log 2> gpurun_out/bench_2rank.err; tail -c 600 gpurun_out/bench_2rank.log
