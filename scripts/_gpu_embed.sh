# embedding-lookup / position-gradient kernels: their tests, the engine parity tests, smoke, main bench arm
make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 1200 python -m pytest tests/test_embed_gpu.py tests/test_gpt_gpu.py tests/test_multiproc_gpu.py tests/test_prefetch_gpu.py -m gpu -q -p no:cacheprovider 2>&1 | tail -4
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for i in 1 2; do
  timeout 600 python bench.py --no-offload --no-nvme --no-cpu --no-config3 > gpurun_out/emb_$i.log 2> gpurun_out/emb_$i.err
  python - "$i" <<'P'
import json, sys
d = json.loads(open(f"gpurun_out/emb_{sys.argv[1]}.log").read().strip().splitlines()[-1])
print(sys.argv[1], d["value"], d["ms_per_step"], d["e2e"]["value"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d["gpu_launches"])
P
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv python scripts/profile_step.py --graph > gpurun_out/launches_emb.csv 2>/dev/null; wc -l gpurun_out/launches_emb.csv
