# LayerNorm backward with the row statistics prefetched a stage ahead: tests, kernel timing, step
make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_fused_gpu.py tests/test_gpt_gpu.py -m gpu -q -p no:cacheprovider 2>&1 | tail -2
for r in 1 2; do timeout 300 python scripts/bench_fused.py 2>&1 | grep ln_bwd; done
timeout 600 ncu --set full --clock-control none -k regex:"ln_bwd_split" -s 2 -c 1 -o gpurun_out/lnb_ncu2 python scripts/bench_fused.py > /dev/null 2>&1
ncu -i gpurun_out/lnb_ncu2.ncu-rep --page raw --csv > gpurun_out/lnb_raw2.csv 2>/dev/null
for r in 1 2; do
  timeout 600 python bench.py --no-offload --no-nvme --no-cpu --no-config3 > gpurun_out/lnpf_$r.log 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/lnpf_$r.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks']['sm_mhz'])"
done
