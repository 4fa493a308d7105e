# deferred block folds: their tests, engine invariance tests, smoke, interleaved A/B of the main arm
make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests/test_fused_gpu.py tests/test_gpt_gpu.py tests/test_multiproc_gpu.py tests/test_prefetch_gpu.py tests/test_fullsize_gpu.py -m gpu -q -p no:cacheprovider 2>&1 | tail -4
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for r in 1 2 3; do for d in 1 0; do
  ZI_FOLD_DEFER=$d timeout 600 python bench.py --no-offload --no-nvme --no-cpu --no-config3 > gpurun_out/fold_${d}_$r.log 2> gpurun_out/fold_${d}_$r.err
  python - "$d" "$r" <<'P'
import json, sys
d = json.loads(open(f"gpurun_out/fold_{sys.argv[1]}_{sys.argv[2]}.log").read().strip().splitlines()[-1])
print("defer", sys.argv[1], "round", sys.argv[2], d["value"], d["ms_per_step"], d["e2e"]["value"], d["clocks"]["sm_mhz"], d["gpu_launches"])
P
done; done
