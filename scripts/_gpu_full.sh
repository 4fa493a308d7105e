# round-end style: store differential on the GPU path, full default bench (all legs), launch list of the graphed step
make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_store.py -m gpu -q -p no:cacheprovider 2>&1 | tail -3
T0=$(date +%s); timeout 2400 python bench.py > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err; echo "bench wall $(( $(date +%s) - T0 )) s"
: timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv python scripts/profile_step.py --graph > gpurun_out/launches_r2.csv 2>/dev/null; wc -l gpurun_out/launches_r2.csv
timeout 300 python scripts/bench_attn.py 2>&1 | tail -3
timeout 300 python scripts/bench_attn.py 8 16 1024 128 --trace 2>&1 | head -14
