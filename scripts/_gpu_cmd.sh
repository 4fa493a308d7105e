make -j8 >/dev/null 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests $?; tail -2 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_s3b.json 2> gpurun_out/bench_s3b.err; echo bench $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_s3b.csv python scripts/profile_step.py --graph > /dev/null 2>&1; echo ncu $?
