make -j8 >/dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err; echo bench $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_final.csv python scripts/profile_step.py --graph > /dev/null 2>&1; echo ncu $?
