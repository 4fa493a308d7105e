# ncu --set full of every zi_gemm_sk launch of one (2-layer) 1.3B-shape engine step:
# per-launch DRAM traffic for bench.py's tensor roofline (profiles/ncu_traffic.json)
make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 900 ncu --set full --clock-control none --profile-from-start off -k regex:gemm_sk_kernel \
  -o /tmp/step_gemm_full python scripts/profile_step.py --nl 2 > gpurun_out/step_gemm_full.log 2>&1
tail -3 gpurun_out/step_gemm_full.log
ncu -i /tmp/step_gemm_full.ncu-rep --page raw --csv \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  > gpurun_out/step_gemm_full.csv 2>/dev/null
wc -l gpurun_out/step_gemm_full.csv
