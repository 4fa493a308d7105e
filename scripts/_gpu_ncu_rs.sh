# fused RS + Adam (zi_rs_adam_dc, K=1 as at N=1): warm timing, then ncu --set full with source
make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 300 python scripts/bench_rs_adam.py 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rs_kernel" -s 2 -c 1 \
  -o gpurun_out/rs_ncu python scripts/bench_rs_adam.py > gpurun_out/rs_ncu.log 2>&1; ls gpurun_out/rs_ncu*
ncu -i gpurun_out/rs_ncu.ncu-rep --page raw --csv > gpurun_out/rs_raw.csv 2>/dev/null
ncu -i gpurun_out/rs_ncu.ncu-rep --page source --csv --print-source sass > gpurun_out/rs_source.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ln_fwd_warp" -s 2 -c 1 \
  -o gpurun_out/lnf_ncu python scripts/bench_fused.py > /dev/null 2>&1
ncu -i gpurun_out/lnf_ncu.ncu-rep --page raw --csv > gpurun_out/lnf_raw.csv 2>/dev/null
ncu -i gpurun_out/lnf_ncu.ncu-rep --page source --csv --print-source sass > gpurun_out/lnf_source.csv 2>/dev/null
wc -l gpurun_out/rs_*.csv gpurun_out/lnf_*.csv
