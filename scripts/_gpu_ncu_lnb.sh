# LayerNorm backward (two-phase ring kernel): warm timings, then ncu --set full of one launch
make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 300 python scripts/bench_fused.py 2>&1 | head -4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ln_bwd_split" -s 2 -c 1 \
  -o gpurun_out/lnb_ncu python scripts/bench_fused.py > gpurun_out/lnb_ncu.log 2>&1; ls gpurun_out/lnb_ncu*
ncu -i gpurun_out/lnb_ncu.ncu-rep --page raw --csv > gpurun_out/lnb_raw.csv 2>/dev/null
ncu -i gpurun_out/lnb_ncu.ncu-rep --page details --csv > gpurun_out/lnb_details.csv 2>/dev/null
ncu -i gpurun_out/lnb_ncu.ncu-rep --page source --csv --print-source sass > gpurun_out/lnb_source.csv 2>/dev/null
wc -l gpurun_out/lnb_*.csv
