make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ln_bwd_split" -s 2 -c 1 -o gpurun_out/lnb_ncu python scripts/bench_fused.py > /dev/null 2>&1; ls gpurun_out/lnb_ncu*
