make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ln_bwd_split|ln_fwd_warp|colrow|softmax_ce_ring" -s 3 -c 4 -o gpurun_out/ew_ncu python scripts/bench_fused.py > gpurun_out/ew_ncu.log 2>&1; tail -2 gpurun_out/ew_ncu.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fwd2_kernel|bwd_dkdv|bwd_dq" -c 3 -o gpurun_out/attn_r2_ncu python scripts/bench_attn.py 8 16 1024 128 --once > /dev/null 2>&1; ls gpurun_out/*.ncu-rep
