make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fwd2_kernel|bwd_dkdv" -c 2 -o gpurun_out/attn2_ncu python scripts/bench_attn.py 8 16 1024 128 --once > gpurun_out/attn_ncu.log 2>&1; tail -3 gpurun_out/attn_ncu.log
