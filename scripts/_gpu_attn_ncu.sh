make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fwd_kernel|bwd_dkdv|bwd_dq" -c 3 -o gpurun_out/attn_ncu python scripts/bench_attn.py 8 16 1024 128 --once > gpurun_out/attn_ncu.log 2>&1; tail -3 gpurun_out/attn_ncu.log
