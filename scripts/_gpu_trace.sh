make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 300 python scripts/bench_attn.py 8 16 1024 128 --trace-bwd 2>&1 | head -40
