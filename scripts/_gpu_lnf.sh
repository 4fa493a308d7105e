make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
for m in 1 3 4; do echo "MINB=$m"; ZI_LNF_MINB=$m timeout 300 python scripts/bench_fused.py 2>&1 | grep ln_fwd; done
