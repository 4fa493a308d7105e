# attention forward: PV of each kv tile in two key halves (ZI_ATTN_PVSPLIT=1) vs one MMA chain
make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
ZI_ATTN_PVSPLIT=1 timeout 600 python -m pytest tests/test_attn_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
for r in 1 2 3; do for v in 0 1; do echo -n "PVSPLIT=$v "; ZI_ATTN_PVSPLIT=$v timeout 120 python scripts/bench_attn.py 2>/dev/null | grep -i "zi" | head -2 | tr '\n' ' '; echo; done; done
bash scripts/_gpu_ab.sh ZI_ATTN_PVSPLIT "0 1" 2
