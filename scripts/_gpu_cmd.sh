make -j8 >/dev/null 2>&1
CACHE=11 timeout 1200 python scripts/ab_config5.py 2:12 2:16 1:16 2:20 2:12 2>&1 | grep -v Warn | tail -6
