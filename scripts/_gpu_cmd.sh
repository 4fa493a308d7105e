make -j8 >/dev/null 2>&1
timeout 600 python scripts/step_gaps.py 2>&1 | grep -v Warn | tail -30
