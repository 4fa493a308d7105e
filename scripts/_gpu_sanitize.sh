make -j16 >/dev/null 2>&1 || { echo build failed; exit 1; }
for t in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize_r2.py > gpurun_out/san_$t.log 2>&1
  echo "$t rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|^ok" gpurun_out/san_$t.log | tail -3
done
