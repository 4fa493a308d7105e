make -j8 >/dev/null 2>&1
for tool in memcheck synccheck racecheck; do
timeout 900 compute-sanitizer --tool $tool --print-limit 5 python scripts/sanitize_s3.py > gpurun_out/san_$tool.log 2>&1; echo $tool rc $?; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|^ok" gpurun_out/san_$tool.log | tail -3
done
