rm -f gpurun_out/sanitize_summary.txt
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 7 python tools/sanitize_run.py > gpurun_out/sanitize_$t.log 2>&1; echo "sanitizer $t rc=$?" >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt
grep -h "ERROR SUMMARY\|RACECHECK SUMMARY\|hazard\|Error" gpurun_out/sanitize_*.log | sort | uniq -c | head -20
