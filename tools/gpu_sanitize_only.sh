mkdir -p gpurun_out; rm -f gpurun_out/sanitize_summary.txt
python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 7 python tools/sanitize_run.py > gpurun_out/sanitize_$t.log 2>&1; echo "sanitizer $t rc=$?" >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt
