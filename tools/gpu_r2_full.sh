# round-2 evidence: bench line, launch list of the bench command, ncu --set full
# captures of the top kernels (C5) and of the C4 kernels, sanitizers
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
CG_BENCH_ALLOW_SHORT=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-f1 --no-configs > gpurun_out/ncu_bench.log 2>&1
for k in k_probe_global k_bucket_rank k_onesweep k_pack k_global_index k_tile_copy; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/prof_$k -f python tools/diag_stages.py 26 1 > gpurun_out/ncu_$k.log 2>&1
done
for k in k_probe_global k_gather_rows k_tie_fix_prefix k_pack; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/c4prof_$k -f python tools/configs_timing.py C4 1 > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_small -c 1 -o gpurun_out/c1prof_k_small_build -f python tools/configs_timing.py C1 1 > /dev/null 2>&1
rm -f gpurun_out/sanitize_summary.txt
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 7 python tools/sanitize_run.py > gpurun_out/sanitize_$t.log 2>&1; echo "sanitizer $t rc=$?" >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt
cat gpurun_out/bench.json
