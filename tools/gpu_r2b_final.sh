# round-2 refresh on the sweep path: GPU tests, sanitizers, bench launch list,
# ncu --set full captures of the top kernels (tag r2b)
set -x
mkdir -p gpurun_out
python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
timeout 900 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_r2b.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_r2b.log
bash tools/gpu_sanitize.sh
CG_BENCH_ALLOW_SHORT=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2b.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-f1 --no-configs > gpurun_out/ncu_bench.log 2>&1; echo "ncu bench rc=$?"
for k in k_probe_global k_bucket_rank k_pack_sweep k_region_sweep k_tile_copy; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/prof_$k -f python tools/diag_stages.py 26 1 > gpurun_out/ncu_$k.log 2>&1
done
ls gpurun_out
