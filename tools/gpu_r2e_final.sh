# final round-2 capture (tag r2e): bench line, launch list of the bench command,
# ncu --set full of the kernels changed since r2c
set -x
mkdir -p gpurun_out
python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
timeout 600 python bench.py > gpurun_out/bench_r2e.json 2> gpurun_out/bench_r2e.err; echo "bench rc=$?"
CG_BENCH_ALLOW_SHORT=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2e.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-f1 --no-configs > gpurun_out/ncu_bench.log 2>&1; echo "ncu bench rc=$?"
for k in k_probe_global k_bucket_rank k_pack_sweep k_region_sweep_p k_tile_copy; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/prof_$k -f python tools/diag_stages.py 26 1 > gpurun_out/ncu_$k.log 2>&1
done
ls gpurun_out
