# launch list of the bench command + ncu --set full captures of the top kernels (source-level)
set -x
mkdir -p gpurun_out
python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
CG_BENCH_ALLOW_SHORT=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-f1 > gpurun_out/ncu_bench.log 2>&1
for k in ${KERNELS:-k_probe_global k_bucket_rank k_onesweep k_pack k_global_index k_tile_copy}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c ${NCOUNT:-1} -o gpurun_out/prof_$k -f python tools/diag_stages.py 26 1 > gpurun_out/ncu_$k.log 2>&1
done
ls gpurun_out
