# launch list + ncu --set full of the sweep-path kernels at C5 (tools/diag_stages.py 26 1)
set -x
mkdir -p gpurun_out
python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2b.csv python tools/diag_stages.py 26 1 > gpurun_out/ncu_launch.log 2>&1
for k in k_pack_sweep k_region_sweep k_bucket_rank k_probe_global k_global_index; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/r2b_$k -f python tools/diag_stages.py 26 1 > gpurun_out/ncu_$k.log 2>&1
done
ls -la gpurun_out
