# source-level ncu captures of the C5 probe and bucket-rank kernels
set -x
mkdir -p gpurun_out
python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_probe_global -c 1 -o gpurun_out/src_probe -f python tools/diag_stages.py 26 1 > gpurun_out/ncu_src_probe.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bucket_rank -c 1 -o gpurun_out/src_bucket -f python tools/diag_stages.py 26 1 > gpurun_out/ncu_src_bucket.log 2>&1
ls -la gpurun_out
