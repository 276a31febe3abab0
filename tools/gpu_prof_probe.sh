# C5 stage timings + source-level ncu capture of the probe kernel
set -x
mkdir -p gpurun_out
python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
timeout 300 python tools/diag_stages.py 26 4 2>&1 | grep '"rep"' | cut -c1-300
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_probe_global -c 1 -o gpurun_out/src_probe2 -f python tools/diag_stages.py 26 1 > gpurun_out/ncu_src_probe2.log 2>&1
tail -3 gpurun_out/ncu_src_probe2.log
