# source-level ncu capture of one kernel (regex $K) in a C5 build
set -x
mkdir -p gpurun_out
python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/src_$K -f python tools/diag_stages.py 26 1 > gpurun_out/ncu_src_$K.log 2>&1
tail -2 gpurun_out/ncu_src_$K.log
