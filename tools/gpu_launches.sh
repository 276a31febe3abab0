# per-kernel launch list (ncu gpu__time_duration) of 2 C5 builds
set -x
mkdir -p gpurun_out
python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_q.csv python tools/diag_stages.py 26 2 > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_q.csv 2>&1 | tail -25
