set -x
mkdir -p gpurun_out
python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
timeout 600 python tools/dist_stages.py 26 8 2>&1 | tail -1 | cut -c1-300
timeout 900 ncu --nvtx --nvtx-include "merge/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dist_launches.csv python tools/dist_merge_only.py 26 8 3 > gpurun_out/dist_prof.log 2>&1
tail -3 gpurun_out/dist_prof.log
python tools/launches.py gpurun_out/dist_launches.csv 100000 2>&1 | head -30
