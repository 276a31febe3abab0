# per-kernel launch lists of one build of each small config (C1, C2, C3, C4)
set -x
mkdir -p gpurun_out
python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
timeout 300 python tools/configs_timing.py ${CFGS:-C1,C2,C3,C4} 7
for c in ${CFGS:-C1 C2 C3 C4}; do
  c=${c//,/ }
done
for c in C1 C2 C3 C4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_$c.csv python tools/configs_timing.py $c 2 > /dev/null 2>&1
  echo "== $c"; python tools/launches.py gpurun_out/launch_$c.csv 200 2>&1 | tail -40
done
