set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches2.csv python tools/diag_stages.py 26 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_probe -c 1 -o gpurun_out/prof_probe -f python tools/diag_stages.py 26 1 > gpurun_out/ncu_probe.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_bucket_sort -c 1 -o gpurun_out/prof_bucket -f python tools/diag_stages.py 26 1 > gpurun_out/ncu_bucket.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_onesweep -c 2 -o gpurun_out/prof_onesweep -f python tools/diag_stages.py 26 1 > gpurun_out/ncu_onesweep.log 2>&1
tail -2 gpurun_out/ncu_*.log
ls -la gpurun_out
