python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l1.csv python tools/diag_stages.py 26 2 > /dev/null 2>&1
python tools/launches.py gpurun_out/l1.csv | grep onesweep
CG_OS_NOLB=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l2.csv python tools/diag_stages.py 26 2 > /dev/null 2>&1
python tools/launches.py gpurun_out/l2.csv | grep onesweep
