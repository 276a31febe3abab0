python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
timeout 300 python tools/f1_stages.py 26 2 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_signatures -c 1 -o gpurun_out/src_sign -f python tools/f1_stages.py 24 1 > /dev/null 2>&1
