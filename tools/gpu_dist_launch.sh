python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
timeout 600 python -m pytest tests/test_gpu_dist.py -m gpu -x -q 2>&1 | tail -1
CHUNK_BITS=0 python tools/dist_stages.py 26 8 2>&1 | tail -1 | cut -c1-120
CHUNK_BITS=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dl.csv python tools/dist_stages.py 24 8 > /dev/null 2>&1
python tools/launches.py gpurun_out/dl.csv 400 | head -25
