# dist iteration: logical-rank tests, dist stage times at G = 1 / 8 on C5
set -x
mkdir -p gpurun_out
python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
timeout 900 python -m pytest tests/test_gpu_dist.py -m gpu -x -q > gpurun_out/pytest_dist.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_dist.log
timeout 600 python tools/dist_stages.py 26 2>&1 | tail -8
