# full GPU suite + per-config timings (C1..C4) + C5 stage line
set -x
mkdir -p gpurun_out
python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 300 python tools/configs_timing.py ${CFGS:-C1,C2,C3,C4} 7
timeout 300 python tools/diag_stages.py 26 4 2>&1 | grep '"rep": 3' | cut -c1-400
