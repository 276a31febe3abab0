# one iteration: full parity suite (fail fast) + C5 stage timings + all configs
set -x
mkdir -p gpurun_out
python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_iter.log
timeout 300 python tools/diag_stages.py 26 6 2>&1 | grep '"rep"' | cut -c1-420 | tail -3
timeout 300 python tools/configs_timing.py 2>&1 | cut -c1-400
