# round-start baseline: parity suite + C5 stage timings + every config's build time
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2base.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_r2base.log
timeout 300 python tools/diag_stages.py 26 6 2>&1 | grep '"rep"' | cut -c1-700 > gpurun_out/stages_r2base.log
cat gpurun_out/stages_r2base.log
timeout 300 python tools/configs_timing.py > gpurun_out/configs_r2base.log 2>&1
cat gpurun_out/configs_r2base.log
