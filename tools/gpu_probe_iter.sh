# probe iteration: parity on the probe-heavy tests, C5 stage times, source-level ncu of the probe
set -x
mkdir -p gpurun_out
python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_probe.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_probe.log
timeout 300 python tools/diag_stages.py 26 5 2>&1 | grep '"rep"' | cut -c1-330 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_probe_global -c 1 -o gpurun_out/src_probe_new -f python tools/diag_stages.py 26 1 > gpurun_out/ncu_src_probe_new.log 2>&1
tail -2 gpurun_out/ncu_src_probe_new.log
