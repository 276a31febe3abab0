# probe A/B: parity tests on the default build, then interleaved C5 timings of the variants
set -x
mkdir -p gpurun_out
python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -x -q > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ab.log
L=paper_1503_06029_b200/lib/ab
timeout 900 python tools/ab_time.py ${CFG:-C5} ${REPS:-7} $(for v in $VARIANTS; do echo $L/libcg_$v.so; done) 2>&1 | tail -12
