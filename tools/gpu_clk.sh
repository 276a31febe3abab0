python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
for ms in 50 0 500; do CG_CLOCK_MS=$ms timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --steps 20 | python -c "import json,sys; d=json.load(sys.stdin); print($ms, d['ms_per_step'], d['stage_us'], d['clocks'])"; done
