python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
timeout 600 python bench.py --dist --steps 5 --warmup 3 --e2e-steps 2 2>&1 | tail -3 | cut -c1-2500
timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'], d['gpu_launches'], d['roofline']['frac'])"
