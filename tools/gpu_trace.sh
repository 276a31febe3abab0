python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
for i in 1 2 3; do CG_TRACE=1 timeout 600 python bench.py --e2e-steps 0 --no-cpu-baseline 2>&1 | grep -v "^\[cg\] [a-z]* *[0-9.]* us" | tail -20 | cut -c1-200; done
