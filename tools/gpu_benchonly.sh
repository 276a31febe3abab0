python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
for i in 1 2; do timeout 600 python bench.py $BENCH_ARGS > gpurun_out/bench_$i.json 2>gpurun_out/bench_$i.err; python -c "
import json; d=json.load(open('gpurun_out/bench_$i.json'))
print(d['ms_per_step'], d['stage_us'])"; done
