set -x
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --dist --steps 5 --warmup 3 > gpurun_out/bench_dist1.json 2> gpurun_out/bench_dist1.err; tail -5 gpurun_out/bench_dist1.err
cat gpurun_out/bench_dist1.json
