# multi-GPU bench on the available GPUs (1 here): torchrun path with N=1 and logical test
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/pytest_dist.txt 2>&1; tail -3 gpurun_out/pytest_dist.txt
NG=$(nvidia-smi -L | wc -l)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $NG --steps 5 --warmup 3 > gpurun_out/bench_dist.json 2> gpurun_out/bench_dist.err; tail -2 gpurun_out/bench_dist.err
cat gpurun_out/bench_dist.json
