#!/bin/bash
# One GPU verification pass: gpu tests (incl. multi-GPU parity when >=2 devices), then bench N=1,2,4.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_n1.log 2>&1
NG=$(nvidia-smi -L | wc -l)
for N in 2 4; do
  if [ $NG -ge $N ]; then
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/bench_n$N.log 2>&1
  fi
done
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/bench_n*.log
