#!/bin/bash
O=gpurun_out/n8; mkdir -p $O
nvidia-smi -L > $O/gpus.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29597 bench.py --gpus 8 > $O/bench_n8.json 2>&1
tail -c 2500 $O/bench_n8.json
