#!/bin/bash
O=gpurun_out/thr; mkdir -p $O
b() { local N=$1; shift; timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2960$N bench.py --gpus $N --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['config']['chunks'], round(d['ms_per_step'],3))"; }
for K in 0 2 4; do b 4 --grid 480,480,480 --chunks $K; done
for K in 0 2 4; do b 2 --grid 256,256,256 --precision f64 --strategy slab --chunks $K; done
for K in 0 2 4; do b 4 --grid 256,256,256 --precision f64 --strategy slab --chunks $K; done
for K in 0 2 4; do b 4 --grid 768,768,384 --precision f64 --kind r2c --chunks $K; done
