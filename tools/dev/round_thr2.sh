#!/bin/bash
b() { local N=$1; shift; timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N bench.py --gpus $N --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['config']['chunks'], round(d['ms_per_step'],3), round(d['north_star_roofline']['frac'],3))"; }
b 4 --grid 768,768,384 --precision f64 --kind r2c
b 4 --grid 512,512,512
b 2 --grid 512,512,512
b 2 --grid 768,768,384 --precision f64 --kind r2c
b 4
b 2
