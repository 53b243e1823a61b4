#!/bin/bash
b() { local N=$1; shift; if [ $N -eq 1 ]; then timeout 400 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@"; else timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2962$N bench.py --gpus $N --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@"; fi 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['config']['workload'], d['config']['chunks'], round(d['ms_per_step'],3), round(d['north_star_roofline']['frac'],3))"; }
for N in 1 2 4; do
  b $N --grid 768,768,384 --precision f64 --kind r2c --poisson
  b $N --grid 768,768,384 --precision f64 --kind r2r
done
b 2 --grid 256,256,256 --precision f64 --strategy slab
b 4 --grid 256,256,256 --precision f64 --strategy slab
