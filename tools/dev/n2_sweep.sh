#!/bin/bash
mkdir -p gpurun_out
run() { timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e "$@" 2>/dev/null | grep '^{' ; }
for ex in p2p ce hybrid; do for K in 1 2 4 8 16; do
  echo "== $ex K=$K"; run --exchange $ex --chunks $K | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['north_star_roofline']['frac'], {k: round(v,3) for k,v in d['phase_ms_per_step'].items()})"
done; done
