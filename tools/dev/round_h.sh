#!/bin/bash
O=gpurun_out/h; mkdir -p $O
timeout 1200 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
run() { timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], round(d['north_star_roofline']['frac'],3), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()})" ; }
for K in 4 8; do for S in 80 90 100 110; do echo "== K=$K NVL=$S" >> $O/sweep.log; DFFT_NVL_SMS=$S run --chunks $K >> $O/sweep.log 2>&1; done; done
tail -3 $O/pytest.log; cat $O/sweep.log
