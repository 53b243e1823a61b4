#!/bin/bash
O=gpurun_out/f; mkdir -p $O
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29515 tests/mp_check.py > $O/mp.log 2>&1; echo "mp exit $?" >> $O/mp.log
run() { timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], round(d['north_star_roofline']['frac'],3), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()})" ; }
echo "== default (bulk, K=1)" >> $O/sweep.log; run >> $O/sweep.log 2>&1
echo "== no bulk" >> $O/sweep.log; DFFT_NO_BULK=1 run >> $O/sweep.log 2>&1
for K in 2 4; do for S in 100 124; do echo "== K=$K NVL=$S" >> $O/sweep.log; DFFT_NVL_SMS=$S run --chunks $K >> $O/sweep.log 2>&1; done; done
echo "== 1x4" >> $O/sweep.log; run --grid-p 1,4 >> $O/sweep.log 2>&1
echo "== 4x1" >> $O/sweep.log; run --grid-p 4,1 >> $O/sweep.log 2>&1
tail -2 $O/mp.log; cat $O/sweep.log
