#!/bin/bash
O=gpurun_out/t; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "fused_store or simulated or r2r" > $O/t.log 2>&1; echo "exit $?" >> $O/t.log; tail -2 $O/t.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29516 tests/mp_check.py > $O/mp.log 2>&1; echo "mp exit $?" >> $O/mp.log; tail -2 $O/mp.log
b() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], {k: round(v,3) for k,v in d['phase_ms_per_step'].items()})"; }
for rep in 1 2; do
echo "== no bc 1xP" >> $O/k.log; DFFT_NO_BC_1XP=1 b >> $O/k.log
for K in 2 4 8; do for S in 80 100; do echo "== K=$K NVL=$S" >> $O/k.log; DFFT_NVL_SMS=$S b --chunks $K >> $O/k.log; done; done
done
cat $O/k.log
