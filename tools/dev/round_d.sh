#!/bin/bash
O=gpurun_out/d; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "fused_store or simulated" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 tests/mp_check.py > $O/mp.log 2>&1; echo "mp exit $?" >> $O/mp.log
run() { timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], round(d['north_star_roofline']['frac'],3), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()})" ; }
echo "== bulk" >> $O/sweep.log; run >> $O/sweep.log 2>&1
echo "== no bulk" >> $O/sweep.log; DFFT_NO_BULK=1 run >> $O/sweep.log 2>&1
echo "== bulk K=4 NVL 100" >> $O/sweep.log; DFFT_NVL_SMS=100 run --chunks 4 >> $O/sweep.log 2>&1
echo "== bulk K=4 NVL 120" >> $O/sweep.log; DFFT_NVL_SMS=120 run --chunks 4 >> $O/sweep.log 2>&1
tail -2 $O/pytest.log; tail -2 $O/mp.log; cat $O/sweep.log
