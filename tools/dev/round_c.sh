#!/bin/bash
mkdir -p gpurun_out/c
O=gpurun_out/c
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "fused_store or simulated" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
for sk in 8 12 16; do
  timeout 300 ncu --set full --import-source on --clock-control none --launch-skip $sk --launch-count 1 -o /tmp/rep$sk -f \
     python tools/sim_time.py 1024,1024,1024 2,2 p2p f32 1 > $O/ncu$sk.log 2>&1
  ncu -i /tmp/rep$sk.ncu-rep --page raw --csv > $O/raw$sk.csv 2>/dev/null
  ncu -i /tmp/rep$sk.ncu-rep --page details --csv > $O/details$sk.csv 2>/dev/null
done
run() { timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], round(d['north_star_roofline']['frac'],3), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()})" ; }
for K in 1 2 4 8; do for S in 48 64 96; do echo "== K=$K NVL_SMS=$S" >> $O/sweep.log; DFFT_NVL_SMS=$S run --chunks $K >> $O/sweep.log 2>&1; done; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 tests/mp_check.py > $O/mp.log 2>&1; echo "mp exit $?" >> $O/mp.log
tail -2 $O/pytest.log; cat $O/sweep.log; tail -3 $O/mp.log
