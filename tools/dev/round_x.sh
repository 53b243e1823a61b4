#!/bin/bash
O=gpurun_out/x; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log; tail -2 $O/smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log; tail -2 $O/pytest.log
timeout 400 python bench.py > $O/bench_default.json 2>&1; tail -c 2500 $O/bench_default.json
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $O/ref.json 2>&1; tail -c 800 $O/ref.json
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29591 bench.py --gpus 4 > $O/bench_n4_default.json 2>&1; grep '^{' $O/bench_n4_default.json | tail -c 1500
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29592 bench.py --gpus 4 --impl reference --steps 2 --warmup 1 > $O/ref_n4.json 2>&1; tail -c 300 $O/ref_n4.json
