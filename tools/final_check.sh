#!/bin/bash
# Final verification of the committed build: GPU tests (incl. multi-GPU parity when >= 2 GPUs),
# smoke(), and the default bench line at N=1 (and N=4 when available).
O=gpurun_out/final; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log; tail -2 $O/smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log; tail -2 $O/pytest.log
timeout 400 python bench.py > $O/bench_n1.json 2>&1; grep '^{' $O/bench_n1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=1', d['ms_per_step'], d['north_star_roofline']['frac'], d['gpu_launches'])"
if [ $(nvidia-smi -L | wc -l) -ge 4 ]; then
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29599 bench.py --gpus 4 > $O/bench_n4.json 2>&1; grep '^{' $O/bench_n4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=4', d['ms_per_step'], d['north_star_roofline']['frac'], d['gpu_launches'])"
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29598 bench.py --gpus 2 > $O/bench_n2.json 2>&1; grep '^{' $O/bench_n2.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=2', d['ms_per_step'], d['north_star_roofline']['frac'], d['gpu_launches'])"
fi
