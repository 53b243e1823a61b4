#!/bin/bash
O=gpurun_out/f1; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "radix57" > $O/t.log 2>&1; echo "exit $?" >> $O/t.log; tail -3 $O/t.log
b() { local N=$1; shift; timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2959$N bench.py --gpus $N --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>&1 | grep '^{'; }
for g in 480,480,480 720,720,720 840,840,840; do for N in 2 4; do b $N --grid $g > $O/c64_${g%%,*}_n$N.json; done; done
for f in $O/*.json; do python - "$f" <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1].split('/')[-1], d['n_gpus'], d['config']['workload'], round(d['ms_per_step'],3), 'ms', round(d['value']), 'GFLOP/s', 'ns-frac', round(d['north_star_roofline']['frac'],3))
PY
done
