#!/bin/bash
O=gpurun_out/u; mkdir -p $O
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log; tail -2 $O/pytest.log
b() { local N=$1; shift; if [ $N -eq 1 ]; then timeout 300 python bench.py --steps 10 --warmup 3 "$@"; else timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2957$N bench.py --gpus $N --steps 10 --warmup 3 "$@"; fi 2>&1 | grep '^{'; }
for N in 1 2 4; do b $N > $O/bench_n$N.json; done
for N in 2 4; do
  b $N --grid 256,256,256 --precision f64 --strategy slab --no-e2e --no-cpu-baseline > $O/cfg2_n$N.json
  b $N --grid 512,512,512 --no-e2e --no-cpu-baseline > $O/cfg3_n$N.json
done
for N in 1 2 4; do
  b $N --grid 768,768,384 --precision f64 --kind r2c --no-e2e --no-cpu-baseline > $O/cfg5_n$N.json
  b $N --grid 768,768,384 --precision f64 --kind r2c --poisson --no-e2e --no-cpu-baseline > $O/poisson_n$N.json
  b $N --grid 768,768,384 --precision f64 --kind r2r --no-e2e --no-cpu-baseline > $O/r2r_n$N.json
done
b 4 --grid-p 1,4 --no-e2e --no-cpu-baseline > $O/bench_n4_1x4.json
b 4 --strategy slab --no-e2e --no-cpu-baseline > $O/bench_n4_slab.json
for f in $O/*.json; do python - "$f" <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1].split('/')[-1], d['n_gpus'], d['config']['workload'], round(d['ms_per_step'],3), 'ms', round(d['value']), 'GFLOP/s', 'ns-frac', round(d['north_star_roofline']['frac'],3), 'k-frac', round(d['roofline']['frac'],3), 'e2e', round((d.get('e2e') or {}).get('value') or 0))
PY
done
