#!/bin/bash
O=gpurun_out/q; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "r2r or graph or poisson or r2c" > $O/t.log 2>&1; echo "exit $?" >> $O/t.log
tail -5 $O/t.log
for g in 768,768,384; do timeout 300 python bench.py --grid $g --precision f64 --kind r2r --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' > $O/r2r_n1.json; done
timeout 300 python bench.py --grid 512,512,512 --kind r2r --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' > $O/r2r512_n1.json
timeout 300 python bench.py --grid 64,64,64 --precision f64 --strategy slab --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' > $O/cfg1.json
for f in $O/*.json; do python - "$f" <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1].split('/')[-1], d['n_gpus'], d['config']['workload'], round(d['ms_per_step'],4), 'ms', round(d['value']), 'GFLOP/s', 'ns-frac', round(d['north_star_roofline']['frac'],3), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()})
PY
done
