#!/bin/bash
O=gpurun_out/i; mkdir -p $O
b() { local N=$1; shift; if [ $N -eq 1 ]; then timeout 300 python bench.py --steps 10 --warmup 3 "$@"; else timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N --steps 10 --warmup 3 "$@"; fi 2>&1 | grep '^{'; }
# scaling table, headline workload, defaults
for N in 1 2 4; do b $N > $O/bench_n$N.json; done
# 2x2: B->C chunks vs one chunk, same box
for K in 1 4; do echo "== 2x2 K=$K" >> $O/k.log; b 4 --chunks $K --no-e2e --no-cpu-baseline >> $O/k.log; done
# cfg5 box r2c f64 and the Poisson solve (f3)
for N in 1 2 4; do
  b $N --grid 768,768,384 --precision f64 --kind r2c --no-e2e --no-cpu-baseline > $O/r2c_n$N.json
  b $N --grid 768,768,384 --precision f64 --kind r2c --poisson --no-e2e --no-cpu-baseline > $O/poisson_n$N.json
done
# 512^3 c64 (cfg3) and 256^3 c128 slab (cfg2)
for N in 2 4; do
  b $N --grid 512,512,512 --no-e2e --no-cpu-baseline > $O/c512_n$N.json
  b $N --grid 256,256,256 --precision f64 --strategy slab --no-e2e --no-cpu-baseline > $O/c256slab_n$N.json
done
for f in $O/*.json $O/k.log; do python - "$f" <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1].split('/')[-1], d['n_gpus'], d['config']['workload'], round(d['ms_per_step'],3), 'ms', round(d['value']), 'GFLOP/s', 'ns-frac', round(d['north_star_roofline']['frac'],3), 'k-frac', round(d['roofline']['frac'],3))
PY
done
