#!/bin/bash
O=gpurun_out/m; mkdir -p $O
for rep in 1 2; do for v in old cur; do
  echo "== $v" >> $O/ab.log
  if [ $v = old ]; then L=paper_2601_12209_b200/libdfft_old.so; else L=paper_2601_12209_b200/libdfft.so; fi
  DFFT_LIB=$L timeout 300 python tools/quick_time.py 1024,1024,1024 f32 10 >> $O/ab.log 2>&1
done; done
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 > $O/bench_n1.json 2>&1
for N in 2 4; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N bench.py --gpus $N --steps 10 --warmup 3 2>&1 | grep '^{' > $O/bench_n$N.json; done
timeout 300 python bench.py --grid 768,768,384 --precision f64 --kind r2c --poisson --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/poisson_n1.json 2>&1
cat $O/ab.log; tail -3 $O/pytest.log
for f in $O/bench_n*.json $O/poisson_n1.json; do python - "$f" <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1].split('/')[-1], d['n_gpus'], d['config']['workload'], round(d['ms_per_step'],3), 'ms', round(d['value']), 'GFLOP/s', 'ns-frac', round(d['north_star_roofline']['frac'],3), 'k-frac', round(d['roofline']['frac'],3), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()})
PY
done
