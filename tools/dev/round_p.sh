#!/bin/bash
O=gpurun_out/p; mkdir -p $O
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29515 tests/mp_check.py > $O/mp.log 2>&1; echo "mp exit $?" >> $O/mp.log
b() { local N=$1; shift; if [ $N -eq 1 ]; then timeout 300 python bench.py --steps 10 --warmup 3 "$@"; else timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N --steps 10 --warmup 3 "$@"; fi 2>&1 | grep '^{'; }
for N in 1 2 4; do b $N > $O/bench_n$N.json; done
for N in 1 2 4; do b $N --grid 768,768,384 --precision f64 --kind r2r --no-e2e --no-cpu-baseline > $O/r2r_n$N.json; done
for N in 1 4; do b $N --grid 512,512,512 --kind r2r --no-e2e --no-cpu-baseline > $O/r2r512_n$N.json; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file $O/launches_bench_n1.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_bench.log 2>&1
tail -2 $O/mp.log
for f in $O/*.json; do python - "$f" <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1].split('/')[-1], d['n_gpus'], d['config']['workload'], round(d['ms_per_step'],3), 'ms', round(d['value']), 'GFLOP/s', 'ns-frac', round(d['north_star_roofline']['frac'],3), 'k-frac', round(d['roofline']['frac'],3), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()})
PY
done
