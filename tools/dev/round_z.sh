#!/bin/bash
O=gpurun_out/z; mkdir -p $O
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log; tail -2 $O/pytest.log
b() { local N=$1; shift; if [ $N -eq 1 ]; then timeout 400 python bench.py --steps 10 --warmup 3 "$@"; else timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2958$N bench.py --gpus $N --steps 10 --warmup 3 "$@"; fi 2>&1 | grep '^{'; }
for N in 1 2 4; do b $N > $O/bench_n$N.json; done
for S in 64 72 88; do echo "== 1x2 NVL=$S" >> $O/k.log; DFFT_NVL_SMS=$S b 2 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])" >> $O/k.log; done
for S in 72 88; do echo "== 2x2 NVL=$S" >> $O/k.log; DFFT_NVL_SMS=$S b 4 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])" >> $O/k.log; done
b 1 --grid 1024,1024,1024 --precision f64 --no-e2e --no-cpu-baseline > $O/c128_n1.json
b 4 --grid 1024,1024,1024 --precision f64 --no-e2e --no-cpu-baseline > $O/c128_n4.json
for f in $O/*.json; do python - "$f" <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1].split('/')[-1], d['n_gpus'], d['config']['workload'], round(d['ms_per_step'],3), 'ms', round(d['value']), 'GFLOP/s', 'ns-frac', round(d['north_star_roofline']['frac'],3), 'k-frac', round(d['roofline']['frac'],3), 'launches', d['gpu_launches'], 'e2e', round((d.get('e2e') or {}).get('value') or 0))
PY
done
cat $O/k.log
