#!/bin/bash
O=gpurun_out/v; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "r2r" > $O/t.log 2>&1; echo "exit $?" >> $O/t.log; tail -3 $O/t.log
for v in "DFFT_NO_TMA=1" "X=1"; do
  echo "== $v" >> $O/b.log
  env $v timeout 300 python bench.py --grid 768,768,384 --precision f64 --kind r2r --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], {k: round(v,3) for k,v in d['phase_ms_per_step'].items()})" >> $O/b.log
  env $v timeout 300 python bench.py --grid 512,512,512 --kind r2r --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], {k: round(v,3) for k,v in d['phase_ms_per_step'].items()})" >> $O/b.log
done
cat $O/b.log
