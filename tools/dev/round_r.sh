#!/bin/bash
O=gpurun_out/r; mkdir -p $O
for rep in 1 2; do for v in "DFFT_SINGLE_FWD_ZREAD=1" "X=1" "DFFT_SINGLE_INV_YWRITE=1"; do
  echo "== $v" >> $O/ab.log
  env $v timeout 300 python tools/quick_time.py 1024,1024,1024 f32 10 >> $O/ab.log 2>&1
done; done
echo "== f64 new" >> $O/ab.log; timeout 300 python tools/quick_time.py 1024,1024,1024 f64 5 >> $O/ab.log 2>&1
echo "== f64 old" >> $O/ab.log; DFFT_SINGLE_FWD_ZREAD=1 timeout 300 python tools/quick_time.py 1024,1024,1024 f64 5 >> $O/ab.log 2>&1
cat $O/ab.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > $O/t.log 2>&1; echo "exit $?" >> $O/t.log; tail -3 $O/t.log
timeout 300 python bench.py --grid 768,768,384 --precision f64 --kind r2r --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], {k: round(v,3) for k,v in d['phase_ms_per_step'].items()})"
