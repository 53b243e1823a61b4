#!/bin/bash
O=gpurun_out/t2; mkdir -p $O
for rep in 1 2; do for v in "X=1" "DFFT_TMA2=1"; do
  echo "== $v" >> $O/ab.log
  env $v timeout 120 python tools/quick_time.py 1024,1024,1024 f32 10 >> $O/ab.log 2>&1
  env $v timeout 120 python tools/quick_time.py 1024,1024,1024 f64 5 >> $O/ab.log 2>&1
done; done
cat $O/ab.log
