#!/bin/bash
O=gpurun_out/y; mkdir -p $O
for rep in 1 2; do for v in "X=1" "DFFT_XPASS_ZFAST=1"; do
  echo "== $v" >> $O/ab.log
  env $v timeout 300 python tools/quick_time.py 1024,1024,1024 f32 10 >> $O/ab.log 2>&1
done; done
cat $O/ab.log
