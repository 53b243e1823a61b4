#!/bin/bash
O=gpurun_out/k; mkdir -p $O
for rep in 1 2 3; do
for v in "DFFT_LIB=paper_2601_12209_b200/libdfft_old.so" "DFFT_SINGLE_LEGACY=1"; do
  echo "== $v" >> $O/ab.log
  env $v timeout 300 python tools/quick_time.py 1024,1024,1024 f32 10 >> $O/ab.log 2>&1
done; done
cat $O/ab.log
