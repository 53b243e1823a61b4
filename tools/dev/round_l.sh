#!/bin/bash
O=gpurun_out/l; mkdir -p $O
for rep in 1 2; do
for v in old nospec notb nog0 none; do
  echo "== $v" >> $O/ab.log
  DFFT_LIB=paper_2601_12209_b200/libdfft_$v.so DFFT_SINGLE_LEGACY=1 timeout 300 python tools/quick_time.py 1024,1024,1024 f32 10 >> $O/ab.log 2>&1
done; done
cat $O/ab.log
