#!/bin/bash
O=gpurun_out/w; mkdir -p $O
for rep in 1 2; do for v in libdfft libdfft_w4; do
  echo "== $v" >> $O/ab.log
  DFFT_LIB=paper_2601_12209_b200/$v.so timeout 300 python tools/quick_time.py 1024,1024,1024 f32 10 >> $O/ab.log 2>&1
  DFFT_LIB=paper_2601_12209_b200/$v.so timeout 300 python tools/quick_time.py 512,512,512 f32 10 >> $O/ab.log 2>&1
done; done
cat $O/ab.log
