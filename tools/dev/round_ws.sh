#!/bin/bash
O=gpurun_out/ws; mkdir -p $O
for rep in 1 2; do for v in "X=1" "DFFT_TMA_WS=1" "DFFT_LIB=paper_2601_12209_b200/libdfft_r16.so"; do
  echo "== $v" >> $O/ab.log
  env $v timeout 120 python tools/quick_time.py 1024,1024,1024 f32 10 >> $O/ab.log 2>&1
done; done
cat $O/ab.log
DFFT_TMA_WS=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "headline_1024cubed_c64_single or 3d_single or cfg1 or closed_forms" > $O/t.log 2>&1; echo "exit $?" >> $O/t.log; tail -3 $O/t.log
