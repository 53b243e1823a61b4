#!/bin/bash
O=gpurun_out/promo; mkdir -p $O
for rep in 1 2; do for v in "X=1" "DFFT_TMA_PROMO128=1" "DFFT_TMA_PROMO256=1"; do
  echo "== $v" >> $O/ab.log
  env $v timeout 120 python tools/quick_time.py 1024,1024,1024 f32 10 >> $O/ab.log 2>&1
done; done
for v in "X=1" "DFFT_TMA_PROMO128=1" "DFFT_TMA_PROMO256=1"; do
  echo "== sim2x2 $v" >> $O/ab.log
  env $v timeout 200 python tools/sim_time.py 1024,1024,1024 2,2 p2p f32 3 >> $O/ab.log 2>&1
done
cat $O/ab.log
