#!/bin/bash
O=gpurun_out/g; mkdir -p $O
for cfg in "X=1" "DFFT_TMA_PROMO128=1" "DFFT_TMA_PROMO256=1" "DFFT_G0_FWD_C=1" "DFFT_G0_FWD_C=0"; do
  echo "== $cfg" >> $O/sim.log
  env $cfg timeout 300 python tools/sim_time.py 1024,1024,1024 2,2 p2p f32 3 >> $O/sim.log 2>&1
  env $cfg timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none --csv \
    --log-file $O/l_$cfg.csv python tools/sim_time.py 1024,1024,1024 2,2 p2p f32 1 > /dev/null 2>&1
  python tools/ncu_summary.py $O/l_$cfg.csv fft_ 2>/dev/null | head -28 >> $O/sim.log
done
for cfg in "X=1" "DFFT_TMA_PROMO128=1" "DFFT_TMA_PROMO256=1"; do
  echo "== single $cfg" >> $O/sim.log; env $cfg timeout 300 python tools/quick_time.py 1024,1024,1024 f32 10 >> $O/sim.log 2>&1
done
cat $O/sim.log
