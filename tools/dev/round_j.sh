#!/bin/bash
O=gpurun_out/j; mkdir -p $O
for rep in 1 2; do
for v in "DFFT_LIB=paper_2601_12209_b200/libdfft_old.so" "DFFT_SINGLE_LEGACY=1" "X=1"; do
  echo "== $v" >> $O/ab.log
  env $v timeout 300 python tools/quick_time.py 1024,1024,1024 f32 10 >> $O/ab.log 2>&1
done; done
timeout 1200 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 > $O/bench_n1.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none --csv \
    --log-file $O/launches_n1.csv python tools/quick_time.py 1024,1024,1024 f32 1 > /dev/null 2>&1
cat $O/ab.log; tail -3 $O/pytest.log; python tools/ncu_summary.py $O/launches_n1.csv fft_ | head -12
if [ $(nvidia-smi -L | wc -l) -ge 2 ]; then ./tools/p2p_tma > $O/p2p_tma.log 2>&1; cat $O/p2p_tma.log; fi
