#!/bin/bash
O=gpurun_out/n; mkdir -p $O
for rep in 1 2; do for v in "DFFT_TST_WORK=1" "X=1"; do
  echo "== $v" >> $O/ab.log
  env $v timeout 300 python tools/quick_time.py 1024,1024,1024 f32 10 >> $O/ab.log 2>&1
  env $v timeout 300 python tools/quick_time.py 1024,1024,1024 f64 5 >> $O/ab.log 2>&1
done; done
cat $O/ab.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
tail -3 $O/pytest.log
