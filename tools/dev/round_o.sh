#!/bin/bash
O=gpurun_out/o; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "r2r" > $O/r2r.log 2>&1; echo "exit $?" >> $O/r2r.log
tail -30 $O/r2r.log
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
tail -3 $O/pytest.log
timeout 300 python tools/quick_time.py 1024,1024,1024 f32 10 > $O/qt.log 2>&1; cat $O/qt.log
for g in 512,512,512 1024,512,512; do timeout 300 python bench.py --grid $g --kind c2c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> $O/r2r_bench.log; done
