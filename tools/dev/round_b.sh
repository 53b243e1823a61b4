#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "fused_store or simulated" > gpurun_out/b_pytest.log 2>&1; echo "exit $?" >> gpurun_out/b_pytest.log
timeout 600 ncu --set full --import-source on --clock-control none --launch-skip 4 --launch-count 9 -o gpurun_out/b_sim22 -f \
   python tools/sim_time.py 1024,1024,1024 2,2 p2p f32 1 > gpurun_out/b_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fft_strided_tma --launch-skip 0 --launch-count 2 -o gpurun_out/b_single -f \
   python tools/quick_time.py 1024,1024,1024 f32 1 > gpurun_out/b_ncu1.log 2>&1
tail -2 gpurun_out/b_pytest.log; tail -3 gpurun_out/b_ncu.log gpurun_out/b_ncu1.log
