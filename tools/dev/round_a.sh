#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "fused_store or simulated" > gpurun_out/a_pytest.log 2>&1; echo "exit $?" >> gpurun_out/a_pytest.log
for cfg in "" "DFFT_NO_TBLOCK=1" "DFFT_G0_FWD_C=0 DFFT_G0_INV_B=0" "DFFT_G0_FWD_C=1" "DFFT_G0_FWD_C=8" "DFFT_G0_FWD_C=2"; do
  echo "== $cfg" >> gpurun_out/a_sim.log
  env $cfg timeout 300 python tools/sim_time.py 1024,1024,1024 2,2 p2p f32 3 >> gpurun_out/a_sim.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/a_sim_launches.csv python tools/sim_time.py 1024,1024,1024 2,2 p2p f32 1 > gpurun_out/a_ncu.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e > gpurun_out/a_bench_n2.log 2>&1
tail -2 gpurun_out/a_pytest.log; cat gpurun_out/a_sim.log; tail -c 1500 gpurun_out/a_bench_n2.log
