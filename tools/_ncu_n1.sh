cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_executor.py -q -k "radix_by_plan or launch_counter or product_executor" 2>&1 | tail -1
python tools/quick_time.py 1024,1024,1024 f32 3 > /dev/null 2>&1 && echo "plain rc=0"
ncu --set full --clock-control none --import-source on -k regex:"fft_" -c 6 -o /tmp/n1 python tools/quick_time.py 1024,1024,1024 f32 1 > gpurun_out/n1_ncu_full.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/n1.ncu-rep --page details --csv > gpurun_out/n1_full_details.csv
ncu -i /tmp/n1.ncu-rep --page raw --csv > gpurun_out/n1_full_raw.csv
