# r02 xz8 evidence: bench line, ncu launch list of the same bench command, ncu --set full of the stage kernels
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/r02_xz8_bench_n1.json 2> gpurun_out/r02_xz8_bench_n1.err
tail -c 400 gpurun_out/r02_xz8_bench_n1.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02_xz8_launches_n1.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02_xz8_ncu_launch.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"fft_" -c 6 -o /tmp/stages python tools/quick_time.py 1024,1024,1024 f32 1 > gpurun_out/r02_xz8_ncu_full.log 2>&1
echo "full rc=$?"
ncu -i /tmp/stages.ncu-rep --page details --csv > gpurun_out/r02_xz8_full_details.csv
ncu -i /tmp/stages.ncu-rep --page raw --csv > gpurun_out/r02_xz8_full_raw.csv
ls -la gpurun_out | tail -8
