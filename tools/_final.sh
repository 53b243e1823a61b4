# r02 final evidence (4-GPU box): smoke, GPU tests, bench N=1/2/4 (+ secondary configs), ncu launch list, reference arm
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/final
O=gpurun_out/final
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.txt
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.txt 2>&1; tail -1 $O/pytest_gpu.txt
run() { n=$1; shift; python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 500)) bench.py --gpus $n "$@"; }
python bench.py --steps 20 --warmup 5 > $O/bench_n1.json 2> $O/bench_n1.err; tail -c 300 $O/bench_n1.json; echo
run 2 --steps 20 --warmup 5 > $O/bench_n2.json 2> $O/bench_n2.err; echo "n2 rc=$?"
run 4 --steps 20 --warmup 5 > $O/bench_n4.json 2> $O/bench_n4.err; echo "n4 rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > $O/ref_n1.json 2> $O/ref_n1.err; echo "ref rc=$?"
run 4 --steps 10 --warmup 3 --no-e2e --grid 768,768,384 --precision f64 --kind r2c > $O/bench_n4_cfg5.json 2>/dev/null; echo "cfg5 rc=$?"
run 4 --steps 10 --warmup 3 --no-e2e --grid 512,512,512 > $O/bench_n4_cfg3.json 2>/dev/null; echo "cfg3 rc=$?"
run 4 --steps 10 --warmup 3 --no-e2e --grid 256,256,256 --precision f64 --strategy slab > $O/bench_n4_cfg2.json 2>/dev/null; echo "cfg2 rc=$?"
run 4 --steps 10 --warmup 3 --no-e2e --exchange nccl > $O/bench_n4_nccl.json 2>/dev/null; echo "nccl rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_n1.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "ncu rc=$?"
ls -la $O
