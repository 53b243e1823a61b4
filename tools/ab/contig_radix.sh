# A/B: contig radix-32 (libdfft.so) vs radix-16 (libdfft_c16.so); N=1 whole-axis plan, N=2, N=4
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_executor.py tests/test_gpu_kinds.py -q -m gpu -x 2>&1 | tail -1
run() { n=$1; shift; python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 500)) bench.py --gpus $n "$@"; }
show() { python - "$1" "$2" <<'PY'
import json,sys
lines=[l for l in open(sys.argv[1]) if l.startswith('{')]
d=json.loads(lines[-1]); t=d['timing']
print(sys.argv[2], 'b2b', round(t['back_to_back_ms'],3), 'graph', t['cuda_graph_ms'] and round(t['cuda_graph_ms'],3))
for s in d['roofline']['stages']: print('   ', s['kernel'][:52], s['bound'], round(s['avg_launch_ms'],3), round(s['ms_per_step'],3), round(s['frac'],3))
PY
}
for lib in libdfft.so libdfft_c16.so; do
  export DFFT_LIB=$PWD/paper_2601_12209_b200/$lib
  DFFT_NO_XZ8=1 python tools/quick_time.py 1024,1024,1024 f32 10 2>/dev/null | tail -2
  run 2 --steps 20 --warmup 5 --no-e2e > gpurun_out/a2.json 2>/dev/null; show gpurun_out/a2.json "$lib N=2"
  run 4 --steps 20 --warmup 5 --no-e2e > gpurun_out/a4.json 2>/dev/null; show gpurun_out/a4.json "$lib N=4"
  python bench.py --steps 10 --warmup 3 --grid 768,768,384 --precision f64 --kind r2c --no-e2e --no-cpu-baseline > gpurun_out/a5.json 2>/dev/null; show gpurun_out/a5.json "$lib cfg5 N=1"
done
