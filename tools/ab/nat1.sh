cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_executor.py tests/test_gpu_parity.py tests/test_gpu_kinds.py tests/test_multi_gpu.py -q -m gpu 2>&1 | tail -2
run() { n=$1; shift; python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 500)) bench.py --gpus $n "$@"; }
show() { python - "$1" "$2" <<'PY'
import json,sys
lines=[l for l in open(sys.argv[1]) if l.startswith('{')]
d=json.loads(lines[-1]); t=d['timing']
print(sys.argv[2], 'b2b', round(t['back_to_back_ms'],3), 'graph', t['cuda_graph_ms'] and round(t['cuda_graph_ms'],3))
for s in d['roofline']['stages']: print('   ', s['kernel'][:52], s['bound'], round(s['avg_launch_ms'],3), round(s['ms_per_step'],3), round(s['frac'],3))
PY
}
for rep in 1 2; do
run 2 --steps 20 --warmup 5 --no-e2e > gpurun_out/n2.json 2>/dev/null; show gpurun_out/n2.json "nat1 N=2"
DFFT_NO_NAT1=1 run 2 --steps 20 --warmup 5 --no-e2e > gpurun_out/n2b.json 2>/dev/null; show gpurun_out/n2b.json "blocked N=2"
done
run 2 --steps 10 --warmup 3 --no-e2e --grid 768,768,384 --precision f64 --kind r2c > gpurun_out/n2c.json 2>/dev/null; show gpurun_out/n2c.json "cfg5 N=2 nat1"
