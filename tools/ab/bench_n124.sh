# N=1/2/4 bench lines + multi-GPU tests (4-GPU box)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multi_gpu.py -q -m gpu -x 2>&1 | tail -2
run() { n=$1; shift; python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 500)) bench.py --gpus $n "$@"; }
show() { python - "$1" <<'PY'
import json,sys
lines=[l for l in open(sys.argv[1]) if l.startswith('{')]
d=json.loads(lines[-1]); t=d['timing']
print(sys.argv[1].split('/')[-1], 'b2b', round(t['back_to_back_ms'],3), 'graph', t['cuda_graph_ms'] and round(t['cuda_graph_ms'],3), 'ns', round(d['north_star_roofline']['frac'],3))
for s in d['roofline']['stages']: print('   ', s['kernel'][:52], s['bound'], round(s['avg_launch_ms'],3), round(s['ms_per_step'],3), round(s['frac'],3))
PY
}
python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/g1.json 2>/dev/null; show gpurun_out/g1.json
run 2 --steps 20 --warmup 5 --no-e2e > gpurun_out/g2.json 2>/dev/null; show gpurun_out/g2.json
run 4 --steps 20 --warmup 5 --no-e2e > gpurun_out/g4.json 2>/dev/null; show gpurun_out/g4.json
