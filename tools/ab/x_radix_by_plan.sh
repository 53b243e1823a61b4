cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_executor.py tests/test_gpu_parity.py tests/test_multi_gpu.py -q -m gpu 2>&1 | tail -1
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
run 4 --steps 20 --warmup 5 --no-e2e > gpurun_out/r4.json 2>/dev/null; show gpurun_out/r4.json "r16@P1>1 N=4"
DFFT_CONTIG_R32=1 run 4 --steps 20 --warmup 5 --no-e2e > gpurun_out/r4b.json 2>/dev/null; show gpurun_out/r4b.json "r32 N=4"
done
run 2 --steps 20 --warmup 5 --no-e2e > gpurun_out/r2.json 2>/dev/null; show gpurun_out/r2.json "N=2"
run 4 --steps 10 --warmup 3 --no-e2e --grid 768,768,384 --precision f64 --kind r2c > gpurun_out/r4c.json 2>/dev/null; show gpurun_out/r4c.json "cfg5 N=4"
