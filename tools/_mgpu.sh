timeout 900 python -m pytest tests/test_multi_gpu.py tests/test_gpu_executor.py tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
run() { n=$1; shift; python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 500)) bench.py --gpus $n "$@"; }
show() { python -c "
import json,sys
lines=[l for l in open('$1') if l.startswith('{')]
d=json.loads(lines[-1]); t=d['timing']
print('$1'.split('/')[-1], 'b2b', round(t['back_to_back_ms'],3), 'iter', round(t['per_iteration_ms']['median'],3), 'graph', round(t['cuda_graph_ms'],3), 'host', round(t['host_enqueue_ms_per_step'],3), 'ns', round(d['north_star_roofline']['frac'],3))
"; }
python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/g1.json 2>/dev/null; show gpurun_out/g1.json
run 2 --steps 20 --warmup 5 --no-e2e > gpurun_out/g2.json 2>/dev/null; show gpurun_out/g2.json
run 4 --steps 20 --warmup 5 --no-e2e > gpurun_out/g4.json 2>/dev/null; show gpurun_out/g4.json
DFFT_NO_GRAPH=1 run 4 --steps 20 --warmup 5 --no-e2e > gpurun_out/g4n.json 2>/dev/null; show gpurun_out/g4n.json
