timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "generic" 2>&1 | tail -3
run() { n=$1; shift; python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 500)) bench.py --gpus $n "$@"; }
show() { python -c "
import json,sys
lines=[l for l in open('$1') if l.startswith('{')]
d=json.loads(lines[-1]); t=d['timing']; p=d['phase_ms_per_step']
print('$2', 'b2b', round(t['back_to_back_ms'],3), 'fwd', round(t['forward_only_ms']['median'],3), ' '.join(f'{k}={v:.2f}' for k,v in p.items()))
"; }
for k in 4 8 16; do for sms in 80 96; do DFFT_NVL_SMS=$sms run 4 --steps 10 --warmup 3 --no-e2e --no-graph --chunks $k > gpurun_out/s.json 2>/dev/null; show gpurun_out/s.json "graph K=$k sms=$sms"; done; done
for k in 4 8; do run 2 --steps 10 --warmup 3 --no-e2e --no-graph --chunks $k > gpurun_out/s.json 2>/dev/null; show gpurun_out/s.json "N=2 graph K=$k"; done
