run() { n=$1; shift; python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 500)) bench.py --gpus $n "$@"; }
show() { python -c "
import json,sys
lines=[l for l in open('$1') if l.startswith('{')]
d=json.loads(lines[-1]); t=d['timing']; p=d['phase_ms_per_step']
print('$2', 'b2b', round(t['back_to_back_ms'],3), 'fwd', round(t['forward_only_ms']['median'],3), ' '.join(f'{k}={v:.2f}' for k,v in p.items()))
"; }
for sms in 64 96 112; do DFFT_NVL_SMS=$sms run 4 --steps 10 --warmup 3 --no-e2e --no-graph > gpurun_out/s.json 2>/dev/null; show gpurun_out/s.json "sms=$sms"; done
for k in 2 8; do run 4 --steps 10 --warmup 3 --no-e2e --no-graph --chunks $k > gpurun_out/s.json 2>/dev/null; show gpurun_out/s.json "K=$k"; done
