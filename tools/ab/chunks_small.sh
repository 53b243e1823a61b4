# K sweep for the secondary configs at N=4 (the plan's size-based default vs explicit chunks)
cd $GRAFT_REPO_ROOT
run() { n=$1; shift; python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 500)) bench.py --gpus $n "$@"; }
ms() { python - "$1" <<'PY'
import json,sys
lines=[l for l in open(sys.argv[1]) if l.startswith('{')]
d=json.loads(lines[-1]); print(round(d['ms_per_step'],3), 'graph', round(d['timing']['cuda_graph_ms'],3), 'chunks', d['config'].get('chunks'))
PY
}
for cfg in "--grid 512,512,512" "--grid 768,768,384 --precision f64 --kind r2c"; do
  for k in 0 1 2 4; do printf "%s K=%s: " "$cfg" $k; run 4 --steps 20 --warmup 5 --no-e2e $cfg --chunks $k > /tmp/k.json 2>/dev/null; ms /tmp/k.json; done
done
