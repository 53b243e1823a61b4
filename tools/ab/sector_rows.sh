cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2 | head -1
for sh in "1024,1024,1024 f32" "720,720,720 f64" "720,720,720 f32" "480,480,480 f64" "840,840,840 f32" "768,768,768 f64"; do
  echo "== $sh"; python tools/quick_time.py $sh 2>/dev/null | tail -2
done
python bench.py --steps 10 --warmup 3 --grid 768,768,384 --precision f64 --kind r2c --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5 r2c N=1', d['ms_per_step']); [print('  ', s['kernel'][:50], round(s['avg_launch_ms'],3), round(s['frac'],3)) for s in d['roofline']['stages']]"
