cd $GRAFT_REPO_ROOT
timeout 1000 python -m pytest tests -q -m gpu 2>&1 | tail -1
for sh in "1024,1024,1024 f32"; do python tools/quick_time.py $sh 2>/dev/null | tail -2; DFFT_NO_XZ8=1 python tools/quick_time.py $sh 2>/dev/null | tail -2; done
python bench.py --steps 10 --warmup 3 --grid 768,768,384 --precision f64 --kind r2c --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5 r2c N=1', d['ms_per_step']); [print('  ', s['kernel'][:50], round(s['avg_launch_ms'],3), round(s['frac'],3)) for s in d['roofline']['stages']]"
python bench.py --steps 20 --warmup 5 2>/dev/null | tail -1 > gpurun_out/b1.json; python -c "import json; d=json.loads(open('gpurun_out/b1.json').read()); print('N=1', d['ms_per_step'], 'e2e', d['e2e']['ms_per_step'], d['clocks'])"
