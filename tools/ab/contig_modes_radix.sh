# A/B: radix-32 passes for the R2C / C2R / DCT / DST x-stages (libdfft_r32all.so) vs c2c only (default)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kinds.py -q -k "r2c or c2r or poisson or kinds or dct or dst or r2r" 2>&1 | tail -1
st() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  ', round(d['ms_per_step'],3), ' '.join(s['kernel'].split(' ')[1][:10] + '=' + str(round(s['avg_launch_ms'],3)) for s in d['roofline']['stages']))"; }
for lib in libdfft.so libdfft_r32all.so; do
  export DFFT_LIB=$PWD/paper_2601_12209_b200/$lib
  for kind in r2c r2r; do echo "$lib 1024^3 f32 $kind"; python bench.py --steps 10 --warmup 3 --kind $kind --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | st; done
  echo "$lib 512^3 f32 r2c"; python bench.py --steps 10 --warmup 3 --grid 512,512,512 --kind r2c --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | st
done
