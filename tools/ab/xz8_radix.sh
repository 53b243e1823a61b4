# A/B of the xz8 kernel variants (dev builds via DFFT_LIB); same box, interleaved
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "xz8 or headline" 2>&1 | tail -2
for rep in 1 2; do
for lib in libdfft.so libdfft_m3.so libdfft_r16.so; do
  echo "== $lib"; DFFT_LIB=$PWD/paper_2601_12209_b200/$lib python tools/quick_time.py 1024,1024,1024 f32 10 2>&1 | tail -2
done; done
for lib in libdfft.so libdfft_m3.so; do
  echo "== $lib 2048x512x512 / 512^3"; DFFT_LIB=$PWD/paper_2601_12209_b200/$lib python tools/quick_time.py 2048,512,512 f32 10 2>&1 | tail -2
  DFFT_LIB=$PWD/paper_2601_12209_b200/$lib python tools/quick_time.py 512,512,512 f32 10 2>&1 | tail -2
done
