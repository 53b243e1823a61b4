cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_executor.py -q -x 2>&1 | tail -2
for rep in 1 2; do
for lib in libdfft.so libdfft_nh.so; do
  echo "== $lib"; DFFT_LIB=$PWD/paper_2601_12209_b200/$lib python tools/quick_time.py 1024,1024,1024 f32 10 2>&1 | tail -2
done; done
for sh in "2048,512,512 f32" "1024,512,512 f64" "512,512,512 f64" "768,768,768 f64" "1024,1024,512 f64"; do
  echo "== $sh xz8 / whole-axis"; python tools/quick_time.py $sh 2>/dev/null | tail -2 ; DFFT_NO_XZ8=1 python tools/quick_time.py $sh 2>/dev/null | tail -2
done
