timeout 300 python -m pytest tests/test_gpu_executor.py -q -m gpu -x -k "fused_xy" 2>&1 | tail -3
echo "xpct 50"; timeout 120 python tools/quick_time.py 1024,1024,1024 f32 10 2>&1 | tail -2
echo "f64"; timeout 120 python tools/quick_time.py 1024,1024,512 f64 10 2>&1 | tail -2
echo "f64 classic"; DFFT_NO_FUSED_XY=1 timeout 120 python tools/quick_time.py 1024,1024,512 f64 10 2>&1 | tail -2
echo "512^3"; timeout 120 python tools/quick_time.py 512,512,512 f32 10 2>&1 | tail -2
echo "512^3 classic"; DFFT_NO_FUSED_XY=1 timeout 120 python tools/quick_time.py 512,512,512 f32 10 2>&1 | tail -2
