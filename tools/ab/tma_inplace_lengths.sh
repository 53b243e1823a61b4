# per-length A/B of the in-place TMA variant: xz8 M-point z passes (nz = 8·M) and whole-axis y passes
cd $GRAFT_REPO_ROOT
for sh in "512,512,384 f32" "1024,512,768 f32" "512,512,1024 f32" "512,512,1536 f32" "512,256,2048 f32" "256,256,3072 f32" \
          "512,384,256 f32" "512,768,256 f32" "512,1024,256 f32" "256,1536,256 f32" "512,512,384 f64" "512,512,1024 f64" "512,768,128 f64" "512,1024,128 f64"; do
  for ip in 1 0; do printf "%-22s IP=%s " "$sh" $ip; DFFT_TMA_IP=$ip python tools/quick_time.py $sh 5 2>/dev/null | tail -1; done
done
