# A/B: in-place TMA-store variant (three stages in flight) vs the work-tile kernel (DFFT_TMA_IP=0)
cd $GRAFT_REPO_ROOT
timeout 1000 python -m pytest tests -q -m gpu 2>&1 | tail -1
for rep in 1 2; do
  for ip in 1 0; do echo "== DFFT_TMA_IP=$ip"; DFFT_TMA_IP=$ip python tools/quick_time.py 1024,1024,1024 f32 10 2>&1 | tail -2; done
done
for sh in "768,768,768 f64" "512,512,512 f32" "768,768,768 f32"; do
  for ip in 1 0; do echo "== $sh IP=$ip"; DFFT_TMA_IP=$ip python tools/quick_time.py $sh 2>/dev/null | tail -2; done
done
