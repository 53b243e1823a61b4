#!/bin/bash
O=gpurun_out/e; mkdir -p $O
# 1-GPU strided kernels under ncu --set full (raw csv only; reports stay on the box)
timeout 600 ncu --set full --clock-control none -k regex:fft_strided_tma --launch-skip 0 --launch-count 2 -o /tmp/single -f \
   python tools/quick_time.py 1024,1024,1024 f32 1 > $O/ncu1.log 2>&1
ncu -i /tmp/single.ncu-rep --page raw --csv > $O/raw_single.csv 2>/dev/null
ncu -i /tmp/single.ncu-rep --page details --csv > $O/details_single.csv 2>/dev/null
# the paper's GPU shapes (radix 5/7) and BASELINE configs at N=1
for g in 480,480,480 720,720,720 840,840,840 512,512,512 256,256,256; do
  for p in f32 f64; do
    echo "== $g $p" >> $O/shapes.log
    timeout 300 python bench.py --grid $g --precision $p --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' >> $O/shapes.log
  done
done
cat $O/shapes.log | python -c "
import sys,json
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print(d['config']['workload'], round(d['ms_per_step'],3), 'ms', round(d['value']), 'GFLOP/s', round(d['north_star_roofline']['frac'],3))
  else: print(l.strip())"
