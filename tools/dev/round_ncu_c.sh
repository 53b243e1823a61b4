#!/bin/bash
O=gpurun_out/nc; mkdir -p $O
timeout 600 ncu --set full --clock-control none -k regex:fft_strided_tma --launch-skip 16 --launch-count 1 -o /tmp/cst -f \
   python tools/sim_time.py 1024,1024,1024 2,2 p2p f32 1 > $O/ncu.log 2>&1
ncu -i /tmp/cst.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
ncu -i /tmp/cst.ncu-rep --page details --csv > $O/details.csv 2>/dev/null
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/nc/raw.csv')))
h=rows[0]; d=dict(zip(h,rows[2]))
for k in ['Kernel Name','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','lts__t_sectors_srcunit_tex_op_read.sum','launch__grid_size','sm__warps_active.avg.pct_of_peak_sustained_active']:
    print(k, d.get(k))
PY
