for g in "2 2" "2 4"; do
  set -- $g
  python tools/sim_stage_traffic.py $1 $2 > gpurun_out/sim_${1}x${2}_plain.txt 2>&1 || { cat gpurun_out/sim_${1}x${2}_plain.txt; continue; }
  cat gpurun_out/sim_${1}x${2}_plain.txt
  ns=$(grep -o "[0-9]* stage launches" gpurun_out/sim_${1}x${2}_plain.txt | cut -d' ' -f1)
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"fft_(strided|contig|generic)" \
      -s $ns -c $ns --csv --log-file gpurun_out/sim_${1}x${2}_ncu.csv python tools/sim_stage_traffic.py $1 $2 > /dev/null 2>&1
  wc -l gpurun_out/sim_${1}x${2}_ncu.csv
done
