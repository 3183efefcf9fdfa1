#!/bin/bash
# Per-choice before/after ncu lines: for each variant build (one choice off, build/ab/*.so, from
# tools/build_choice_variants.sh) and the default build, one ncu pass over C5's two kernels and C2's, recording
# duration, DRAM bytes, warp-instructions and issue activity per kernel.
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active
for lib in paper_1811_06378_b200/libfht.so build/ab/*.so; do
  name=$(basename $lib .so)
  for c in 5 2; do
    FHT_LIB=$lib python tools/prof_call.py --config $c --reps 2 > /dev/null 2>&1 || { echo "$name C$c plain run failed"; continue; }
    FHT_LIB=$lib ncu --metrics $M --clock-control none -k regex:"k_p1|k_p2" -s 2 -c 2 --csv \
      python tools/prof_call.py --config $c --reps 2 > gpurun_out/choice_${name}_c$c.csv 2> /dev/null
  done
done
ls gpurun_out/choice_*.csv | wc -l
