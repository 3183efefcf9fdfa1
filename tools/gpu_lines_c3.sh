#!/bin/bash
# source-line / SASS-region profile of C3's pass kernels (where the L1-bound passes spend their instructions)
mkdir -p gpurun_out
python tools/prof_call.py --config 3 --reps 2 > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_p1|k_p2" -s 2 -c 2 -o gpurun_out/prof_c3_src python tools/prof_call.py --config 3 --reps 2 > gpurun_out/ncu_c3_src.log 2>&1
ncu -i gpurun_out/prof_c3_src.ncu-rep --page source --csv --print-source sass -k regex:k_p2 > gpurun_out/sass_c3_p2.csv 2>&1
ncu -i gpurun_out/prof_c3_src.ncu-rep --page source --csv --print-source sass -k regex:k_p1 > gpurun_out/sass_c3_p1.csv 2>&1
ncu -i gpurun_out/prof_c3_src.ncu-rep --page details --csv 2>/dev/null | grep -i -E "Bank Conflicts|shared" | head -20 > gpurun_out/ncu_c3_smem.txt
rm -f gpurun_out/prof_c3_src.ncu-rep
ls -la gpurun_out/*.csv
