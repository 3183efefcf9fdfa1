#!/bin/bash
# round-2 (session 2) check: GPU suite + smoke + default bench, then source-line ncu of both C5 passes
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
python tools/prof_call.py --config 5 --reps 2 > gpurun_out/plain5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_p1|k_p2" -s 2 -c 2 -o gpurun_out/prof_c5_src python tools/prof_call.py --config 5 --reps 2 > gpurun_out/ncu_c5_src.log 2>&1
python tools/ncu_lines_r2.py gpurun_out/prof_c5_src.ncu-rep 60 > gpurun_out/lines_c5.txt 2>&1
python tools/ncu_report.py gpurun_out/prof_c5_src.ncu-rep c5 > gpurun_out/ncu_c5_src.txt 2>&1
ncu -i gpurun_out/prof_c5_src.ncu-rep --page source --csv --print-source sass -k regex:k_p2 > gpurun_out/sass_p2.csv 2>&1
ncu -i gpurun_out/prof_c5_src.ncu-rep --page source --csv --print-source sass -k regex:k_p1 > gpurun_out/sass_p1.csv 2>&1
rm -f gpurun_out/prof_c5_src.ncu-rep
tail -3 gpurun_out/pytest_gpu.log
du -sh gpurun_out
