#!/bin/bash
# round-2 ncu evidence: launch list of the short default bench, full captures of the top kernels
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --extra-configs none --no-shift-bench --no-cpu-baseline"
$B > gpurun_out/bench_short.json 2> gpurun_out/bench_short.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5.csv $B > gpurun_out/ncu_launches.log 2>&1
python tools/prof_call.py --config 5 > gpurun_out/plain5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_p2 -s 1 -c 1 -o gpurun_out/prof_c5_p2 python tools/prof_call.py --config 5 > gpurun_out/ncu_c5_p2.log 2>&1
python tools/prof_call.py --config 5 --single > gpurun_out/plain5s.log 2>&1 && \
ncu --set full --clock-control none -k regex:k_p2 -s 1 -c 1 -o gpurun_out/prof_c5s_p2 python tools/prof_call.py --config 5 --single > gpurun_out/ncu_c5s_p2.log 2>&1
python tools/prof_call.py --config 2 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_p1|k_p2" -s 2 -c 2 -o gpurun_out/prof_c2 python tools/prof_call.py --config 2 > gpurun_out/ncu_c2.log 2>&1
python tools/prof_call.py --config 3 > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none -k regex:"k_p1|k_p2" -s 2 -c 2 -o gpurun_out/prof_c3 python tools/prof_call.py --config 3 > gpurun_out/ncu_c3.log 2>&1
python tools/prof_call.py --config 4 > gpurun_out/plain4.log 2>&1 && \
ncu --set full --clock-control none -k regex:"k_p1|k_p2|k_range" -s 3 -c 3 -o gpurun_out/prof_c4 python tools/prof_call.py --config 4 > gpurun_out/ncu_c4.log 2>&1
ls -la gpurun_out/*.ncu-rep
# summarise on the box and keep only the C5 / C2 reports (gpurun brings back <= 64 MiB)
for r in c5_p2 c5s_p2 c2 c3 c4; do
  python tools/ncu_report.py gpurun_out/prof_$r.ncu-rep "$r" > gpurun_out/ncu_$r.txt 2>&1
done
python tools/ncu_summary.py gpurun_out/prof_c5_p2.ncu-rep c5_full_f32_16x2048 > gpurun_out/sum_c5.txt 2>&1
python tools/ncu_summary.py gpurun_out/prof_c2.ncu-rep c2_full_f32_1024 > gpurun_out/sum_c2.txt 2>&1
python tools/ncu_summary.py gpurun_out/prof_c3.ncu-rep c3_full_u8_64x512 > gpurun_out/sum_c3.txt 2>&1
python tools/ncu_summary.py gpurun_out/prof_c4.ncu-rep c4_range_f32_4096 > gpurun_out/sum_c4.txt 2>&1
rm -f gpurun_out/prof_c5s_p2.ncu-rep gpurun_out/prof_c3.ncu-rep gpurun_out/prof_c4.ncu-rep
du -sh gpurun_out
