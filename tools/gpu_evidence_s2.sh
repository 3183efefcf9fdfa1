#!/bin/bash
# round-2 evidence on the committed code: GPU suite, smoke, the default bench line (C5 headline), the ncu
# launch list of the short bench, and ncu --set full captures of the pass kernels for C5 / C2 / C3 / C4
# (summaries + per-launch DRAM traffic for bench.py's roofline.traffic).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
if [ -z "$NO_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
B="python bench.py --steps 3 --warmup 3 --extra-configs none --no-shift-bench --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5.csv $B > gpurun_out/ncu_launches.log 2>&1
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
for c in 5 2 3 4; do
  case $c in 5) W=c5_full_f32_16x2048; K='k_p1|k_p2'; S=2; N=2;; 2) W=c2_full_f32_1024; K='k_p1|k_p2'; S=2; N=2;;
             3) W=c3_full_u8_64x512; K='k_p1|k_p2'; S=2; N=2;; 4) W=c4_range_f32_4096; K='k_p1|k_p2|k_range'; S=3; N=3;; esac
  python tools/prof_call.py --config $c > gpurun_out/plain$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none -k regex:"$K" -s $S -c $N -o gpurun_out/prof_c$c python tools/prof_call.py --config $c > gpurun_out/ncu_c$c.log 2>&1
  python tools/ncu_report.py gpurun_out/prof_c$c.ncu-rep $W > gpurun_out/ncu_c${c}.txt 2>&1
  python tools/ncu_summary.py gpurun_out/prof_c$c.ncu-rep $W --traffic gpurun_out/ncu_traffic.json > gpurun_out/sum_c$c.txt 2>&1
  rm -f gpurun_out/prof_c$c.ncu-rep
done
python tools/prof_call.py --config 5 --single > gpurun_out/plain5s.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:k_p2 -s 1 -c 1 -o gpurun_out/prof_c5s python tools/prof_call.py --config 5 --single > gpurun_out/ncu_c5s.log 2>&1
python tools/ncu_report.py gpurun_out/prof_c5s.ncu-rep c5_single > gpurun_out/ncu_c5s.txt 2>&1
rm -f gpurun_out/prof_c5s.ncu-rep
tail -3 gpurun_out/pytest_gpu.log; du -sh gpurun_out
