mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --extra-configs none"
$B > gpurun_out/plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $B > gpurun_out/ncu_l.log 2>&1
$B > gpurun_out/plain_c2b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_p -s 8 -c 2 -o gpurun_out/prof_c2 $B > gpurun_out/ncu_f.log 2>&1
B5="python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --extra-configs none"
$B5 > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_p -s 64 -c 2 -o gpurun_out/prof_c5 $B5 > gpurun_out/ncu_f5.log 2>&1
tail -2 gpurun_out/ncu_f.log gpurun_out/ncu_f5.log gpurun_out/ncu_l.log
