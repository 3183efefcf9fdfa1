mkdir -p gpurun_out
B="python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline --extra-configs none"
$B > gpurun_out/plain_c5d.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none -k regex:k_p -s 40 -c 8 --csv --log-file gpurun_out/dram_c5.csv $B > gpurun_out/ncu_d.log 2>&1
tail -2 gpurun_out/ncu_d.log
