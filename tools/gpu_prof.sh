mkdir -p gpurun_out
B="python bench.py --config ${CFG:-2} --steps 3 --warmup 3 --no-cpu-baseline --extra-configs none"
$B > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_p -s ${SKIP:-8} -c 2 -o gpurun_out/${OUT:-prof} $B > gpurun_out/ncu_f.log 2>&1
tail -2 gpurun_out/ncu_f.log
