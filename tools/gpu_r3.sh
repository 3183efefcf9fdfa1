set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --extra-configs ''"
eval "$B" > gpurun_out/plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $B > gpurun_out/ncu_l.log 2>&1
eval "$B" > gpurun_out/plain_c2b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_p -s 8 -c 2 -o gpurun_out/prof_c2 $B > gpurun_out/ncu_f.log 2>&1
B5="python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --extra-configs ''"
eval "$B5" > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_p -s 8 -c 2 -o gpurun_out/prof_c5 $B5 > gpurun_out/ncu_f5.log 2>&1
tail -15 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/smoke.log; tail -3 gpurun_out/bench.log; tail -3 gpurun_out/ncu_f.log
