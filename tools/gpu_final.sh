# Round-end style evidence: GPU tests, smoke, default bench, ncu launch list + full capture of the
# dominant kernels for C2 and C5 (each ncu run only after the identical command exited 0).
mkdir -p gpurun_out/final
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1
S=$(date +%s); timeout 900 python bench.py > gpurun_out/final/bench.json 2>gpurun_out/final/bench.err; echo "default bench wall $(( $(date +%s) - S )) s" > gpurun_out/final/bench_wall.txt
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-shift-bench --extra-configs none"
$B > gpurun_out/final/plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches_c2.csv $B > gpurun_out/final/ncu_l.log 2>&1
# full capture of the launch the roofline describes: one stream, merged 4-slot pass pair (eager)
BM="$B --no-graph --no-aux"
$BM > gpurun_out/final/plain_c2b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_p -s 8 -c 2 -o gpurun_out/final/prof_c2 $BM > gpurun_out/final/ncu_f2.log 2>&1
# C5: the whole batch is one chunk; one stream so the captured pair is the per-kernel loop's launch
B5="python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-shift-bench --extra-configs none --no-aux"
$B5 > gpurun_out/final/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_p -s 6 -c 2 -o gpurun_out/final/prof_c5 $B5 > gpurun_out/final/ncu_f5.log 2>&1
B4="python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-shift-bench --extra-configs none"
$B4 > gpurun_out/final/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_p -s 8 -c 2 -o gpurun_out/final/prof_c4 $B4 > gpurun_out/final/ncu_f4.log 2>&1
tail -3 gpurun_out/final/pytest_gpu.log gpurun_out/final/smoke.log; tail -c 400 gpurun_out/final/bench.json
