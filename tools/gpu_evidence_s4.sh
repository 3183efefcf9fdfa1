# Round-2 session-4 evidence (persistent pass 1): GPU suite, smoke, default bench, ncu launch list and full
# captures of the C5 pass kernels (each ncu run only after the identical command exited 0); then the GPU suite and
# tools/sanitize_cases.py under the bounds-checked build (build/libfht_checks.so, tools/checks_build.py).
O=gpurun_out/s4
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
S=$(date +%s); timeout 900 python bench.py > $O/bench.json 2>$O/bench.err; echo "default bench wall $(( $(date +%s) - S )) s" > $O/bench_wall.txt
B5="python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-shift-bench --extra-configs none --no-aux"
$B5 > $O/plain_c5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv $B5 > $O/ncu_l5.log 2>&1
$B5 > $O/plain_c5b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_p -s 6 -c 2 -o $O/prof_c5 $B5 > $O/ncu_f5.log 2>&1
if [ -f build/libfht_checks.so ]; then
  FHT_LIB=build/libfht_checks.so timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $O/pytest_gpu_checks.log
  FHT_LIB=build/libfht_checks.so timeout 600 python tools/sanitize_cases.py > $O/checks_cases.log 2>&1
fi
tail -n 3 $O/pytest_gpu.log $O/smoke.log $O/pytest_gpu_checks.log $O/checks_cases.log; tail -c 300 $O/bench.json
