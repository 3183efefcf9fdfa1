mkdir -p gpurun_out
for c in "7 9 u8 0" "64 300 f32 0" "300 64 f32 2" "300 700 f32 1" "300 700 u8 3"; do
  echo "== $c"; CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/dbg_case.py $c 2>&1 | grep -E "^ok|Error|error" | head -3
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
tail -30 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --cpu-seconds 2 > gpurun_out/bench.log 2>&1; tail -c 3000 gpurun_out/bench.log
