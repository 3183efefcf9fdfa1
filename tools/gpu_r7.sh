mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --cpu-seconds 2 > gpurun_out/bench.log 2>&1; python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1])
print('C2', d['ms_per_step'], 'step frac', d['step_roofline']['frac'], 'p2 frac', d['roofline']['frac'], d['kernels'])
for k,v in d['configs'].items(): print(k, v.get('ms_per_step'), 'step', v.get('step_frac_of_measured_hbm'), 'p2', v.get('pass2_frac_of_measured_hbm'), v.get('kernels'))
PY
