mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 900 python tools/abbench.py $AB_LIBS --configs ${AB_CFGS:-2,5} --rounds ${AB_ROUNDS:-2}
