timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/abbench.py build/ab/base.so build/ab/aux.so --configs 3,5 --rounds 1
AB_AUX=1 timeout 600 python tools/abbench.py build/ab/aux.so --configs 3,5,2 --rounds 1
