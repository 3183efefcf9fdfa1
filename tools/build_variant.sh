#!/bin/bash
# Build an A/B variant of libfht.so: tools/build_variant.sh NAME "-DFHT_X=0 ..." -> build/ab/NAME.so
set -e
cd "$(dirname "$0")/.."
mkdir -p build/ab
python -c "
import sys; sys.path.insert(0, '.')
import __graft_entry__ as g
import os; g.build(out=os.path.abspath('build/ab/$1.so'), extra_flags='$2'.split(), load=False)
"
