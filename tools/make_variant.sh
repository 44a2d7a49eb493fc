#!/bin/bash
# Build a variant of libsppo with extra nvcc defines into tmp_<name>/ (a copy of
# the package + bench deps) for on-box A/B runs:  tools/make_variant.sh v3 -DSPPO_EMU_EVERY=3
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
dst=$root/tmp_$name
rm -rf $dst; mkdir -p $dst
cp -r $root/paper_2503_10377_b200 $root/synth $root/tools $root/include $root/examples $root/bench.py $dst/
mkdir -p $dst/tests && cp -r $root/tests/cuda $dst/tests/
rm -f $dst/paper_2503_10377_b200/libsppo.so
cd $dst && NVCC_EXTRA="$*" python -c "
import os, sys
sys.path.insert(0, '.')
from paper_2503_10377_b200 import build as b
b.BUILD = os.path.join('$dst', 'build')
b.FLAGS = b.FLAGS + os.environ['NVCC_EXTRA'].split()
b.build(force=True)
print('built', b.LIB)"
