#!/bin/bash
# GEMM A/B on one box: tools/gemm_bench.py in the repo and in each tmp_<variant>/ dir
#   gpurun -- 'bash tools/gpu_gemm_ab.sh g4 g16'
for rep in 1 2; do
  for v in . "$@"; do
    d=$v; [ "$v" != "." ] && d=tmp_$v
    echo "== $v"; (cd $d && timeout 300 python tools/gemm_bench.py --iters 20 2>/dev/null | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print('%-10s %7.1f (cublas %7.1f)' % (d['gemm'], d['tflops'], d['cublas_tflops']))")
  done
done
