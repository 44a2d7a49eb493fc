#!/bin/bash
# pair-kernel variants: correctness (forced pair) + A/B of the GEMM bench, default and forced-pair selection
for v in "$@"; do (cd tmp_$v && SPPO_GEMM_PAIR=2 timeout 300 python -m pytest tests/test_gpu_layer_ops.py tests/test_gpu_layer.py -q -x -k "not gpt7b" 2>&1 | tail -1); done
for rep in 1 2; do
  for v in . "$@"; do
    d=$v; [ "$v" != "." ] && d=tmp_$v
    for pe in 1 2; do
      echo "== $v pair=$pe"; (cd $d && SPPO_GEMM_PAIR=$pe timeout 300 python tools/gemm_bench.py --iters 20 2>/dev/null | python -c "
import json,sys
print('  '.join('%s %.0f' % (d['gemm'].replace(' ',''), d['tflops']) for d in map(json.loads, sys.stdin)))")
    done
  done
done
