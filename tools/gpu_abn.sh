#!/bin/bash
# A/B/n on one box: bench (C2, kernels only) in the repo and in each tmp_<variant>/ dir, interleaved.
#   gpurun -- 'bash tools/gpu_abn.sh v3 v2 ...'
run() { (cd $1 && timeout 600 python bench.py --steps 4 --warmup 3 --no-e2e --no-offload --no-cpu --no-c3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%-6s step %7.1f fwd %7.1f bwd %7.1f  %s MHz' % ('$2', d['value'], d['fwd_tflops'], d['bwd_tflops'], d['clocks']['sm_mhz']))"); }
for rep in 1 2; do
  run . base
  for v in "$@"; do run tmp_$v $v; done
done
