#!/bin/bash
# A/B: tmp_old (previous commit's build) vs the working tree, interleaved bench runs.
mkdir -p gpurun_out
run() { timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-offload --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', {k:d[k] for k in ('value','fwd_tflops','bwd_tflops')}, d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'))"; }
for i in 1 2; do
  (cd tmp_old && cp ../bench.py . 2>/dev/null; run OLD)
  run NEW
done
