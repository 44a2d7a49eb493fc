#!/bin/bash
# grouped multi-chunk forward: tests + C5 per-GPU share resident (groups of 3 = ~10 waves) vs per-chunk
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_persistent_bwd.py -q -x 2>&1 | tail -1
for m in 1 0; do
  SPPO_FWD_MULTI=$m timeout 1200 python bench.py --config C5 --shard-of 8 --steps 1 --warmup 1 --no-e2e --no-offload --no-cpu --no-c3 > gpurun_out/c5_group$m.json 2> gpurun_out/c5_group$m.err
  tail -1 gpurun_out/c5_group$m.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5 share FWD_MULTI=$m (groups)', d['value'], 'fwd', d['fwd_tflops'], 'bwd', d['bwd_tflops'], d['clocks']['sm_mhz'])"
done
