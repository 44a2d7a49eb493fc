#!/bin/bash
# C5 per-GPU share (resident): forward as one multi-chunk launch vs per-chunk launches
mkdir -p gpurun_out
for m in 0 1; do
  SPPO_FWD_MULTI=$m timeout 1200 python bench.py --config C5 --shard-of 8 --steps 1 --warmup 1 --no-e2e --no-offload --no-cpu --no-c3 > gpurun_out/c5_multi$m.json 2> gpurun_out/c5_multi$m.err
  tail -1 gpurun_out/c5_multi$m.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5 share FWD_MULTI=$m', d['value'], 'fwd', d['fwd_tflops'], 'bwd', d['bwd_tflops'], d['clocks']['sm_mhz'])"
done
