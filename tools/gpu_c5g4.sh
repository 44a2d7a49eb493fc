#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_persistent_bwd.py -q -x 2>&1 | tail -1
for g in 4 3; do
  SPPO_FWD_GROUP=$g timeout 1200 python bench.py --config C5 --shard-of 8 --steps 1 --warmup 1 --no-e2e --no-offload --no-cpu --no-c3 > gpurun_out/c5_g$g.json 2> gpurun_out/c5_g$g.err
  tail -1 gpurun_out/c5_g$g.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5 share group $g', d['value'], 'fwd', d['fwd_tflops'], 'bwd', d['bwd_tflops'], d['clocks']['sm_mhz'])"
done
