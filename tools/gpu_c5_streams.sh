#!/bin/bash
# C5 per-GPU share (rank 0 of 8), full KV offload grouped by 2: forward on 1 vs 2 streams.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_policies.py tests/test_gpu_streams.py -q -x -p no:cacheprovider 2>&1 | tail -1
for fs in 2 1; do
  timeout 1500 python bench.py --config C5 --shard-of 8 --kv-hot 0 --kv-window 8 --kv-group 2 --fwd-streams $fs \
    --steps 1 --warmup 1 --no-e2e --no-offload --no-cpu --no-c3 > gpurun_out/c5_fs$fs.json 2> gpurun_out/c5_fs$fs.err
  tail -1 gpurun_out/c5_fs$fs.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kv_stream']; print('fwd_streams $fs: resident', d['value'], 'fwd', d['fwd_tflops'], 'bwd', d['bwd_tflops'], '| kv grouped ms', k['ms_per_step'], 'resident ms', k['resident_ms_per_step'], 'exposed', k['exposed_pct'], d['clocks']['sm_mhz'])"
done
