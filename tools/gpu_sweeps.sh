#!/bin/bash
# N-sweep of the C2 layer + the C5 per-GPU share (rank 0 of the 8-GPU head split), resident
mkdir -p gpurun_out
timeout 900 python tools/n_sweep.py > gpurun_out/n_sweep_persist.json 2> gpurun_out/n_sweep_persist.err
python -c "
import json; d=json.load(open('gpurun_out/n_sweep_persist.json'))
for r in d['sweep']: print(r['N'], r['chunk_len'], r['tflops'], r['fwd_tflops'], r['bwd_tflops'])"
timeout 1200 python bench.py --config C5 --shard-of 8 --steps 1 --warmup 1 --no-e2e --no-offload --no-cpu --no-c3 > gpurun_out/c5_share_persist.json 2> gpurun_out/c5_share_persist.err
tail -1 gpurun_out/c5_share_persist.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5 share', d['value'], 'fwd', d['fwd_tflops'], 'bwd', d['bwd_tflops'], d['clocks'])"
