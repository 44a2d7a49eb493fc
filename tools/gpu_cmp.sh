#!/bin/bash
mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_gpu_bf16.py -q -x 2>&1 | tail -3
export SPPO_TRACE_CHUNK=15 SPPO_TRACE_KIND=bwd
SPPO_TRACE=gpurun_out/trace_new.txt timeout 300 python tools/trace_run.py > /dev/null 2>&1
echo NEW; python tools/trace_stats.py gpurun_out/trace_new.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-offload --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ('value','ms_per_step','fwd_tflops','bwd_tflops','clocks')})"
