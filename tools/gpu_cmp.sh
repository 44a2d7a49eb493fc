#!/bin/bash
mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_policies.py tests/test_gpu_edge.py -q -x -m "not slow" 2>&1 | tail -3
export SPPO_TRACE_CHUNK=15 SPPO_TRACE_KIND=bwd
SPPO_TRACE=gpurun_out/trace_new.txt timeout 300 python tools/trace_run.py > /dev/null 2>&1
echo NEW; python tools/trace_stats.py gpurun_out/trace_new.txt
bash tools/gpu_ab.sh
