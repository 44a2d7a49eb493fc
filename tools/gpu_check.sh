#!/bin/bash
# One gpurun call: GPU tests (fast set), then the default bench line.
#   gpurun --timeout 1500 -- 'bash tools/gpu_check.sh'
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m "gpu and not slow" 2>&1 | tail -3
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
tail -1 gpurun_out/bench_default.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d.get(k) for k in ('value','ms_per_step','fwd_tflops','bwd_tflops','e2e','offload','clocks')})"
