#!/bin/bash
# Full GPU test suite as the driver runs it, then the default bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=25 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
tail -40 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_default.json
