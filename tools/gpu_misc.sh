#!/bin/bash
# Descriptor recycle stress test, then the MSP layer bench (layer-balanced partition).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_streams.py -q -x -p no:cacheprovider > gpurun_out/pytest_streams.log 2>&1
echo "streams rc=$?"; tail -3 gpurun_out/pytest_streams.log
bash tools/gpu_msp.sh
