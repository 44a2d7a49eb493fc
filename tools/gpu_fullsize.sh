#!/bin/bash
# Full-size parity of every timed configuration (tests/test_gpu_fullsize.py).
mkdir -p gpurun_out
free -g > gpurun_out/free.txt
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -v -p no:cacheprovider --durations=10 -x ${1:+-k "$1"} > gpurun_out/pytest_fullsize.log 2>&1
echo "rc=$?"; tail -30 gpurun_out/pytest_fullsize.log
