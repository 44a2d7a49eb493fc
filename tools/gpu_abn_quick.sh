#!/bin/bash
# Guarded smoke, then interleaved A/B/n bench (tools/gpu_abn.sh) of tmp_<variant> dirs.
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1 || { echo smoke failed; tail gpurun_out/smoke.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_bf16.py -q -x -p no:cacheprovider 2>&1 | tail -1
bash tools/gpu_abn.sh "$@"
