#!/bin/bash
# Parity subset (two-stream backward included at small sizes), then the N-sweep.
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1 || { echo smoke failed; tail gpurun_out/smoke.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_edge.py tests/test_gpu_policies.py tests/test_gpu_streams.py tests/test_gpu_fp32.py -q -x -m "gpu and not slow" -p no:cacheprovider > gpurun_out/pytest_ns.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_ns.log
timeout 900 python tools/n_sweep.py > gpurun_out/n_sweep.json 2> gpurun_out/n_sweep.err; echo "sweep rc=$?"
python -c "import json; d=json.load(open('gpurun_out/n_sweep.json')); [print(r) for r in d['sweep']]"
