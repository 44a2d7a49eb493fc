#!/bin/bash
# Guarded smoke, backward parity subset, A/B vs variants (tools/make_variant.sh) and a bwd trace.
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1 || { echo smoke failed; tail gpurun_out/smoke.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_edge.py tests/test_gpu_policies.py tests/test_gpu_streams.py -q -x -m "gpu and not slow" -p no:cacheprovider > gpurun_out/pytest_bwd.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_bwd.log
bash tools/gpu_abn.sh "$@"
SPPO_TRACE=gpurun_out/trace_bwd.txt SPPO_TRACE_CHUNK=15 SPPO_TRACE_KIND=bwd timeout 120 python tools/trace_run.py > /dev/null 2>&1
python tools/trace_stats.py gpurun_out/trace_bwd.txt bwd 2>&1 | head -16
