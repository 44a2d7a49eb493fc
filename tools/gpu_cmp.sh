#!/bin/bash
# One gpurun call for a kernel change: fast GPU tests, a bwd (or fwd) trace of C2
# chunk 15 with per-phase medians, and an interleaved bench A/B against variants
# built by tools/make_variant.sh.   gpurun -- 'bash tools/gpu_cmp.sh bwd v1 v2'
kind=${1:-bwd}; shift
mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_policies.py tests/test_gpu_edge.py -q -x -m "not slow" 2>&1 | tail -1
SPPO_TRACE=gpurun_out/trace_$kind.txt SPPO_TRACE_CHUNK=15 SPPO_TRACE_KIND=$kind timeout 300 python tools/trace_run.py > /dev/null 2>&1
python tools/trace_stats.py gpurun_out/trace_$kind.txt $kind
[ $# -gt 0 ] && bash tools/gpu_abn.sh "$@"
