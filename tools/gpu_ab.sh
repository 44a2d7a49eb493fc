#!/bin/bash
# Parity subset on the repo build + interleaved A/B of variants (tools/make_variant.sh).
#   gpurun --timeout 1800 -- 'bash tools/gpu_ab.sh <tag> v1 v2 ...'
tag=$1; shift
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_edge.py -q -x > gpurun_out/ab_${tag}_pytest.log 2>&1; tail -1 gpurun_out/ab_${tag}_pytest.log
bash tools/gpu_abn.sh "$@" 2>&1 | tee gpurun_out/ab_${tag}.txt
