#!/bin/bash
# Parity subset + interleaved A/B of variants (tools/make_variant.sh) + source-level ncu
# of the bwd kernel (per-SASS shared-memory wavefronts / stalls).
#   gpurun --timeout 2400 -- 'bash tools/gpu_ab_src.sh <tag> v1 v2 ...'
tag=$1; shift
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_edge.py -q -x > gpurun_out/ab_${tag}_pytest.log 2>&1; tail -1 gpurun_out/ab_${tag}_pytest.log
bash tools/gpu_abn.sh "$@" 2>&1 | tee gpurun_out/ab_${tag}.txt
SPPO_TRACE_KIND=bwd timeout 900 ncu --set full --clock-control none --import-source on -k regex:bwd_kernel \
  --launch-skip 0 -c 1 -f -o gpurun_out/src_bwd_$tag python tools/trace_run.py > /dev/null 2>&1
ncu -i gpurun_out/src_bwd_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/src_bwd_${tag}_sass.csv 2>/dev/null
ncu -i gpurun_out/src_bwd_$tag.ncu-rep --page raw --csv > gpurun_out/src_bwd_${tag}_raw.csv 2>/dev/null
rm -f gpurun_out/src_bwd_$tag.ncu-rep
ls -la gpurun_out | tail -5
