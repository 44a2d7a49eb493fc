#!/bin/bash
# Source-level (per-SASS) ncu captures of the chunk-15 fwd / bwd launches of a C2 step:
# warp-stall samples and shared-memory wavefronts per instruction.
#   gpurun --timeout 1800 -- 'bash tools/gpu_src.sh <tag> [fwd] [bwd]'
tag=$1; shift
mkdir -p gpurun_out
for k in "$@"; do
  skip=15; [ $k = bwd ] && skip=0
  SPPO_TRACE_KIND=$k SPPO_FWD_MULTI=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:${k}_kernel \
    --launch-skip $skip -c 1 -f -o gpurun_out/src_${k}_$tag python tools/trace_run.py > gpurun_out/src_${k}_$tag.log 2>&1
  ncu -i gpurun_out/src_${k}_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${k}_${tag}_sass.csv 2>/dev/null
  ncu -i gpurun_out/src_${k}_$tag.ncu-rep --page raw --csv > gpurun_out/src_${k}_${tag}_raw.csv 2>/dev/null
  rm -f gpurun_out/src_${k}_$tag.ncu-rep
done
ls -la gpurun_out | tail -5
