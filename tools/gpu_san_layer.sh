#!/bin/bash
# compute-sanitizer over the layer kernels (tools/sanitize_layer.py): default GEMM
# selection (CTA pair, 128-deep stages) and the single-CTA kernel (SPPO_GEMM_PAIR=0)
mkdir -p gpurun_out
for t in memcheck synccheck racecheck; do
  timeout 600 compute-sanitizer --tool $t python tools/sanitize_layer.py > gpurun_out/san_layer_$t.txt 2>&1; echo $t; tail -1 gpurun_out/san_layer_$t.txt
  SPPO_GEMM_PAIR=0 timeout 600 compute-sanitizer --tool $t python tools/sanitize_layer.py > gpurun_out/san_layer_single_$t.txt 2>&1; echo single $t; tail -1 gpurun_out/san_layer_single_$t.txt
done
