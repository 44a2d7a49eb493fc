#!/bin/bash
# compute-sanitizer over the layer kernels (tools/sanitize_layer.py), default and forced-pair GEMM selection
mkdir -p gpurun_out
for t in memcheck synccheck racecheck; do
  timeout 600 compute-sanitizer --tool $t python tools/sanitize_layer.py > gpurun_out/san_layer_$t.txt 2>&1; echo $t; tail -1 gpurun_out/san_layer_$t.txt
  SPPO_GEMM_PAIR=2 timeout 600 compute-sanitizer --tool $t python tools/sanitize_layer.py > gpurun_out/san_layer_pair_$t.txt 2>&1; echo pair $t; tail -1 gpurun_out/san_layer_pair_$t.txt
done
