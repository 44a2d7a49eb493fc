#!/bin/bash
# One gpurun call after a layer-kernel change: layer tests, GEMM bench, layer bench line, ncu of two GEMMs.
#   gpurun --timeout 1800 -- 'bash tools/gpu_layer_round.sh <tag>'
tag=${1:-r01}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_layer_ops.py tests/test_gpu_layer.py tests/test_gpu_pipeline.py -q -x 2>&1 | tail -1
timeout 300 python tools/gemm_bench.py --iters 20 > gpurun_out/gemm_bench_$tag.jsonl 2>&1; cat gpurun_out/gemm_bench_$tag.jsonl | cut -c1-200
timeout 600 python bench.py --workload layer --steps 3 --warmup 3 > gpurun_out/bench_layer_c2_$tag.json 2> gpurun_out/bench_layer_c2_$tag.err
tail -1 gpurun_out/bench_layer_c2_$tag.json | cut -c1-400
for pair in "fc1fwd:23" "fc1dgrad:69"; do
  name=${pair%%:*}; skip=${pair##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm --launch-skip $skip -c 1 -f \
    -o gpurun_out/prof_gemm_${name}_$tag python tools/gemm_bench.py --iters 20 > /dev/null 2>&1
  ncu -i gpurun_out/prof_gemm_${name}_$tag.ncu-rep --page raw --csv > gpurun_out/prof_gemm_${name}_${tag}_raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_gemm_${name}_$tag.ncu-rep --page details --csv > gpurun_out/prof_gemm_${name}_${tag}_details.csv 2>/dev/null
done
