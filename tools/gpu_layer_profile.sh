#!/bin/bash
# One gpurun call: layer bench line (C2 shape) + ncu --set full of two layer GEMMs
# (fc1 forward: K-major x K-major; fc1 data gradient: K-major x MN-major).
#   gpurun --timeout 1800 -- 'bash tools/gpu_layer_profile.sh <tag>'
tag=${1:-r01}
mkdir -p gpurun_out
timeout 900 python bench.py --workload layer --steps 3 --warmup 3 > gpurun_out/bench_layer_c2_$tag.json 2> gpurun_out/bench_layer_c2_$tag.err
tail -1 gpurun_out/bench_layer_c2_$tag.json | cut -c1-300
for pair in "fc1fwd:23" "fc1dgrad:69"; do
  name=${pair%%:*}; skip=${pair##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel --launch-skip $skip -c 1 -f \
    -o gpurun_out/prof_gemm_${name}_$tag python tools/gemm_bench.py --iters 20 > /dev/null 2>&1
  ncu -i gpurun_out/prof_gemm_${name}_$tag.ncu-rep --page raw --csv > gpurun_out/prof_gemm_${name}_${tag}_raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_gemm_${name}_$tag.ncu-rep --page details --csv > gpurun_out/prof_gemm_${name}_${tag}_details.csv 2>/dev/null
done
ls -la gpurun_out | tail -8
