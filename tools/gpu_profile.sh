#!/bin/bash
# One gpurun call: bench lines (C2 default, C3) + ncu launch list of one C2 step
# + ncu --set full of the largest fwd/bwd launch (chunk 15 of a C2 step).
#   gpurun --timeout 3000 -- 'bash tools/gpu_profile.sh <tag>'
tag=${1:-r01}
mkdir -p gpurun_out
if [ "$2" != "ncu-only" ]; then
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2_$tag.json 2> gpurun_out/bench_c2_$tag.err
tail -1 gpurun_out/bench_c2_$tag.json | cut -c1-400
timeout 900 python bench.py --config C3 --steps 2 --warmup 3 --no-e2e --no-offload > gpurun_out/bench_c3_$tag.json 2> gpurun_out/bench_c3_$tag.err
tail -1 gpurun_out/bench_c3_$tag.json | cut -c1-300
fi
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_$tag.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-offload --no-cpu > /dev/null 2>&1
for k in bwd fwd; do
  skip=0   # bwd: chunk 15 = first launch (N-1 .. 0); fwd: the one multi-chunk launch of the step
  SPPO_TRACE_KIND=$k timeout 900 ncu --set full --clock-control none --import-source on -k regex:${k}_kernel \
    --launch-skip $skip -c 1 -f -o gpurun_out/prof_${k}_$tag python tools/trace_run.py > /dev/null 2>&1
  ncu -i gpurun_out/prof_${k}_$tag.ncu-rep --page details --csv > gpurun_out/prof_${k}_${tag}_details.csv 2>/dev/null
  ncu -i gpurun_out/prof_${k}_$tag.ncu-rep --page raw --csv > gpurun_out/prof_${k}_${tag}_raw.csv 2>/dev/null
done
ls -la gpurun_out | tail -12
