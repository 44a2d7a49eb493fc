#!/bin/bash
# Forward kernel trace (CTA (0,0) of chunk 15 at C2) + per-phase medians.
mkdir -p gpurun_out
free -g > gpurun_out/free.txt
SPPO_TRACE=gpurun_out/trace_fwd.txt SPPO_TRACE_CHUNK=15 SPPO_TRACE_KIND=fwd timeout 300 python tools/trace_run.py > gpurun_out/trace_fwd_run.txt 2>&1
python tools/trace_stats.py gpurun_out/trace_fwd.txt fwd > gpurun_out/trace_fwd_stats.txt 2>&1
cat gpurun_out/trace_fwd_stats.txt
