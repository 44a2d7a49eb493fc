#!/bin/bash
mkdir -p gpurun_out
SPPO_TRACE=gpurun_out/trace_pb_n16.txt SPPO_TRACE_CHUNK=15 SPPO_TRACE_KIND=bwd timeout 300 python tools/trace_run.py > /dev/null 2>&1
python tools/trace_boundary.py gpurun_out/trace_pb_n16.txt 64
