#!/bin/bash
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1 || { echo smoke failed; tail gpurun_out/smoke.log; exit 1; }
SPPO_TRACE=gpurun_out/trace_fwd64.txt SPPO_TRACE_CHUNK=15 SPPO_TRACE_KIND=fwd timeout 120 python tools/trace_run.py > /dev/null 2>&1
echo done
