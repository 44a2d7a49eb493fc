SPPO_TRACE=gpurun_out/trace_fwd15.txt SPPO_TRACE_CHUNK=15 SPPO_TRACE_KIND=fwd timeout 300 python tools/trace_run.py 2>&1 | tail -12
