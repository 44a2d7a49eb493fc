timeout 300 python -m pytest tests/test_gpu_bf16.py -q -x 2>&1 | tail -3
SPPO_TRACE=gpurun_out/trace_bwd15.txt SPPO_TRACE_CHUNK=15 SPPO_TRACE_KIND=bwd timeout 300 python tools/trace_run.py 2>&1 | tail -30
