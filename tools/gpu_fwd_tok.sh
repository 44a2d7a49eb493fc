#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_edge.py tests/test_gpu_persistent_bwd.py -q -x > gpurun_out/tok_pytest.log 2>&1; tail -1 gpurun_out/tok_pytest.log
bash tools/gpu_abn.sh "$@" 2>&1 | tee gpurun_out/ab_tok.txt
SPPO_FWD_MULTI=0 SPPO_TRACE=gpurun_out/trace_fwd_tok.txt SPPO_TRACE_CHUNK=15 SPPO_TRACE_KIND=fwd timeout 300 python tools/trace_run.py 2>&1 | tail -16
