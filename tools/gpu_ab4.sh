#!/bin/bash
# parity subset + A/B + bwd item-boundary trace of the repo build
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_edge.py -q -x > gpurun_out/ab4_pytest.log 2>&1; tail -1 gpurun_out/ab4_pytest.log
for v in "$@"; do (cd tmp_$v && timeout 600 python -m pytest tests/test_gpu_bf16.py -q -x 2>&1 | tail -1 | sed "s/^/$v: /"); done 2>/dev/null
bash tools/gpu_abn.sh "$@" 2>&1 | tee gpurun_out/ab4.txt
for N in 64; do for d in . "${@/#/tmp_}"; do (cd $d && timeout 300 python tools/lib_attn_bench.py --impl sppo --seq 131072 --chunks $N 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d N=$N fwd', d['fwd_tflops'], 'bwd', d['bwd_tflops'])"); done; done
for d in . "${@/#/tmp_}"; do (cd $d && SPPO_TRACE=/tmp/tr_$$.txt SPPO_TRACE_CHUNK=15 SPPO_TRACE_KIND=bwd timeout 300 python tools/trace_run.py > /dev/null 2>&1; echo "$d"; python tools/trace_boundary.py /tmp/tr_$$.txt 64 | head -6 | tail -4); done
