#!/bin/bash
# parity subset + interleaved A/B (variants tmp_<v>) + the N=4 / N=64 splits of the C2 layer
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_edge.py tests/test_gpu_policies.py tests/test_gpu_streams.py -q -x > gpurun_out/ab3_pytest.log 2>&1; tail -1 gpurun_out/ab3_pytest.log
bash tools/gpu_abn.sh "$@" 2>&1 | tee gpurun_out/ab3.txt
for N in 4 64; do for d in . "${@/#/tmp_}"; do (cd $d && timeout 300 python tools/lib_attn_bench.py --impl sppo --seq 131072 --chunks $N 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d N=$N bwd', d['bwd_tflops'])"); done; done
