#!/bin/bash
# Persistent bwd: parity (bf16/edge/policies/streams) + A/B against the per-item-launch build (tmp_old)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_edge.py tests/test_gpu_policies.py tests/test_gpu_streams.py -q -x > gpurun_out/persist_pytest.log 2>&1; tail -3 gpurun_out/persist_pytest.log
grep -E "FAIL|Error|error" gpurun_out/persist_pytest.log | head -5
bash tools/gpu_abn.sh old 2>&1 | tee gpurun_out/ab_persist.txt
for N in 64 4; do
  for d in . tmp_old; do (cd $d && timeout 300 python tools/lib_attn_bench.py --impl sppo --seq 131072 --chunks $N 2>/dev/null | sed "s/^/$(basename $d) /" | cut -c1-200); done
done | tee -a gpurun_out/ab_persist.txt
[ -d tmp_life ] && bash tools/gpu_life.sh
SPPO_TRACE=gpurun_out/trace_pb_n16.txt SPPO_TRACE_CHUNK=15 SPPO_TRACE_KIND=bwd timeout 300 python tools/trace_run.py > /dev/null 2>&1
python tools/trace_boundary.py gpurun_out/trace_pb_n16.txt 64 | head -4
