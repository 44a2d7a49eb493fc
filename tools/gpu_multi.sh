#!/bin/bash
# Multi-chunk forward: guarded smoke, parity subset, A/B (SPPO_FWD_MULTI=1 / 0) at C2 and the C5 share, sanitizers.
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1 || { echo smoke failed; tail gpurun_out/smoke.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_edge.py tests/test_gpu_policies.py tests/test_gpu_streams.py tests/test_gpu_large.py -q -x -p no:cacheprovider > gpurun_out/pytest_multi.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_multi.log
for m in 1 0 1 0; do
  SPPO_FWD_MULTI=$m timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-offload --no-cpu --no-c3 > gpurun_out/ab_multi$m.json 2>/dev/null
  echo "multi $m C2: $(tail -1 gpurun_out/ab_multi$m.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['fwd_tflops'], d['bwd_tflops'], d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
done
for m in 1 0; do
  SPPO_FWD_MULTI=$m timeout 300 python bench.py --shard-of 8 --steps 5 --warmup 3 --no-e2e --no-offload --no-cpu --no-c3 > gpurun_out/ab_multi_s8_$m.json 2>/dev/null
  echo "multi $m C2 share 1/8: $(tail -1 gpurun_out/ab_multi_s8_$m.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['fwd_tflops'], d['bwd_tflops'], d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
done
bash tools/gpu_san.sh
