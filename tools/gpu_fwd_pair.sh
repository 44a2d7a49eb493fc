#!/bin/bash
# Pair forward (SPPO_FWD_KERNEL=pair) vs default: guarded smoke + parity subset with pair, A/B, trace.
mkdir -p gpurun_out
SPPO_FWD_KERNEL=pair timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1 || { echo smoke failed; tail gpurun_out/smoke.log; exit 1; }
SPPO_FWD_KERNEL=pair timeout 600 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_edge.py tests/test_gpu_policies.py tests/test_gpu_streams.py -q -x -m "gpu and not slow" -p no:cacheprovider > gpurun_out/pytest_pair.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_pair.log
for k in pair 128 pair 128; do
  SPPO_FWD_KERNEL=$k timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-offload --no-cpu --no-c3 > gpurun_out/ab_$k.json 2> gpurun_out/ab_$k.err
  echo "kernel $k: $(tail -1 gpurun_out/ab_$k.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['fwd_tflops'], d['bwd_tflops'], d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
done
SPPO_FWD_KERNEL=pair SPPO_TRACE=gpurun_out/trace_fwd2.txt SPPO_TRACE_CHUNK=15 SPPO_TRACE_KIND=fwd timeout 120 python tools/trace_run.py > /dev/null 2>&1
echo traced
