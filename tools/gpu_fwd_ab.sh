#!/bin/bash
# Split-row forward: a guarded smoke first (a hang must not eat the call), parity
# tests, interleaved A/B bench (SPPO_FWD_KERNEL=1 old, 2 new) and a trace.
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
rc=$?; echo "smoke rc=$rc"; tail -3 gpurun_out/smoke.log
[ $rc -ne 0 ] && exit 1
timeout 900 python -m pytest tests -q -x -m "gpu and not slow" -p no:cacheprovider > gpurun_out/pytest_fwd2.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_fwd2.log
for k in 2 1 2 1; do
  SPPO_FWD_KERNEL=$k timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-offload --no-cpu --no-c3 > gpurun_out/ab_fwd$k.json 2> gpurun_out/ab_fwd$k.err
  echo "kernel $k: $(tail -1 gpurun_out/ab_fwd$k.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['fwd_tflops'], d['bwd_tflops'], d['clocks']['sm_mhz'])")"
done
SPPO_TRACE=gpurun_out/trace_fwd2.txt SPPO_TRACE_CHUNK=15 SPPO_TRACE_KIND=fwd timeout 120 python tools/trace_run.py > /dev/null 2>&1
python tools/trace_stats.py gpurun_out/trace_fwd2.txt fwd
