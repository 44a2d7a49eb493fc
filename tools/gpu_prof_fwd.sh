#!/bin/bash
# ncu --set full with source-level stall sampling of the chunk-15 forward launch, both kernels.
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1 || { echo smoke failed; tail gpurun_out/smoke.log; exit 1; }
for k in 1 2; do
  SPPO_FWD_KERNEL=$k SPPO_TRACE_KIND=fwd timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd \
    --launch-skip 15 -c 1 -f -o gpurun_out/prof_fwdk$k python tools/trace_run.py > gpurun_out/prof_fwdk$k.log 2>&1
  ncu -i gpurun_out/prof_fwdk$k.ncu-rep --page source --csv > gpurun_out/prof_fwdk${k}_source.csv 2>/dev/null
  ncu -i gpurun_out/prof_fwdk$k.ncu-rep --page details --csv > gpurun_out/prof_fwdk${k}_details.csv 2>/dev/null
  ncu -i gpurun_out/prof_fwdk$k.ncu-rep --page raw --csv > gpurun_out/prof_fwdk${k}_raw.csv 2>/dev/null
done
ls -la gpurun_out/prof_fwdk*
timeout 600 python -m pytest tests/test_gpu_msp.py -q -x -p no:cacheprovider > gpurun_out/pytest_msp.log 2>&1
echo "msp pytest rc=$?"; tail -3 gpurun_out/pytest_msp.log
