#!/bin/bash
# Per-CTA lifetime trace of the largest bwd launch (tmp_life = -DSPPO_BWD_LIFE=1 build):
# C2 (chunk 15 of 16), 2K chunks (63 of 64), 32K chunks (3 of 4).
mkdir -p gpurun_out
cd tmp_life
for cfg in "16 15" "64 63" "4 3"; do
  set -- $cfg
  SPPO_TRACE=../gpurun_out/life_n$1.txt SPPO_TRACE_LIFE=1 SPPO_TRACE_CHUNK=$2 SPPO_TRACE_KIND=bwd TN=$1 \
    timeout 300 python tools/trace_run.py > /dev/null 2>&1
  echo "N=$1"; python ../tools/life_persist.py ../gpurun_out/life_n$1.txt
done
