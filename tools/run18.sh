timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 15 -c 1 -o gpurun_out/prof_fwd3 python bench.py --steps 1 --warmup 0 --no-e2e --no-offload --no-cpu > gpurun_out/ncu_fwd3.log 2>&1
tail -2 gpurun_out/ncu_fwd3.log
