timeout 900 python bench.py --steps 5 --warmup 3 --kv-hot 8 > gpurun_out/bench_r01_c2.json 2> gpurun_out/bench_r01_c2.err
tail -2 gpurun_out/bench_r01_c2.err
timeout 1500 python bench.py --config C3 --steps 2 --warmup 1 --no-e2e --no-offload --no-cpu > gpurun_out/bench_r01_c3.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-offload --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bwd_kernel -s 0 -c 1 -o gpurun_out/prof_bwd_r01 python bench.py --steps 1 --warmup 0 --no-e2e --no-offload --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 15 -c 1 -o gpurun_out/prof_fwd_r01 python bench.py --steps 1 --warmup 0 --no-e2e --no-offload --no-cpu > /dev/null 2>&1
ls gpurun_out
