set -x
timeout 300 python -m pytest tests/test_gpu_bf16.py -q 2>&1 | tail -3
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err
tail -3 gpurun_out/bench1.err
cat gpurun_out/bench1.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-offload --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bwd_kernel -s 0 -c 1 -o gpurun_out/prof_bwd python bench.py --steps 1 --warmup 0 --no-e2e --no-offload --no-cpu > gpurun_out/ncu_bwd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 15 -c 1 -o gpurun_out/prof_fwd python bench.py --steps 1 --warmup 0 --no-e2e --no-offload --no-cpu > gpurun_out/ncu_fwd.log 2>&1
ls -la gpurun_out
