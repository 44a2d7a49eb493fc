set -x
timeout 300 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_fp32.py -q 2>&1 | tail -3
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err
tail -3 gpurun_out/bench2.err
cat gpurun_out/bench2.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bwd_kernel -s 0 -c 1 -o gpurun_out/prof_bwd2 python bench.py --steps 1 --warmup 0 --no-e2e --no-offload --no-cpu > gpurun_out/ncu_bwd2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 15 -c 1 -o gpurun_out/prof_fwd2 python bench.py --steps 1 --warmup 0 --no-e2e --no-offload --no-cpu > gpurun_out/ncu_fwd2.log 2>&1
