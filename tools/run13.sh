timeout 300 python -m pytest tests/test_gpu_bf16.py -q -x 2>&1 | tail -2
timeout 1200 python bench.py --config C3 --steps 1 --warmup 1 --no-e2e --no-offload --no-cpu 2>&1 | tail -1 > gpurun_out/bench_c3.json
python -c "import json; d=json.load(open('gpurun_out/bench_c3.json')); print({k:d[k] for k in ('value','ms_per_step','fwd_tflops','bwd_tflops','pct_bf16_peak','clocks')})"
