timeout 600 python -m pytest tests/test_gpu_policies.py tests/test_gpu_bf16.py tests/test_gpu_fp32.py -q -x 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_large.py -q -x 2>&1 | tail -5
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --kv-hot 8 --kv-window 4 2>&1 | tail -1 > gpurun_out/bench3.json
python -c "import json; d=json.load(open('gpurun_out/bench3.json')); print({k:d[k] for k in ('value','ms_per_step','fwd_tflops','bwd_tflops','offload','kv_stream','e2e')})"
