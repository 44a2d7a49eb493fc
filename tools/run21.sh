timeout 300 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_policies.py -q -x 2>&1 | tail -2
for e in 1; do timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-offload --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ('value','ms_per_step','fwd_tflops','bwd_tflops','clocks')})"; done
