timeout 600 compute-sanitizer --tool synccheck --print-limit 5 python tools/sanitize_step.py 2>&1 | tail -2
timeout 300 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_policies.py -q -x 2>&1 | tail -1
