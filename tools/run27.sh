python tools/mma_bench.py | grep random
timeout 900 python -m pytest tests/test_gpu_edge.py -q -x 2>&1 | tail -4
