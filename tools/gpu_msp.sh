#!/bin/bash
# MSP on the GPU: real-layer executor test, then the layer bench line with the MSP model.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_msp.py -q -x -p no:cacheprovider > gpurun_out/pytest_msp.log 2>&1
echo "msp pytest rc=$?"; tail -3 gpurun_out/pytest_msp.log
timeout 900 python bench.py --workload layer --partition layer-balanced --steps 3 --warmup 2 --no-e2e --no-cpu --no-offload > gpurun_out/bench_layer_msp.json 2> gpurun_out/bench_layer_msp.err
echo "layer bench rc=$?"
tail -1 gpurun_out/bench_layer_msp.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']); print(json.dumps(d.get('pipeline_model'), indent=1))"
