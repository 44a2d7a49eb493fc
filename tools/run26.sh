timeout 1500 python bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-offload --no-cpu --kv-hot 16 --kv-window 4 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
tail -2 gpurun_out/bench_c4.err
python -c "import json; d=json.load(open('gpurun_out/bench_c4.json')); print({k:d[k] for k in ('value','ms_per_step','fwd_tflops','bwd_tflops','pct_bf16_peak')}, d['kv_stream'])"
timeout 2400 python bench.py --config C5 --shard-of 8 --steps 1 --warmup 1 --no-e2e --no-offload --no-cpu --kv-hot 0 --kv-window 8 > gpurun_out/bench_c5shard.json 2> gpurun_out/bench_c5shard.err
tail -2 gpurun_out/bench_c5shard.err
python -c "import json; d=json.load(open('gpurun_out/bench_c5shard.json')); print({k:d[k] for k in ('value','ms_per_step','fwd_tflops','bwd_tflops','pct_bf16_peak')}, d['kv_stream'])"
