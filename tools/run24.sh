timeout 300 python -m pytest tests/test_gpu_policies.py -q -x 2>&1 | tail -2
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --partition balanced > gpurun_out/bench_balanced.json 2>gpurun_out/bench_balanced.err
tail -2 gpurun_out/bench_balanced.err
python -c "import json; d=json.load(open('gpurun_out/bench_balanced.json')); o=d['offload']; print(d['value'], d['ms_per_step'], o['exposed_pct'], o['fixed_alpha1'], o['alpha'][:6], o['fwd_ms_per_chunk'][:6], o['d2h_ms_per_chunk_alpha1'][:6])"
