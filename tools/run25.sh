SPPO_BENCH_DEVICE=0 SPPO_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err
echo rc=$?
tail -3 gpurun_out/bench_2rank.err
python -c "import json; d=json.load(open('gpurun_out/bench_2rank.json')); print({k:d[k] for k in ('value','n_gpus','ms_per_step','scaling','gather')}, d['config']['heads_per_gpu'])"
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 2>&1 | tail -1
