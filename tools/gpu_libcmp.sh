#!/bin/bash
# Library context: cuDNN SDPA (sm_100 fused attention) causal fwd/bwd on this box next
# to the SPPO engine on the same shapes (interleaved), + cuDNN's launch list and one
# ncu --set full capture of its kernels (config, tensor pipe, smem, L2 traffic).
#   gpurun --timeout 1500 -- 'bash tools/gpu_libcmp.sh [ncu]'
mkdir -p gpurun_out
for rep in 1 2; do
for s in 131072 16384; do
  timeout 600 python tools/lib_attn_bench.py --seq $s 2>> gpurun_out/lib_cmp.err | tee -a gpurun_out/lib_cmp.jsonl
  timeout 600 python tools/lib_attn_bench.py --impl sppo --seq $s --chunks 1 2>> gpurun_out/lib_cmp.err | tee -a gpurun_out/lib_cmp.jsonl
done
timeout 600 python tools/lib_attn_bench.py --impl sppo --seq 131072 --chunks 16 2>> gpurun_out/lib_cmp.err | tee -a gpurun_out/lib_cmp.jsonl
done
[ "$1" = ncu ] || exit 0
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__cluster_dim_x,launch__shared_mem_per_block_dynamic,launch__registers_per_thread --clock-control none --csv --log-file gpurun_out/lib_cudnn_launches.csv \
  python tools/lib_attn_bench.py --seq 32768 --reps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -c 14 -f -o gpurun_out/lib_cudnn_full python tools/lib_attn_bench.py --seq 16384 --reps 0 > /dev/null 2>&1
ncu -i gpurun_out/lib_cudnn_full.ncu-rep --page raw --csv > gpurun_out/lib_cudnn_full_raw.csv 2>/dev/null
ncu -i gpurun_out/lib_cudnn_full.ncu-rep --page details --csv > gpurun_out/lib_cudnn_full_details.csv 2>/dev/null
rm -f gpurun_out/lib_cudnn_full.ncu-rep
