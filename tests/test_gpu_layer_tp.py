"""Tensor-parallel layer (heads partitioned over ranks, Megatron column / row
parallel projections, all-reduce of the partial sums; engine_layer tp=...): 2
ranks sharing the one GPU (gloo, host-staged all-reduce).  Each rank's z, dx and
its shard of every parameter gradient against the fp64 oracle of the whole layer
(tolerances as test_gpu_layer.py, reading L17)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle.layer as L
import synth

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, S, H, heads, N, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_10377_b200 import engine_layer, sppo
    torch.cuda.set_device(0)
    ctx = sppo.Context(0)
    full = synth.make_layer_params(H, seed=21)
    shard = {k: v.cuda() for k, v in engine_layer.shard_params(full, H, heads, rank, world).items()}
    io = synth.make_layer_io(S, H, seed=21)
    lay = engine_layer.ChunkedLayer(ctx, H, heads, sppo.partition_equal(S, N), shard, tp=(rank, world, None))
    o = lay.step(io["x"].cuda(), io["dz"].cuda())
    torch.cuda.synchronize()
    np.savez(os.path.join(out, f"r{rank}.npz"), z=o["z"].float().cpu().numpy(), dx=o["dx"].float().cpu().numpy(),
             **{k: v.cpu().numpy() for k, v in o["grads"].items()})
    dist.barrier()
    dist.destroy_process_group()
    ctx.close()


def _check(name, got, ref, frob):
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    rms = np.sqrt(np.mean(ref ** 2))
    assert rel <= frob, (name, rel)
    assert (np.abs(got - ref) <= 5e-2 * np.abs(ref) + 5e-2 * rms).all(), name


def test_tensor_parallel_layer_two_ranks(tmp_path):
    from paper_2503_10377_b200 import engine_layer
    S, H, heads, N, world = 1024, 256, 2, 4, 2
    mp.spawn(_worker, args=(world, _free_port(), S, H, heads, N, str(tmp_path)), nprocs=world, join=True)
    full = synth.make_layer_params(H, seed=21)
    io = synth.make_layer_io(S, H, seed=21)
    p64 = {k: v.double().numpy() for k, v in full.items()}
    z, cache = L.layer_fwd(io["x"].double().numpy(), p64, heads)
    dx, gr = L.layer_bwd(io["dz"].double().numpy(), cache, p64)
    grt = {k: torch.tensor(v) for k, v in gr.items()}
    for r in range(world):
        res = np.load(os.path.join(tmp_path, f"r{r}.npz"))
        _check(f"r{r}.z", res["z"], z, 1e-2)
        _check(f"r{r}.dx", res["dx"], dx, 1e-2)
        ref_shard = engine_layer.shard_params(grt, H, heads, r, world)  # the same slicing applied to the grads
        for k in L.PARAM_NAMES:
            _check(f"r{r}.{k}", res[k], ref_shard[k].numpy(), 2e-2)
