"""Subsequence pipeline of real GPT layers on the B200 kernels:
2 pipeline stages (one layer each) as 2 ranks sharing the one GPU (gloo,
host-staged chunk transfers; NCCL refuses two ranks on one device).  The last
stage's output z and the first stage's dx, and each stage's weight gradients,
are compared with the fp64 oracle of the 2-layer stack (oracle/layer.py) —
tolerances as tests/test_gpu_layer.py (reading L17)."""

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
    from paper_2503_10377_b200 import engine_layer, pipeline, sppo
    torch.cuda.set_device(0)
    ctx = sppo.Context(0)
    off = sppo.partition_equal(S, N)
    params = {k: v.cuda() for k, v in synth.make_layer_params(H, seed=100 + rank).items()}
    lay = engine_layer.ChunkedLayer(ctx, H, heads, off, params)
    io = synth.make_layer_io(S, H, seed=7)
    bf = dict(dtype=torch.bfloat16, device="cuda")
    st = pipeline.SubsequencePipeline(rank, world, [lay], pipeline.StageComm(rank, world),
                                      x_buf=torch.zeros(S, H, **bf), dz_buf=torch.zeros(S, H, **bf))
    z, dx = st.step(x=io["x"].cuda() if rank == 0 else None, dz=io["dz"].cuda() if rank == world - 1 else None)
    torch.cuda.synchronize()
    ctx.sync()
    np.savez(os.path.join(out, f"r{rank}.npz"), z=z.float().cpu().numpy(), dx=dx.float().cpu().numpy(),
             **{k: v.cpu().numpy() for k, v in lay.grads.items()})
    dist.barrier()
    dist.destroy_process_group()
    ctx.close()


def _check(name, got, ref, frob):
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    rms = np.sqrt(np.mean(ref ** 2))
    assert rel <= frob, (name, rel)
    assert (np.abs(got - ref) <= 5e-2 * np.abs(ref) + 5e-2 * rms).all(), name


def test_two_stage_pipeline_matches_two_layer_oracle(tmp_path):
    S, H, heads, N, world = 1024, 256, 2, 4, 2
    mp.spawn(_worker, args=(world, _free_port(), S, H, heads, N, str(tmp_path)), nprocs=world, join=True)
    io = synth.make_layer_io(S, H, seed=7)
    ps = [{k: v.double().numpy() for k, v in synth.make_layer_params(H, seed=100 + r).items()} for r in range(world)]
    res = [np.load(os.path.join(tmp_path, f"r{r}.npz")) for r in range(world)]
    # per stage: the oracle layer on exactly the bf16 rows that stage received
    # (stage r > 0: stage r-1's z; stage r < last: stage r+1's dx)
    ins = [io["x"].double().numpy()] + [res[r]["z"].astype(np.float64) for r in range(world - 1)]
    gins = [res[r + 1]["dx"].astype(np.float64) for r in range(world - 1)] + [io["dz"].double().numpy()]
    for r in range(world):
        z, cache = L.layer_fwd(ins[r], ps[r], heads)
        dx, gr = L.layer_bwd(gins[r], cache, ps[r])
        _check(f"stage{r}.z", res[r]["z"], z, 1e-2)
        _check(f"stage{r}.dx", res[r]["dx"], dx, 1e-2)
        for k in L.PARAM_NAMES:
            _check(f"stage{r}.{k}", res[r][k], gr[k], 2e-2)
    # end to end: the 2-layer stack in fp64 from the model input (errors of both stages compound)
    h = ins[0]
    caches = []
    for r in range(world):
        h, c = L.layer_fwd(h, ps[r], heads)
        caches.append(c)
    g = gins[-1]
    for r in range(world - 1, -1, -1):
        g, _ = L.layer_bwd(g, caches[r], ps[r])
    for name, got, ref in (("z", res[-1]["z"], h), ("dx", res[0]["dx"], g)):
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 2e-2, name
