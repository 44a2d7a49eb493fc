"""MSP execution of real GPT layers on the B200 kernels (
P:420-461 [§6.2]; paper_2503_10377_b200/msp.py): PP pipeline stages, one layer
each, as PP ranks sharing the one GPU (gloo, host-staged transfers and
tensor-parallel all-reduces).  Bubble-adjacent chunks run tensor-parallel over
the stage's Left-SP / Right-SP ranges (reading L18, L20).  Each stage owner's
assembled z, dx and full parameter gradients are compared with the fp64 layer
oracle on exactly the bf16 rows that stage received (tolerances as
tests/test_gpu_layer.py, reading L17), and with the plain pipeline run through
the same executor."""

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
    from paper_2503_10377_b200 import msp, sppo
    torch.cuda.set_device(0)
    ctx = sppo.Context(0)
    off = sppo.partition_equal(S, N)
    prm = [synth.make_layer_params(H, seed=200 + s) for s in range(world)]
    io = synth.make_layer_io(S, H, seed=9)
    res = {}
    for use in (True, False):
        ex = msp.MSPExecutor(ctx, rank, world, H, heads, off, prm, msp=use)
        r = ex.step(io["x"].cuda(), io["dz"].cuda())
        torch.cuda.synchronize()
        res[use] = {k: (v.float().cpu().numpy() if torch.is_tensor(v) else {n: g.cpu().numpy() for n, g in v.items()})
                    for k, v in r.items()}
        res[(use, "tasks")] = sum(1 for t in ex.log if t[0] in "FB" and t[1] != rank and rank in ex.plan.group(t[1], t[2]))
        del ex
    ctx.sync()
    np.save(os.path.join(out, f"r{rank}.npy"), res, allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()
    ctx.close()


def _check(name, got, ref, frob):
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    rms = np.sqrt(np.mean(ref ** 2))
    assert rel <= frob, (name, rel)
    assert (np.abs(got - ref) <= 5e-2 * np.abs(ref) + 5e-2 * rms).all(), name


@pytest.mark.parametrize("world,heads,S,N", [(2, 2, 1024, 4), (3, 6, 1536, 6)])
def test_msp_pipeline_matches_layer_oracle(tmp_path, world, heads, S, N):
    H = heads * 128
    mp.spawn(_worker, args=(world, _free_port(), S, H, heads, N, str(tmp_path)), nprocs=world, join=True)
    ps = [{k: v.double().numpy() for k, v in synth.make_layer_params(H, seed=200 + s).items()} for s in range(world)]
    res = [np.load(os.path.join(tmp_path, f"r{r}.npy"), allow_pickle=True).item() for r in range(world)]
    for r in range(world):
        assert res[r][(True, "tasks")] > 0, "MSP ran no chunk of another stage on this rank"
        assert res[r][(False, "tasks")] == 0
        for use in (True, False):
            o = res[r][use]
            # per stage: the oracle layer on exactly the bf16 rows the stage received
            z, cache = L.layer_fwd(o["x"].astype(np.float64), ps[r], heads)
            dx, gr = L.layer_bwd(o["dz"].astype(np.float64), cache, ps[r])
            _check(f"msp={use} stage{r}.z", o["z"], z, 1e-2)
            _check(f"msp={use} stage{r}.dx", o["dx"], dx, 1e-2)
            for k in L.PARAM_NAMES:
                _check(f"msp={use} stage{r}.{k}", o["grads"][k], gr[k], 2e-2)
        # the stage received the same rows either way (up to bf16 rounding of TP partial sums)
        a, b = res[r][True], res[r][False]
        for k in ("x", "dz"):
            assert np.linalg.norm(a[k] - b[k]) <= 2e-2 * np.linalg.norm(b[k]), (r, k)
