"""Multi-rank host logic of the head-sharded path, world_size 2 on CPU (gloo):
each rank generates only its heads (synth seeds per GLOBAL head), computes its
shard (here with the oracle — the CUDA kernels need a GPU), and the all-gather
reassembles exactly the unsharded result; the timing reduction is a max."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2503_10377_b200.dist import gather_heads, head_range, max_over_ranks
from synth import make_inputs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    S, h, d = 96, 4, 8
    heads = head_range(h, world, rank)
    x = make_inputs(S, heads, d, seed=5, dtype=torch.float32)
    xn = {k: v.double().numpy() for k, v in x.items()}
    off = [0, 40, 96]
    o, lse = oracle.chunked_attention_fwd(xn["q"], xn["k"], xn["v"], off)
    full = gather_heads(torch.from_numpy(o), world)
    t = max_over_ranks(1.0 + rank, world)
    if rank == 0:
        np.save(os.path.join(out_dir, "gathered.npy"), full.numpy())
        np.save(os.path.join(out_dir, "tmax.npy"), np.array([t]))
    dist.barrier()
    dist.destroy_process_group()


def test_head_range():
    assert head_range(32, 8, 3) == [12, 13, 14, 15]
    assert head_range(40, 1, 0) == list(range(40))
    with pytest.raises(ValueError):
        head_range(40, 3, 0)
    assert sum(len(head_range(64, 8, r)) for r in range(8)) == 64


def test_two_rank_shard_and_gather(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    got = np.load(tmp_path / "gathered.npy")
    assert float(np.load(tmp_path / "tmax.npy")[0]) == 2.0
    x = make_inputs(96, range(4), 8, seed=5, dtype=torch.float32)
    xn = {k: v.double().numpy() for k, v in x.items()}
    ref, _ = oracle.causal_attention_dense(xn["q"], xn["k"], xn["v"])
    np.testing.assert_allclose(got, ref, atol=1e-12)
