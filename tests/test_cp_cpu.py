"""Context-parallel ring, host side on CPU: the zigzag chunk
ownership and ring schedule (every own chunk i sees each j in 0..i exactly once,
FIRST/LAST on its first/last window, equal causal work per rank) and the ring
transport over gloo (world size 3)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2503_10377_b200 import sppo
from paper_2503_10377_b200.cp import Ring, owned_chunks, ring_schedule


@pytest.mark.parametrize("N,G", [(2, 1), (4, 2), (8, 2), (8, 4), (16, 8), (24, 3), (64, 8)])
def test_schedule_covers_prefix_exactly_once(N, G):
    own_all = []
    for g in range(G):
        own = owned_chunks(N, G, g)
        own_all += own
        seen = {i: [] for i in own}
        flags = {i: [] for i in own}
        sched = ring_schedule(N, G, g)
        assert len(sched) == G
        for r, (holder, items) in enumerate(sched):
            assert holder == (g - r) % G
            held = set(owned_chunks(N, G, holder))
            for i, w, f in items:
                assert w and set(w) <= held and max(w) <= i
                seen[i] += w
                flags[i].append(f)
        for i in own:
            assert sorted(seen[i]) == list(range(i + 1)), (g, i)
            f = flags[i]
            assert f[0] & sppo.SPPO_FIRST and f[-1] & sppo.SPPO_LAST
            assert all(not (x & sppo.SPPO_FIRST) for x in f[1:]) and all(not (x & sppo.SPPO_LAST) for x in f[:-1])
    assert sorted(own_all) == list(range(N))


@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_zigzag_balances_causal_work(G):
    S, N = 8 * 4096, 4 * G
    off = oracle.offsets_from_lengths(oracle.partition_equal(S, N))
    work = []
    for g in range(G):
        work.append(sum(oracle.causal_pairs(off[i + 1] - off[i], off[i]) for i in owned_chunks(N, G, g)))
    assert max(work) - min(work) <= max(work) * 1e-3
    with pytest.raises(ValueError):
        owned_chunks(6, 4, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ring_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ring = Ring()
    cur = torch.full((5, 3), float(rank))
    got = []
    for _ in range(world):  # a full rotation
        nxt = torch.empty_like(cur)
        ring.exchange([cur], [nxt]).wait()
        cur = nxt
        got.append(int(cur[0, 0]))
    q.put((rank, got))
    dist.barrier()
    dist.destroy_process_group()


def test_ring_exchange_gloo_three_ranks():
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.start_processes(_ring_worker, args=(world, _free_port(), q), nprocs=world, join=True, start_method="spawn")
    res = dict(q.get() for _ in range(world))
    for r in range(world):
        assert res[r] == [(r - k - 1) % world for k in range(world)]  # after G hops: own tensor is back
