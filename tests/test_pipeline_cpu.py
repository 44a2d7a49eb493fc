"""Subsequence pipeline on the CPU: the paper's bubble formula and
MSP table pin the oracle (oracle/plan.py) and the C plan helpers
(sppo_msp_phases, sppo_pipeline_bubble); the stage executor's host logic
(paper_2503_10377_b200/pipeline.py: chunk order, P2P routing, receive
pre-posting) runs over gloo with world size 2 and 3 on test-only stub layers
whose chunk i depends on every earlier chunk (like attention)."""

import json
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from oracle import plan
from paper_2503_10377_b200 import sppo

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")))


def test_bubble_ratio_paper_example_and_simulation():
    g = GOLD["bubble_ratio"]  # p = 4, N = 16 -> 3/16
    assert plan.bubble_ratio(g["p"], g["N"]) == g["ratio"]
    assert sppo.pipeline_bubble(g["p"], g["N"]) == g["ratio"]
    for p, N, tf, tb in [(4, 16, 1.0, 2.0), (2, 8, 1.0, 1.0), (8, 64, 0.5, 1.25), (1, 5, 1.0, 3.0)]:
        T, log = plan.pipeline_makespan(p, N, tf, tb)
        F = N * (tf + tb)
        assert abs(T - (p - 1 + N) / N * F) < 1e-9          # T = (p-1+N)/N F(N)
        assert abs((T - F) / F - plan.bubble_ratio(p, N)) < 1e-9
        for s in range(p):  # every stage: forwards ascending, then backwards descending
            assert [(k, i) for k, i, _, _ in log[s]] == [("fwd", i) for i in range(N)] + \
                   [("bwd", i) for i in range(N - 1, -1, -1)]


def test_makespan_helper_matches_simulation_nonuniform():
    import random
    rnd = random.Random(3)
    for p, N in [(1, 1), (2, 8), (4, 16), (8, 5)]:
        tf = [rnd.uniform(0.5, 3.0) for _ in range(N)]
        tb = [2.5 * t for t in tf]
        T, _ = plan.pipeline_makespan(p, N, tf, tb)
        assert abs(sppo.pipeline_makespan(p, tf, tb) - T) < 1e-9 * T
    # uniform: (p-1+N)/N F(N)
    assert abs(sppo.pipeline_makespan(4, [1.0] * 16, [2.0] * 16) - 19 * 3.0) < 1e-12


def test_msp_phases_match_paper_table():
    g = GOLD["msp_table_pp4_n8"]
    for s, row in enumerate(g["stages"]):
        assert plan.msp_phases(g["PP"], g["N"], s) == row
        assert sppo.msp_phases(g["PP"], g["N"], s) == row


@pytest.mark.parametrize("PP,N", [(1, 1), (2, 2), (3, 7), (8, 64), (5, 5)])
def test_msp_phases_partition_and_ranges(PP, N):
    for s in range(PP):
        ref = plan.msp_phases(PP, N, s)
        assert sppo.msp_phases(PP, N, s) == ref
        assert sorted(ref["left"] + ref["steady"] + ref["right"]) == list(range(N))  # a partition of 0..N-1
        assert len(ref["steady"]) == N - PP + 1                                       # every stage: N-PP+1 steady
        assert len(ref["left"]) + len(ref["right"]) == PP - 1                         # bubble-adjacent ones
    with pytest.raises(sppo.SppoError):
        sppo.msp_phases(4, 3, 0)


# ------------------------------------------------------------------ executor over gloo
class StubLayer:
    """Test-only stand-in for engine_layer.ChunkedLayer: z_p = w x_p + sum_{t<=p} x_t
    (a causal prefix, so chunk i reads the rows of chunks 0..i like attention);
    backward dx_t = w dz_t + sum_{p>=t} dz_p, accumulated chunk by chunk in reverse."""

    def __init__(self, S, H, offsets, w):
        self.off, self.N, self.w = offsets, len(offsets) - 1, w
        self.z = torch.zeros(S, H, dtype=torch.float64)
        self.dx = torch.zeros(S, H, dtype=torch.float64)
        self.acc = torch.zeros(S, H, dtype=torch.float64)

    def rows(self, t, i):
        return t[self.off[i]:self.off[i + 1]]

    def _zero(self):
        self.acc.zero_()

    def forward_chunk(self, i, x, stream=None):
        a, b = self.off[i], self.off[i + 1]
        self.z[a:b] = self.w * x[a:b] + torch.cumsum(x[:b], 0)[a:b]

    def backward_chunk(self, i, x, dz, stream=None):
        a, b = self.off[i], self.off[i + 1]
        v = torch.zeros(b, dz.shape[1], dtype=torch.float64)
        v[a:b] = dz[a:b]
        self.acc[:b] += torch.flip(torch.cumsum(torch.flip(v, [0]), 0), [0])
        self.dx[a:b] = self.w * dz[a:b] + self.acc[a:b]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, S, H, offsets, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_10377_b200 import pipeline
    g = torch.Generator().manual_seed(0)
    x = torch.randn(S, H, generator=g, dtype=torch.float64)
    dz = torch.randn(S, H, generator=g, dtype=torch.float64)
    layers = [StubLayer(S, H, offsets, 1.5 + rank), StubLayer(S, H, offsets, -0.5 - rank)]  # 2 layers per stage
    st = pipeline.SubsequencePipeline(rank, world, layers, pipeline.StageComm(rank, world),
                                      x_buf=torch.zeros(S, H, dtype=torch.float64),
                                      dz_buf=torch.zeros(S, H, dtype=torch.float64))
    z, dx = st.step(x=x if rank == 0 else None, dz=dz if rank == world - 1 else None)
    torch.save({"z": z.clone(), "dx": dx.clone(), "order": st.order}, os.path.join(out, f"r{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,offsets", [(2, [0, 3, 7, 12, 16]), (3, [0, 5, 6, 16])])
def test_pipeline_stages_over_gloo_equal_sequential(tmp_path, world, offsets):
    S, H = offsets[-1], 4
    mp.spawn(_worker, args=(world, _free_port(), S, H, offsets, str(tmp_path)), nprocs=world, join=True)
    g = torch.Generator().manual_seed(0)
    x = torch.randn(S, H, generator=g, dtype=torch.float64)
    dz = torch.randn(S, H, generator=g, dtype=torch.float64)
    ws = [w for r in range(world) for w in (1.5 + r, -0.5 - r)]
    h = x
    for w in ws:  # sequential reference: the whole stack on one process, dense
        h = w * h + torch.cumsum(h, 0)
    gr = dz
    for w in reversed(ws):
        gr = w * gr + torch.flip(torch.cumsum(torch.flip(gr, [0]), 0), [0])
    res = [torch.load(os.path.join(tmp_path, f"r{r}.pt")) for r in range(world)]
    torch.testing.assert_close(res[-1]["z"], h, rtol=1e-12, atol=1e-12)
    torch.testing.assert_close(res[0]["dx"], gr, rtol=1e-12, atol=1e-12)
    N = len(offsets) - 1
    for r in res:
        assert r["order"] == [("fwd", i) for i in range(N)] + [("bwd", i) for i in range(N - 1, -1, -1)]
