"""MSP execution host logic (paper_2503_10377_b200/msp.py; SURVEY §8(f)4,
P:420-461 [§6.2]) on the CPU:

  * the plan: every stage's GPU range per chunk is the paper's worked example
    (Table P:386-404 via sppo_msp_phases, reading L18); every forward / backward
    task appears once and after its predecessors; the schedule model never puts
    two tasks on one rank at once; without MSP it reproduces the subsequence
    pipeline's makespan (sppo_pipeline_makespan, itself pinned to the closed
    form (p-1+N)/N F(N)); with MSP it lies between the work bound and
    the plain pipeline, and closes the bubble for PP=2 (P:322's s_0 example);
  * the executor's communication (inter-stage rows, the four phase-boundary
    moves of K/V and dK/dV, the gradient assembly) with gloo, world sizes 2-4,
    on a stub layer that has the same interface and a causal dependence on the
    K/V of earlier chunks: MSP gives the plain pipeline's outputs and gradients.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle.plan as oracle_plan
from paper_2503_10377_b200 import msp, sppo


def test_plan_groups_match_paper_table():
    plan = msp.MSPPlan(4, 8, sppo.partition_equal(8192, 8))
    # Table: Left SP ranges {0..3},{1..3},{2,3},- ; Right -,{0,1},{0,1,2},{0..3}
    left = {0: (0, 1, 2, 3), 1: (1, 2, 3), 2: (2, 3)}
    right = {1: (0, 1), 2: (0, 1, 2), 3: (0, 1, 2, 3)}
    want_left_ids = {0: [0, 1, 2], 1: [0, 1], 2: [0], 3: []}
    want_right_ids = {0: [], 1: [7], 2: [6, 7], 3: [5, 6, 7]}
    for s in range(4):
        for i in range(8):
            g = plan.group(s, i)
            if i in want_left_ids[s]:
                assert g == left[s]
            elif i in want_right_ids[s]:
                assert g == right[s]
            else:
                assert g == (s,)


@pytest.mark.parametrize("PP,N", [(2, 4), (3, 6), (4, 8), (4, 16), (8, 16), (5, 7)])
def test_plan_tasks_order_and_resources(PP, N):
    plan = msp.MSPPlan(PP, N, sppo.partition_equal(N * 512, N))
    pos = {t: n for n, t in enumerate(plan.tasks)}
    for kind in ("F", "B"):
        assert sorted((s, i) for k, s, i in plan.tasks if k == kind) == [(s, i) for s in range(PP) for i in range(N)]
    for t, preds in plan._deps().items():
        for u in preds:
            assert pos[u] < pos[t], (u, t)
    # the model never runs two tasks on one rank at once
    for r in range(PP):
        iv = sorted((plan.start[t], plan.end[t]) for t in plan.tasks if r in plan.busy(t) and plan.cost(t) > 0)
        for (a0, a1), (b0, b1) in zip(iv, iv[1:]):
            assert b0 >= a1 - 1e-9


@pytest.mark.parametrize("PP,N", [(2, 4), (3, 6), (4, 8), (4, 16), (8, 16)])
def test_plain_makespan_equals_pipeline_and_msp_shrinks_bubble(PP, N):
    g = torch.Generator().manual_seed(PP * 100 + N)
    tf = (torch.rand(N, generator=g) + 0.5).tolist()
    tb = [2 * x for x in tf]
    off = sppo.partition_equal(N * 512, N)
    plain = msp.msp_makespan(PP, N, off, tf, tb, msp=False)
    assert abs(plain - sppo.pipeline_makespan(PP, tf, tb)) < 1e-9
    assert abs(plain - oracle_plan.pipeline_makespan(PP, N, tf, tb)[0]) < 1e-9
    uni = msp.msp_makespan(PP, N, off, [1.0] * N, [2.0] * N, msp=True)
    bound = 3.0 * N  # total work / PP
    assert bound - 1e-9 <= uni < msp.msp_makespan(PP, N, off, [1.0] * N, [2.0] * N, msp=False)
    if PP == 2:
        assert abs(uni - bound) < 1e-9  # s_0's split removes the whole bubble


# ------------------------------------------------------------------ executor on a stub layer
class StubLayer:
    """Same interface as engine_layer.ChunkedLayer, exact fp64 arithmetic:
    k = x_c * w, v = x_c + b on this rank's columns c; o_p = sum_{t <= p} k_t v_t
    (causal over ALL earlier chunks: needs their K/V); z = x + allreduce(o);
    backward by hand, dK/dV accumulated over later chunks like attention's."""

    def __init__(self, params, S, H, offsets, tp):
        self.j, self.g, self.group = tp if tp is not None else (0, 1, None)
        self.H, self.Hl = H, H // self.g
        self.c = slice(self.j * self.Hl, (self.j + 1) * self.Hl)
        self.off = offsets
        self.p = params
        f = dict(dtype=torch.float64)
        self.z, self.dx = torch.zeros(S, H, **f), torch.zeros(S, H, **f)
        self.k, self.v = torch.zeros(S, self.Hl, **f), torch.zeros(S, self.Hl, **f)
        self.dk_acc, self.dv_acc = torch.zeros(S, self.Hl, **f), torch.zeros(S, self.Hl, **f)
        self.grads = {n: torch.zeros(self.Hl, **f) for n in ("w", "b")}

    def _ar(self, t):
        if self.g > 1:
            dist.all_reduce(t, group=self.group)

    def _zero(self):
        for t in (self.dk_acc, self.dv_acc, *self.grads.values()):
            t.zero_()

    def forward_chunk(self, i, x, strm=None):
        a, b = self.off[i], self.off[i + 1]
        xl = x[a:b, self.c]
        self.k[a:b] = xl * self.p["w"]
        self.v[a:b] = xl + self.p["b"]
        o = torch.cumsum(self.k[:b] * self.v[:b], 0)[a:b]
        part = torch.zeros(b - a, self.H, dtype=torch.float64)
        part[:, self.c] = o
        self._ar(part)
        self.z[a:b] = x[a:b] + part

    def backward_chunk(self, i, x, dz, strm=None):
        a, b = self.off[i], self.off[i + 1]
        do = dz[a:b, self.c]
        rc = torch.flip(torch.cumsum(torch.flip(do, [0]), 0), [0])  # sum_{p >= t, p in chunk}
        gk = torch.cat([do.sum(0, keepdim=True).expand(a, -1), rc])  # rows 0..b-1
        self.dk_acc[:b] += gk * self.v[:b]
        self.dv_acc[:b] += gk * self.k[:b]
        xl = x[a:b, self.c]
        dk, dv = self.dk_acc[a:b], self.dv_acc[a:b]
        self.grads["w"] += (dk * xl).sum(0)
        self.grads["b"] += dv.sum(0)
        part = torch.zeros(b - a, self.H, dtype=torch.float64)
        part[:, self.c] = dk * self.p["w"] + dv
        self._ar(part)
        self.dx[a:b] = dz[a:b] + part


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, S, H, N, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = torch.Generator().manual_seed(5)
    prm = [{"w": torch.randn(H, generator=g, dtype=torch.float64) * 0.1,
            "b": torch.randn(H, generator=g, dtype=torch.float64) * 0.1} for _ in range(world)]
    x = torch.randn(S, H, generator=g, dtype=torch.float64)
    dz = torch.randn(S, H, generator=g, dtype=torch.float64)
    off = sppo.partition_equal(S, N)
    res = {}
    for use in (False, True):
        ex = msp.MSPExecutor(None, rank, world, H, 1, off, prm, device="cpu", msp=use,
                             make_layer=lambda p, tp: StubLayer(p, S, H, off, tp),
                             shard=lambda p, j, gg: {k: v[j * H // gg:(j + 1) * H // gg] for k, v in p.items()},
                             unshard=lambda sh: {k: torch.cat([d[k] for d in sh]) for k in sh[0]})
        res[use] = ex.step(x, dz)
        res[(use, "log")] = list(ex.log)
    torch.save(res, os.path.join(out, f"r{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,N", [(2, 4), (3, 6), (4, 8)])
def test_executor_msp_equals_plain_pipeline(tmp_path, world, N):
    S, H = N * 16, 12
    mp.spawn(_worker, args=(world, _free_port(), S, H, N, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        res = torch.load(os.path.join(tmp_path, f"r{r}.pt"))
        a, b = res[False], res[True]
        for k in ("x", "z", "dz", "dx"):
            torch.testing.assert_close(b[k], a[k], rtol=1e-12, atol=1e-12, msg=f"stage {r} {k}")
        for k in a["grads"]:
            torch.testing.assert_close(b["grads"][k], a["grads"][k], rtol=1e-12, atol=1e-12, msg=f"stage {r} d{k}")
        # MSP really multiplexed: this rank computed chunks of other stages
        assert any(t[0] == "F" and t[1] != r for t in res[(True, "log")]) or world == 1
