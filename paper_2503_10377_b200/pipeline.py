"""Subsequence pipeline across stages (P:222 [§3], P:278-287
[§3.3], P:369 [§5.2]).

The layers of the model are split over PP pipeline stages, one process (GPU)
per stage.  The sequence is cut into N subsequences (chunks); stage s runs the
forward of chunk i for its layers as soon as chunk i's activations arrive from
stage s-1, and sends its output rows to stage s+1 — so stage s works on chunk i
while stage s+1 works on chunk i-1 (sequence pipelining).  The backward runs
the chunks in reverse (N-1..0, reading L11): stage s receives dz_i from stage
s+1, runs its layers' backward for chunk i and sends dx_i to stage s-1.  With
uniform per-chunk times the makespan is (PP-1+N)/N F(N) and the bubble ratio
(PP-1)/N (sppo_pipeline_bubble, oracle/plan.py pipeline_makespan).

Inter-stage transfers are point-to-point on the rows of one chunk: NCCL
isend/irecv of device tensors (stream-ordered, NVLink P2P on one node), or
host-staged over gloo (tests: several stages sharing one GPU).  The receive of
chunk i+1 is posted before chunk i's compute so the transfer overlaps it.
Every arithmetic step runs in the layers' ABI calls (engine_layer.ChunkedLayer);
this module only sequences them and moves bytes.

MSP (Left-SP / Steady / Right-SP) is executed by msp.py: the same
stages, with bubble-adjacent chunks tensor-parallel over the stage's SP range.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


class StageComm:
    """Point-to-point transfers between neighbouring pipeline stages."""

    def __init__(self, stage: int, n_stages: int, group=None, ranks=None):
        self.stage, self.n = stage, n_stages
        self.group = group
        self.ranks = list(ranks) if ranks is not None else list(range(n_stages))
        self.nccl = dist.is_initialized() and dist.get_backend(group) == "nccl"

    def _peer(self, stage):
        return self.ranks[stage]

    def send(self, t, to_stage):
        if self.nccl or t.device.type == "cpu":
            return [dist.isend(t, self._peer(to_stage), self.group)]
        h = t.detach().cpu()  # host-staged (gloo): the copy synchronises with the producer
        return [dist.isend(h, self._peer(to_stage), self.group), h]

    def recv(self, t, from_stage):
        """Posts a receive into `t`; returns a handle whose wait() completes it."""
        if self.nccl or t.device.type == "cpu":
            return _Recv(dist.irecv(t, self._peer(from_stage), self.group), None, None)
        h = torch.empty(t.shape, dtype=t.dtype)
        return _Recv(dist.irecv(h, self._peer(from_stage), self.group), h, t)


class _Recv:
    def __init__(self, work, host, dev):
        self.work, self.host, self.dev = work, host, dev

    def wait(self):
        self.work.wait()
        if self.host is not None:
            self.dev.copy_(self.host, non_blocking=False)


class SubsequencePipeline:
    """One pipeline stage: `layers` (engine_layer.ChunkedLayer or any object with
    forward_chunk / backward_chunk / z / dx / rows / N / _zero) applied in order."""

    def __init__(self, stage: int, n_stages: int, layers: list, comm: StageComm, x_buf=None, dz_buf=None):
        self.stage, self.n_stages = stage, n_stages
        self.layers = layers
        self.comm = comm
        self.N = layers[0].N
        self.x_buf = x_buf    # stage > 0: rows of chunk i arrive here from stage - 1
        self.dz_buf = dz_buf  # stage < last: rows of chunk i arrive here from stage + 1
        self.order = []       # (kind, chunk) in execution order (tests / schedule checks)

    @property
    def first(self):
        return self.stage == 0

    @property
    def last(self):
        return self.stage == self.n_stages - 1

    def _inputs(self, x):
        ins = [x]
        for lay in self.layers[:-1]:
            ins.append(lay.z)
        return ins

    def step(self, x=None, dz=None, stream=None):
        """Forward of chunks 0..N-1 then backward of N-1..0 on this stage.
        x: the model input (stage 0 only); dz: the upstream gradient of the last
        stage's output (last stage only).  Returns (z of the last layer, dx of
        the first layer) — meaningful on the last / first stage respectively."""
        for lay in self.layers:
            lay._zero()
        xin = x if self.first else self.x_buf
        ins = self._inputs(xin)
        sends = []
        # ---------------- forward, chunks ascending
        pending = None if self.first else self.comm.recv(self.layers[0].rows(self.x_buf, 0), self.stage - 1)
        for i in range(self.N):
            if pending is not None:
                pending.wait()
                pending = (self.comm.recv(self.layers[0].rows(self.x_buf, i + 1), self.stage - 1)
                           if i + 1 < self.N else None)
            for lay, inp in zip(self.layers, ins):
                lay.forward_chunk(i, inp, stream)
            self.order.append(("fwd", i))
            if not self.last:
                sends += self.comm.send(self.layers[-1].rows(self.layers[-1].z, i), self.stage + 1)
        # ---------------- backward, chunks descending
        gin = dz if self.last else self.dz_buf
        pending = None if self.last else self.comm.recv(self.layers[-1].rows(self.dz_buf, self.N - 1),
                                                         self.stage + 1)
        for i in range(self.N - 1, -1, -1):
            if pending is not None:
                pending.wait()
                pending = (self.comm.recv(self.layers[-1].rows(self.dz_buf, i - 1), self.stage + 1)
                           if i > 0 else None)
            g = gin
            for k in range(len(self.layers) - 1, -1, -1):
                self.layers[k].backward_chunk(i, ins[k], g, stream)
                g = self.layers[k].dx
            self.order.append(("bwd", i))
            if not self.first:
                sends += self.comm.send(self.layers[0].rows(self.layers[0].dx, i), self.stage - 1)
        for w in sends:
            if hasattr(w, "wait"):
                w.wait()
        return self.layers[-1].z, self.layers[0].dx
