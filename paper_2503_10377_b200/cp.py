"""Context parallelism: chunked causal attention with the
sequence sharded over G ranks, K/V rotated around a ring, on top of the same
kernels and the same C ABI as the single-GPU path.

Layout.  The N global chunks (offsets as in sppo_layout) form 2G blocks of
B = N / (2G) consecutive chunks; rank g owns blocks g and 2G-1-g (zigzag), so
every rank holds the same number of causal (query, key) pairs.  Each rank keeps
Q, K, V, dO, O, LSE of its own chunks only.

Forward.  G ring steps.  At step r rank g holds the K/V of rank (g - r) mod G;
for each own chunk i it calls sppo_attn_fwd on the window of held chunks j <= i
(FIRST on i's first non-empty window, LAST on its last: the online-softmax
carry of a2 merges the windows, P:356 + reading L14).  The K/V it holds go to
rank g+1 while it computes (NCCL point-to-point; host-staged over gloo).

Backward.  Same ring with the fp32 dK/dV accumulators of the held chunks
travelling with their K/V; each own chunk i accumulates dQ_i over its windows
(FIRST: Delta and zeroed dQ accumulator, LAST: dQ_i written).  After G steps one
more hop returns every accumulator to its owner, where sppo_finalize (a7) casts
it to dK_j, dV_j.

Every compute step is a libsppo call; this module sequences calls and moves
bytes (torch.distributed).  The schedule is a pure function (`ring_schedule`),
tested on the CPU for exact 0..i coverage.
"""

from __future__ import annotations

import torch

from . import sppo


# ------------------------------------------------------------------ plan (pure)
def owned_chunks(N: int, G: int, g: int):
    """Chunks of rank g: blocks g and 2G-1-g of B = N/(2G) chunks each (ascending)."""
    if N % (2 * G):
        raise ValueError(f"N = {N} chunks must be a multiple of 2G = {2 * G}")
    B = N // (2 * G)
    lo = list(range(g * B, (g + 1) * B))
    hi = list(range((2 * G - 1 - g) * B, (2 * G - g) * B))
    return lo + hi if g != 2 * G - 1 - g else lo


def ring_schedule(N: int, G: int, g: int):
    """steps[r] = (holder, [(i, window_ids, flags), ...]) for ring steps r = 0..G-1 of
    rank g: at step r rank g holds the K/V of `holder` = (g - r) mod G; own chunk i
    attends to window_ids = held chunks j <= i.  Over all steps every own i sees each
    j in 0..i exactly once, FIRST on its first window, LAST on its last."""
    own = owned_chunks(N, G, g)
    steps = []
    for r in range(G):
        h = (g - r) % G
        held = owned_chunks(N, G, h)
        steps.append((h, [(i, [j for j in held if j <= i]) for i in own]))
    first = {}
    last = {}
    for r, (_, wins) in enumerate(steps):
        for i, w in wins:
            if w:
                first.setdefault(i, r)
                last[i] = r
    out = []
    for r, (h, wins) in enumerate(steps):
        items = []
        for i, w in wins:
            if w:
                flags = (sppo.SPPO_FIRST if first[i] == r else 0) | (sppo.SPPO_LAST if last[i] == r else 0)
                items.append((i, w, flags))
        out.append((h, items))
    return out


# ------------------------------------------------------------------ transport
class Ring:
    """Point-to-point exchange with the ring neighbours: send to g+1, receive from
    g-1.  NCCL: device tensors, stream-ordered.  Otherwise (gloo): host-staged."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        if not dist.is_initialized():  # a ring of one (single process)
            self.G, self.g, self.nccl = 1, 0, False
            return
        self.G = dist.get_world_size(group)
        self.g = dist.get_rank(group)
        self.nccl = dist.get_backend(group) == "nccl"

    def exchange(self, send: list, recv: list):
        """Start sending `send` to g+1 and receiving into `recv` from g-1; returns a
        handle whose wait() completes the exchange (on the current stream for NCCL)."""
        dist = self.dist
        if self.G == 1:  # the neighbour is this rank
            for a, b in zip(send, recv):
                b.copy_(a)
            return _Handle([], None)
        nxt = (self.g + 1) % self.G
        prv = (self.g - 1) % self.G
        if self.nccl:
            ops = [dist.P2POp(dist.isend, t, nxt, self.group) for t in send]
            ops += [dist.P2POp(dist.irecv, t, prv, self.group) for t in recv]
            reqs = dist.batch_isend_irecv(ops)
            return _Handle(reqs, None)
        if torch.cuda.is_available():
            torch.cuda.current_stream().synchronize()
        host_send = [t.detach().cpu() for t in send]
        host_recv = [torch.empty(t.shape, dtype=t.dtype) for t in recv]
        reqs = [dist.isend(t, nxt, self.group) for t in host_send]
        reqs += [dist.irecv(t, prv, self.group) for t in host_recv]
        return _Handle(reqs, (host_recv, recv))


class _Handle:
    def __init__(self, reqs, staged):
        self.reqs, self.staged = reqs, staged

    def wait(self):
        for q in self.reqs:
            q.wait()
        if self.staged is not None:
            for h, d in zip(*self.staged):
                d.copy_(h, non_blocking=False)


# ------------------------------------------------------------------ ring attention
class RingAttention:
    """Chunked causal attention of one sequence sharded over the ranks of `group`.

    `layout` describes the GLOBAL chunking (offsets over the whole sequence) and the
    heads each rank computes (all of them).  Inputs and outputs are this rank's own
    tokens, concatenated in ascending chunk order: [own_tokens, heads, d]."""

    def __init__(self, ctx: sppo.Context, layout: sppo.Layout, group=None, device="cuda"):
        self.ctx, self.L = ctx, layout
        self.ring = Ring(group)
        G, g = self.ring.G, self.ring.g
        self.G, self.g = G, g
        N = layout.num_chunks
        self.own = owned_chunks(N, G, g)
        self.sched = ring_schedule(N, G, g)
        self.dev = torch.device(device)
        h, d = layout.heads, layout.head_dim
        self.dt = torch.bfloat16 if layout.dtype == sppo.SPPO_BF16 else torch.float32
        # own-token offsets of each own chunk inside the packed local buffers
        self.loc = {}
        o = 0
        for i in self.own:
            self.loc[i] = (o, o + layout.chunk_len(i))
            o += layout.chunk_len(i)
        self.T = o
        f32 = dict(dtype=torch.float32, device=self.dev)
        self.o = torch.empty((o, h, d), dtype=self.dt, device=self.dev)
        self.lse = torch.empty((o * h,), **f32)   # chunk after chunk, each [h, s_i]
        self.dq = torch.empty((o, h, d), dtype=self.dt, device=self.dev)
        self.dk = torch.empty((o, h, d), dtype=self.dt, device=self.dev)
        self.dv = torch.empty((o, h, d), dtype=self.dt, device=self.dev)
        self._state = {i: (torch.empty((self._len(i), h, d), **f32), torch.empty((h * self._len(i),), **f32),
                           torch.empty((h * self._len(i),), **f32)) for i in self.own}
        self._delta = {i: torch.empty((h * self._len(i),), **f32) for i in self.own}
        self._dq_acc = {i: torch.empty((self._len(i), h, d), **f32) for i in self.own}

    def _len(self, i):
        return self.L.chunk_len(i)

    def _rows(self, t, i):
        a, b = self.loc[i]
        return t[a:b]

    def _lse(self, i):
        a, b = self.loc[i]
        h = self.L.heads
        return self.lse[a * h:b * h]

    def _tokens_of(self, rank):
        return sum(self._len(j) for j in owned_chunks(self.L.num_chunks, self.G, rank))

    def _split(self, buf, rank):
        """views of a packed [tokens of `rank`, h, d] buffer per chunk of `rank`"""
        out, o = {}, 0
        for j in owned_chunks(self.L.num_chunks, self.G, rank):
            out[j] = buf[o:o + self._len(j)]
            o += self._len(j)
        return out

    # -------------------------------------------------------------- forward
    def forward(self, q, k, v, stream=None):
        """q, k, v: this rank's own tokens [T, h, d].  Fills self.o, self.lse."""
        h, d = self.L.heads, self.L.head_dim
        strm = stream or torch.cuda.current_stream()
        cur_k, cur_v = k, v
        for r, (holder, items) in enumerate(self.sched):
            handle = None
            if r + 1 < self.G:
                src = (self.g - r - 1) % self.G
                nk = torch.empty((self._tokens_of(src), h, d), dtype=self.dt, device=self.dev)
                nv = torch.empty_like(nk)
                handle = self.ring.exchange([cur_k, cur_v], [nk, nv])  # overlaps the windows below
            ks, vs = self._split(cur_k, holder), self._split(cur_v, holder)
            for i, w, flags in items:
                st = None if flags == sppo.SPPO_FIRST | sppo.SPPO_LAST else self._state[i]
                self.ctx.attn_fwd(self.L, i, self._rows(q, i), w, [ks[j] for j in w], [vs[j] for j in w],
                                  flags=flags, state=st, o=self._rows(self.o, i), lse=self._lse(i), stream=strm)
            if handle is not None:
                handle.wait()
                cur_k, cur_v = nk, nv
        return self.o

    # -------------------------------------------------------------- backward
    def backward(self, q, k, v, do, stream=None):
        """After forward: dQ, dK, dV of this rank's own tokens (self.dq / dk / dv)."""
        h, d = self.L.heads, self.L.head_dim
        strm = stream or torch.cuda.current_stream()
        f32 = dict(dtype=torch.float32, device=self.dev)
        cur_k, cur_v = k, v
        cur_dk = torch.zeros((self.T, h, d), **f32)
        cur_dv = torch.zeros((self.T, h, d), **f32)
        for r, (holder, items) in enumerate(self.sched):
            kv_handle = None
            src = (self.g - r - 1) % self.G
            if r + 1 < self.G:  # K/V are read-only: start their hop before computing
                nk = torch.empty((self._tokens_of(src), h, d), dtype=self.dt, device=self.dev)
                nv = torch.empty_like(nk)
                kv_handle = self.ring.exchange([cur_k, cur_v], [nk, nv])
            ks, vs = self._split(cur_k, holder), self._split(cur_v, holder)
            dks, dvs = self._split(cur_dk, holder), self._split(cur_dv, holder)
            for i, w, flags in sorted(items, key=lambda x: -x[0]):
                last = bool(flags & sppo.SPPO_LAST)
                self.ctx.attn_bwd(self.L, i, self._rows(q, i), w, [ks[j] for j in w], [vs[j] for j in w],
                                  self._rows(self.o, i), self._lse(i), self._rows(do, i), self._delta[i],
                                  self._dq_acc[i], [dks[j] for j in w], [dvs[j] for j in w],
                                  dq=self._rows(self.dq, i) if last else None, flags=flags, stream=strm)
            # the accumulators move on after this step's windows (every step, plus one
            # final hop that brings each back to its owner)
            ndk = torch.empty((self._tokens_of(src), h, d), **f32)
            ndv = torch.empty_like(ndk)
            acc_handle = self.ring.exchange([cur_dk, cur_dv], [ndk, ndv])
            if kv_handle is not None:
                kv_handle.wait()
                cur_k, cur_v = nk, nv
            acc_handle.wait()
            cur_dk, cur_dv = ndk, ndv
        # after G hops the accumulators are home: a7
        self.ctx.finalize(cur_dk, self.dk, self.L.dtype, stream=strm)
        self.ctx.finalize(cur_dv, self.dv, self.L.dtype, stream=strm)
        return self.dq, self.dk, self.dv
