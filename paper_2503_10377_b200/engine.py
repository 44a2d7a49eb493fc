"""Chunk-loop orchestration of one SPPO attention step over the C ABI.

One step = forward over chunks i = 0..N-1 (ascending) then backward over
i = N-1..0 (reading L11), each chunk's prior-KV set 0..i visited in windows of
at most ``window`` chunks (FIRST/LAST carry).  Every compute
step is a call into libsppo (sppo_attn_fwd / sppo_attn_bwd); this module only
allocates buffers (torch, device memory) and sequences the calls.

Buffer layout in HBM: full-sequence token-major tensors
[S, h, d] whose chunk i is the contiguous row range [c_i, c_{i+1}); LSE stored
chunk after chunk, each chunk head-major [h, s_i]; fp32 dK/dV accumulators for
the whole sequence; per-chunk fp32 scratch (dQ accumulator, Delta, fwd carry)
sized for the longest chunk and reused.
"""

from __future__ import annotations

import torch

from . import sppo

DTYPES = {sppo.SPPO_BF16: torch.bfloat16, sppo.SPPO_FP32: torch.float32}


class ChunkedAttention:
    def __init__(self, ctx: sppo.Context, layout: sppo.Layout, device="cuda", window: int | None = None):
        self.ctx, self.L = ctx, layout
        self.device = torch.device(device)
        self.window = window if window else 10**9
        h, d = layout.heads, layout.head_dim
        S = layout.offsets[-1]
        smax = max(layout.chunk_len(i) for i in range(layout.num_chunks))
        dt = DTYPES[layout.dtype]
        f32 = dict(dtype=torch.float32, device=self.device)
        self.S = S
        self.o = torch.empty((S, h, d), dtype=dt, device=self.device)
        self.lse = torch.empty((S * h,), **f32)
        self.dq = torch.empty((S, h, d), dtype=dt, device=self.device)
        self.dk = torch.empty((S, h, d), dtype=dt, device=self.device)
        self.dv = torch.empty((S, h, d), dtype=dt, device=self.device)
        self.dk_acc = torch.empty((S, h, d), **f32)
        self.dv_acc = torch.empty((S, h, d), **f32)
        self.dq_acc = torch.empty((smax, h, d), **f32)
        self.delta = torch.empty((smax * h,), **f32)
        self.o_acc = torch.empty((smax, h, d), **f32)
        self.m = torch.empty((smax * h,), **f32)
        self.l = torch.empty((smax * h,), **f32)

    # chunk views -----------------------------------------------------------
    def rows(self, t, i):
        c = self.L.offsets
        return t[c[i]:c[i + 1]]

    def lse_view(self, i, base=None):
        c, h = self.L.offsets, self.L.heads
        base = self.lse if base is None else base
        return base[c[i] * h:c[i + 1] * h]

    def windows(self, i):
        ids = list(range(i + 1))
        w = self.window
        return [ids[a:a + w] for a in range(0, len(ids), w)]

    # one step ----------------------------------------------------------------
    def forward_chunk(self, i, q, k, v, stream=None):
        L = self.L
        s = L.chunk_len(i)
        h = L.heads
        wins = self.windows(i)
        state = (self.o_acc[:s], self.m[:s * h], self.l[:s * h])
        for n, ids in enumerate(wins):
            flags = (sppo.SPPO_FIRST if n == 0 else 0) | (sppo.SPPO_LAST if n == len(wins) - 1 else 0)
            self.ctx.attn_fwd(L, i, self.rows(q, i), ids, [self.rows(k, j) for j in ids],
                              [self.rows(v, j) for j in ids], flags=flags,
                              state=None if len(wins) == 1 else state,
                              o=self.rows(self.o, i), lse=self.lse_view(i), stream=stream)

    def backward_chunk(self, i, q, k, v, do, stream=None):
        L = self.L
        s = L.chunk_len(i)
        h = L.heads
        wins = self.windows(i)
        for n, ids in enumerate(wins):
            flags = (sppo.SPPO_FIRST if n == 0 else 0) | (sppo.SPPO_LAST if n == len(wins) - 1 else 0)
            has_i = i in ids
            self.ctx.attn_bwd(L, i, self.rows(q, i), ids, [self.rows(k, j) for j in ids],
                              [self.rows(v, j) for j in ids], self.rows(self.o, i), self.lse_view(i),
                              self.rows(do, i), self.delta[:s * h], self.dq_acc[:s],
                              [self.rows(self.dk_acc, j) for j in ids], [self.rows(self.dv_acc, j) for j in ids],
                              dq=self.rows(self.dq, i), dk=self.rows(self.dk, i) if has_i else None,
                              dv=self.rows(self.dv, i) if has_i else None, flags=flags, stream=stream)

    def step(self, q, k, v, do, stream=None):
        """Full forward + backward over all chunks (resident policy)."""
        N = self.L.num_chunks
        self.dk_acc.zero_()
        self.dv_acc.zero_()
        for i in range(N):
            self.forward_chunk(i, q, k, v, stream)
        for i in range(N - 1, -1, -1):
            self.backward_chunk(i, q, k, v, do, stream)
        return dict(o=self.o, lse=self.lse, dq=self.dq, dk=self.dk, dv=self.dv)

    def lse_heads_major(self):
        """[h, S] view assembled from per-chunk [h, s_i] blocks (for checks)."""
        parts = [self.lse_view(i).view(self.L.heads, -1) for i in range(self.L.num_chunks)]
        return torch.cat(parts, dim=1)
