"""Chunk-loop orchestration of one GPT transformer layer over the C ABI
(include/sppo.h + include/sppo_layer.h).

One step = the layer forward over chunks i = 0..N-1, then its backward over
i = N-1..0 (reading L11).  Per chunk i (token rows [c_i, c_{i+1})):

  forward   a = LN1(x)                       sppo_layernorm_fwd
            [q k v] = a W_qkv^T + b_qkv      sppo_gemm (C split into Q | K | V)
            o = attention(q; K, V of 0..i)   sppo_attn_fwd
            y = x + o W_o^T + b_o            sppo_gemm (bias + residual epilogue)
            b = LN2(y)                       sppo_layernorm_fwd
            g = GELU(u), u = b W_1^T + b_1   sppo_gemm (GELU epilogue, u saved)
            z = y + g W_2^T + b_2            sppo_gemm (bias + residual epilogue)
  backward  du = (dz W_2) * GELU'(u)          sppo_gemm (dGELU epilogue)
            dW_2 += dz^T g, db_2 += sum dz   sppo_gemm (fp32 acc), sppo_col_reduce
            dbn = du W_1; dW_1 += du^T b ...
            dy = dz + LN2_bwd(dbn)           sppo_layernorm_bwd (+ col_reduce for dgamma/dbeta)
            do = dy W_o; dW_o += dy^T o ...
            dq_i, dK_j/dV_j (j <= i)         sppo_attn_bwd (dK_i, dV_i final now, L11)
            da = [dq dk dv] W_qkv; dW_qkv += [dq dk dv]^T a ...
            dx = dy + LN1_bwd(da)

Two-level activation management (P:356 [§5.1]): K_i, V_i stay on the GPU
(Type-0, whole-sequence buffers); the Type-1 tensors of chunk i — a, q, o, y, b,
u, g (13 h bf16 per token) plus LSE and the LayerNorm statistics — live in a
per-chunk set.  Under step_offload they leave after fwd(i) as the
alpha_i-prefix of each tensor on the ctx D2H stream (overlapping fwd(i+1),
P:369) and come back on the H2D stream before bwd(i), at most ``depth`` chunks
ahead; alpha_i = min(1, BW_D2H * T_fwd(i+1) / A_i), alpha_{N-1} = 0
(reading L9).

Memory (``pool``): False = one whole-sequence buffer per Type-1 tensor (chunk
sets are row views; offload then only measures overlap).  True = chunk sets are
separate allocations: once the D2H of chunk i's prefix has completed, the
device copy is released (the suffix, 1 - alpha_i, is kept as a compact copy),
and the backward re-allocates the set, prefetches the prefix and restores the
suffix — so device memory holds K/V, the resident suffixes and a few in-flight
sets instead of every chunk's activations.  Buffers are torch allocations; every
arithmetic step runs in libsppo's kernels.
"""

from __future__ import annotations

import torch

from . import sppo

PARAM_NAMES = ("ln1_g", "ln1_b", "w_qkv", "b_qkv", "w_o", "b_o", "ln2_g", "ln2_b", "w_1", "b_1", "w_2", "b_2")
TYPE1 = ("a", "q", "o", "y", "b", "u", "g")  # token-major bf16 activations offloaded with alpha
STATS = ("lse", "mu1", "rstd1", "mu2", "rstd2")  # fp32 statistics, offloaded whole
LN_EPS = 1e-5


def shard_params(params: dict, hidden: int, heads: int, rank: int, size: int) -> dict:
    """Rank `rank`'s tensor-parallel shard of a layer's parameters (Megatron
    layout): W_qkv / b_qkv rows of this rank's heads (q, k and v parts), W_1 /
    b_1 rows (column-parallel), W_o / W_2 columns (row-parallel); LayerNorm
    parameters, b_o and b_2 replicated.  Contiguous copies (GEMM operands)."""
    H, Hl = hidden, hidden // size
    r = slice(rank * Hl, (rank + 1) * Hl)
    f = slice(rank * 4 * Hl, (rank + 1) * 4 * Hl)
    out = dict(params)
    out["w_qkv"] = torch.cat([params["w_qkv"][k * H:(k + 1) * H][r] for k in range(3)]).contiguous()
    out["b_qkv"] = torch.cat([params["b_qkv"][k * H:(k + 1) * H][r] for k in range(3)]).contiguous()
    out["w_o"] = params["w_o"][:, r].contiguous()
    out["w_1"] = params["w_1"][f].contiguous()
    out["b_1"] = params["b_1"][f].contiguous()
    out["w_2"] = params["w_2"][:, f].contiguous()
    return out


class ChunkedLayer:
    def __init__(self, ctx: sppo.Context, hidden: int, heads: int, offsets, params: dict, device="cuda",
                 timing: bool = False, pool: bool = False, streams: int = 1, tp=None):
        """tp = (rank, size, process group or None): Megatron-style tensor
        parallelism over the heads (P:157 [§2]; the north star's "heads are
        partitioned across the GPUs"): `params` are this rank's shard
        (shard_params), the QKV / fc1 projections are column-parallel, out-proj /
        fc2 row-parallel, and their partial sums (plus the backward's partial
        LayerNorm inputs) are all-reduced — the layer's real exchange steps."""
        self.ctx = ctx
        self.tp_rank, self.tp_size, self.tp_group = tp if tp is not None else (0, 1, None)
        if heads % self.tp_size:
            raise ValueError("heads must divide over the tensor-parallel ranks")
        self.H, self.heads = hidden, heads // self.tp_size  # self.heads: heads on this rank
        self.d = hidden // heads
        self.Hl = self.heads * self.d  # width of this rank's q / k / v / o
        self.L = sppo.Layout(self.heads, self.d, offsets, dtype=sppo.SPPO_BF16)
        self.N = self.L.num_chunks
        if self.N > 256:
            raise ValueError("ChunkedLayer issues one attention window per chunk: N <= 256")
        self.S = S = self.L.offsets[-1]
        self.device = torch.device(device)
        self.p = params
        self.timing = timing
        self.pool = pool
        H, Hl = hidden, self.Hl
        bf = dict(dtype=torch.bfloat16, device=self.device)
        f32 = dict(dtype=torch.float32, device=self.device)
        # Type-0 (resident) and outputs: whole sequence, token-major
        self.k = torch.empty((S, Hl), **bf)
        self.v = torch.empty((S, Hl), **bf)
        self.z = torch.empty((S, H), **bf)
        self.dx = torch.empty((S, H), **bf)
        self.dk_acc = torch.empty((S, Hl), **f32)
        self.dv_acc = torch.empty((S, Hl), **f32)
        # per-chunk backward scratch (longest chunk)
        smax = max(self.L.chunk_len(i) for i in range(self.N))
        self.du = torch.empty((smax, 4 * Hl), **bf)
        for n in ("dbn", "da"):
            setattr(self, n, torch.empty((smax, H), **bf))
        for n in ("dq", "dkc", "dvc"):
            setattr(self, n, torch.empty((smax, Hl), **bf))
        # d_o and dy pass from backward_b(i) to backward_a(i): two sets, so that
        # backward_b(i-1) on a second stream can run while backward_a(i) reads them
        self.dy2 = [torch.empty((smax, H), **bf) for _ in range(2)]
        self.d_o2 = [torch.empty((smax, Hl), **bf) for _ in range(2)]
        self.dq_acc = torch.empty((smax, Hl), **f32)
        self.delta = torch.empty((smax * self.heads,), **f32)
        # Type-1: whole-sequence buffers (resident) or per-chunk allocations (pool)
        self._full = None
        if not pool:
            self._full = {n: torch.empty((S,) + self._t1_shape(n, 1)[0][1:], dtype=self._t1_shape(n, 1)[1],
                                         device=self.device) for n in TYPE1}
            self._full.update({n: torch.empty((S * (self.heads if n == "lse" else 1),), **f32) for n in STATS})
        self.T = [None] * self.N
        self.grads = {n: torch.zeros(tuple(params[n].shape), **f32) for n in PARAM_NAMES}
        self.launches = 0
        self.events = {"fwd": [], "bwd": []}
        self.gemm_events = None  # list: (start, end, FLOPs) of every GEMM call (bench instrumentation)
        self.attn_events = None  # list: (start, end) of every attention call
        self._host = {}
        self.streams = streams
        self._side = None

    # ------------------------------------------------------------------ helpers
    def rows(self, t, i):
        c = self.L.offsets
        return t[c[i]:c[i + 1]]

    def _t1_shape(self, name, s):
        if name in ("u", "g"):
            return (s, 4 * self.Hl), torch.bfloat16
        if name in ("q", "o"):
            return (s, self.Hl), torch.bfloat16
        if name in TYPE1:  # a, y, b: LayerNorm inputs / outputs, full width on every rank
            return (s, self.H), torch.bfloat16
        return ((s * self.heads,) if name == "lse" else (s,)), torch.float32

    def _t1_set(self, i):
        """Chunk i's Type-1 set: row views of the whole-sequence buffers, or fresh allocations."""
        s = self.L.chunk_len(i)
        if not self.pool:
            c = self.L.offsets
            return {n: (t[c[i] * self.heads:c[i + 1] * self.heads] if n == "lse" else self.rows(t, i))
                    for n, t in self._full.items()}
        out = {}
        for n in TYPE1 + STATS:
            shape, dt = self._t1_shape(n, s)
            out[n] = torch.empty(shape, dtype=dt, device=self.device)
        return out

    def _gemm(self, M, N, K, *args, **kw):
        ev = self.gemm_events
        if ev is not None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(kw["stream"])
        self.ctx.gemm(M, N, K, *args, **kw)
        if ev is not None:
            e1.record(kw["stream"])
            ev.append((e0, e1, 2 * M * N * K))
        self.launches += 1

    def _allreduce(self, t, strm):
        """Sum over the tensor-parallel ranks, in place (no-op without TP).  NCCL:
        stream-ordered on `strm` (the current stream inside step); otherwise
        (gloo, tests) host-staged."""
        if self.tp_size == 1 or self.tp_group is False:  # False: a timing-only shard (bench MSP model)
            return
        import torch.distributed as dist
        st = strm if isinstance(strm, torch.cuda.Stream) else torch.cuda.current_stream()
        with torch.cuda.stream(st):
            if dist.get_backend(self.tp_group) == "nccl":
                dist.all_reduce(t, group=self.tp_group)
            else:
                h = t.float().cpu()
                dist.all_reduce(h, group=self.tp_group)
                t.copy_(h)

    def _attn_ev(self, strm):
        if self.attn_events is None:
            return None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(strm)
        self.attn_events.append((e0, e1))
        return e1

    def _ev(self, kind, stream):
        if not self.timing:
            return None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        self.events[kind].append((e0, e1))
        return e1

    def chunk_ms(self, kind):
        """Per-chunk durations (ms) of the recorded fwd / bwd calls, in call order."""
        return [a.elapsed_time(b) for a, b in self.events[kind]]

    def _kv(self, i):
        ids = list(range(i + 1))
        return ids, [self.rows(self.k, j) for j in ids], [self.rows(self.v, j) for j in ids]

    # ------------------------------------------------------------------ forward of chunk i
    def forward_chunk(self, i, x, strm):
        end = self._ev("fwd", strm)
        self.forward_a(i, x, strm)
        self.forward_b(i, x, strm)
        if end is not None:
            end.record(strm)

    def forward_a(self, i, x, strm):
        """LN1, QKV projection, attention of chunk i (needs K/V of chunks <= i)."""
        p, H, s = self.p, self.H, self.L.chunk_len(i)
        T = self.T[i] = self._t1_set(i)
        xi = self.rows(x, i)
        self.ctx.layernorm_fwd(xi, p["ln1_g"], p["ln1_b"], T["a"], T["mu1"], T["rstd1"], eps=LN_EPS, stream=strm)
        self._gemm(s, 3 * self.Hl, H, T["a"], p["w_qkv"], [T["q"], self.rows(self.k, i), self.rows(self.v, i)],
                   bias=p["b_qkv"], stream=strm)
        ids, ks, vs = self._kv(i)
        ae = self._attn_ev(strm)
        self.ctx.attn_fwd(self.L, i, T["q"], ids, ks, vs, o=T["o"], lse=T["lse"], stream=strm)
        if ae is not None:
            ae.record(strm)
        self.launches += 2

    def forward_b(self, i, x, strm):
        """Out-projection + residual, LN2, MLP of chunk i (needs only forward_a(i))."""
        p, H, s = self.p, self.H, self.L.chunk_len(i)
        T = self.T[i]
        Hl, r0 = self.Hl, self.tp_rank == 0
        # row-parallel out-proj: partial sums over the local heads; the bias and the
        # residual enter once (rank 0), then the all-reduce sums the ranks' partials
        self._gemm(s, H, Hl, T["o"], p["w_o"], T["y"], bias=p["b_o"] if r0 else None,
                   residual=self.rows(x, i) if r0 else None, stream=strm)
        self._allreduce(T["y"], strm)
        self.ctx.layernorm_fwd(T["y"], p["ln2_g"], p["ln2_b"], T["b"], T["mu2"], T["rstd2"], eps=LN_EPS,
                               stream=strm)
        self._gemm(s, 4 * Hl, H, T["b"], p["w_1"], T["g"], bias=p["b_1"], aux_out=T["u"],
                   epilogue=sppo.SPPO_EPI_GELU, stream=strm)
        self._gemm(s, H, 4 * Hl, T["g"], p["w_2"], self.rows(self.z, i), bias=p["b_2"] if r0 else None,
                   residual=T["y"] if r0 else None, stream=strm)
        self._allreduce(self.rows(self.z, i), strm)
        self.launches += 1

    # ------------------------------------------------------------------ backward of chunk i
    def backward_chunk(self, i, x, dz, strm):
        end = self._ev("bwd", strm)
        self.backward_b(i, x, dz, strm)
        self.backward_a(i, x, dz, strm)
        if end is not None:
            end.record(strm)

    def backward_b(self, i, x, dz, strm, buf=0):
        """MLP, LN2 and out-projection backward of chunk i (needs only dz_i): writes
        d_o and dy into scratch set `buf`; accumulates w_2, w_1, w_o, LN2 gradients."""
        p, gr, H, s = self.p, self.grads, self.H, self.L.chunk_len(i)
        T = self.T[i]
        ctx = self.ctx
        du, dbn = self.du[:s], self.dbn[:s]
        dy, d_o = self.dy2[buf][:s], self.d_o2[buf][:s]
        dzi = self.rows(dz, i)
        acc = sppo.SPPO_EPI_ACC_F32
        # MLP: fc2 then fc1
        Hl = self.Hl
        self._gemm(s, 4 * Hl, H, dzi, p["w_2"], du, b_mn=1, aux_in=T["u"], epilogue=sppo.SPPO_EPI_DGELU,
                   stream=strm)
        self._gemm(H, 4 * Hl, s, dzi, T["g"], gr["w_2"], a_mn=1, b_mn=1, epilogue=acc, stream=strm)
        ctx.col_reduce(dzi, s, H, gr["b_2"], stream=strm)
        self._gemm(s, H, 4 * Hl, du, p["w_1"], dbn, b_mn=1, stream=strm)
        self._allreduce(dbn, strm)  # the LN2 input gradient sums the ranks' column-parallel fc1 parts
        self._gemm(4 * Hl, H, s, du, T["b"], gr["w_1"], a_mn=1, b_mn=1, epilogue=acc, stream=strm)
        ctx.col_reduce(du, s, 4 * Hl, gr["b_1"], stream=strm)
        # LN2 (+ residual stream gradient dz)
        ctx.layernorm_bwd(dbn, T["y"], p["ln2_g"], T["mu2"], T["rstd2"], dy, dres=dzi, stream=strm)
        ctx.col_reduce(dbn, s, H, gr["ln2_b"], x=T["y"], mean=T["mu2"], rstd=T["rstd2"], prod_acc=gr["ln2_g"],
                       stream=strm)
        # out-proj
        self._gemm(s, Hl, H, dy, p["w_o"], d_o, b_mn=1, stream=strm)
        self._gemm(H, Hl, s, dy, T["o"], gr["w_o"], a_mn=1, b_mn=1, epilogue=acc, stream=strm)
        ctx.col_reduce(dy, s, H, gr["b_o"], stream=strm)
        self.launches += 5

    def backward_a(self, i, x, dz, strm, buf=0):
        """Attention backward of chunk i (after chunk i+1's), QKV projection and LN1
        backward; reads d_o / dy of scratch set `buf`."""
        p, gr, H, s = self.p, self.grads, self.H, self.L.chunk_len(i)
        T = self.T[i]
        ctx = self.ctx
        da, dy, d_o = self.da[:s], self.dy2[buf][:s], self.d_o2[buf][:s]
        dq, dk, dv = self.dq[:s], self.dkc[:s], self.dvc[:s]
        xi = self.rows(x, i)
        acc = sppo.SPPO_EPI_ACC_F32
        # attention of chunk i against K/V of chunks 0..i; dK_i, dV_i final afterwards (L11)
        ids, ks, vs = self._kv(i)
        ae = self._attn_ev(strm)
        ctx.attn_bwd(self.L, i, T["q"], ids, ks, vs, T["o"], T["lse"], d_o, self.delta[:s * self.heads],
                     self.dq_acc[:s], [self.rows(self.dk_acc, j) for j in ids],
                     [self.rows(self.dv_acc, j) for j in ids], dq=dq, dk=dk, dv=dv, stream=strm)
        if ae is not None:
            ae.record(strm)
        # QKV projection from the three gradient parts, then LN1 (+ dy)
        Hl = self.Hl
        self._gemm(s, H, 3 * Hl, [dq, dk, dv], p["w_qkv"], da, b_mn=1, stream=strm)
        self._allreduce(da, strm)  # the LN1 input gradient sums the ranks' column-parallel QKV parts
        self._gemm(3 * Hl, H, s, [dq, dk, dv], T["a"], gr["w_qkv"], a_mn=1, b_mn=1, epilogue=acc, stream=strm)
        ctx.col_reduce([dq, dk, dv], s, 3 * Hl, gr["b_qkv"], stream=strm)
        ctx.layernorm_bwd(da, xi, p["ln1_g"], T["mu1"], T["rstd1"], self.rows(self.dx, i), dres=dy, stream=strm)
        ctx.col_reduce(da, s, H, gr["ln1_b"], x=xi, mean=T["mu1"], rstd=T["rstd1"], prod_acc=gr["ln1_g"],
                       stream=strm)
        self.launches += 3 + 3  # attention bwd (Delta preprocess, main, dQ cast) + LN1 bwd + 2 column reductions
        if self.pool:
            self.T[i] = None  # released: later allocations on this stream are ordered after these kernels

    def _zero(self):
        for t in self.grads.values():
            t.zero_()
        self.dk_acc.zero_()
        self.dv_acc.zero_()

    # ------------------------------------------------------------------ one step, no offload
    def step(self, x, dz, stream=None, mark=None):
        """Forward over chunks 0..N-1 then backward over N-1..0, nothing offloaded.
        With ``self.streams == 2`` the token-wise halves run on a second stream:
        forward_b(i) (out-proj, MLP) overlaps forward_a(i+1) (QKV, attention), and
        backward_b(i-1) overlaps backward_a(i) — the chunk-level parallelism the
        layer has inside one GPU (the attention of chunk i+1 does not depend on
        chunk i's MLP), which fills the tails of each other's launches."""
        strm = stream or torch.cuda.current_stream()
        with torch.cuda.stream(strm):  # torch-side allocations / copies ordered on strm
            return self._step(x, dz, strm, mark)

    def _step(self, x, dz, strm, mark):
        self._zero()
        if self.streams < 2 or self.timing:
            for i in range(self.N):
                self.forward_chunk(i, x, strm)
            if mark is not None:
                mark.record(strm)
            for i in range(self.N - 1, -1, -1):
                self.backward_chunk(i, x, dz, strm)
            return dict(z=self.z, dx=self.dx, grads=self.grads)
        if self._side is None:
            self._side = torch.cuda.Stream(device=self.device)
        s2 = self._side
        ev = lambda st: (lambda e: (e.record(st), e)[1])(torch.cuda.Event())  # noqa: E731
        s2.wait_event(ev(strm))  # zeroed accumulators
        for i in range(self.N):
            self.forward_a(i, x, strm)
            s2.wait_event(ev(strm))
            self.forward_b(i, x, s2)
        strm.wait_event(ev(s2))
        if mark is not None:
            mark.record(strm)
        s2.wait_event(ev(strm))
        done_a = {}
        for i in range(self.N - 1, -1, -1):
            buf = i % 2
            if i + 2 in done_a:
                s2.wait_event(done_a.pop(i + 2))  # backward_a(i+2) has read scratch set `buf`
            self.backward_b(i, x, dz, s2, buf)
            strm.wait_event(ev(s2))
            self.backward_a(i, x, dz, strm, buf)
            done_a[i] = ev(strm)
        strm.wait_event(ev(s2))
        return dict(z=self.z, dx=self.dx, grads=self.grads)

    # ------------------------------------------------------------------ end to end through host buffers
    def step_host_io(self, host_x, host_dz, host_z, host_dx, x, dz, stream=None):
        """One step whose input x and upstream gradient dz start in pinned host
        memory and whose results z, dx end there: x_i arrives H2D chunk by chunk in
        forward order and dz_i in backward order (sppo_kv_prefetch, deferred waits:
        the copies overlap compute), z_i leaves after fwd(i) and dx_i after bwd(i)
        (sppo_kv_offload).  x, dz: device staging buffers [S, h].  Returns
        (h2d_bytes, d2h_bytes, last_d2h_event)."""
        strm = stream or torch.cuda.current_stream()
        H, c = self.H, self.L.offsets
        row = H * 2
        ready_x, ready_dz = [], [None] * self.N
        h2d = d2h = 0
        # copies are ordered after the work already on `strm` (a previous step still
        # reading x / dz); nothing of this step is enqueued yet, so they do not wait
        # on each other's consumers
        for i in range(self.N):  # issue order = consumption order on the H2D stream
            ev = torch.cuda.Event()
            nb = (c[i + 1] - c[i]) * row
            self.ctx.kv_prefetch(i, host_x + c[i] * row, self.rows(x, i), nb, consumer=strm, done=ev,
                                 flags=sppo.SPPO_COPY_DEFER_WAIT)
            ready_x.append(ev)
            h2d += nb
        for i in range(self.N - 1, -1, -1):
            ev = torch.cuda.Event()
            nb = (c[i + 1] - c[i]) * row
            self.ctx.kv_prefetch(i, host_dz + c[i] * row, self.rows(dz, i), nb, consumer=strm, done=ev,
                                 flags=sppo.SPPO_COPY_DEFER_WAIT)
            ready_dz[i] = ev
            h2d += nb
        self._zero()
        # z_i / dx_i device rows are rewritten only after the previous call's D2H of them (WAR)
        prev = getattr(self, "_io_prev", {})
        self._io_prev = cur = {}
        last = None
        for i in range(self.N):
            strm.wait_event(ready_x[i])
            if ("z", i) in prev:
                strm.wait_event(prev[("z", i)])
            self.forward_chunk(i, x, strm)
            nb = (c[i + 1] - c[i]) * row
            last = torch.cuda.Event()
            d2h += self.ctx.kv_offload(i, self.rows(self.z, i), host_z + c[i] * row, nb, 1.0, producer=strm, done=last)
            cur[("z", i)] = last
        for i in range(self.N - 1, -1, -1):
            strm.wait_event(ready_dz[i])
            if ("dx", i) in prev:
                strm.wait_event(prev[("dx", i)])
            self.backward_chunk(i, x, dz, strm)
            nb = (c[i + 1] - c[i]) * row
            last = torch.cuda.Event()
            d2h += self.ctx.kv_offload(i, self.rows(self.dx, i), host_dx + c[i] * row, nb, 1.0, producer=strm,
                                       done=last)
            cur[("dx", i)] = last
        return h2d, d2h, last

    # ------------------------------------------------------------------ Type-1 offload with alpha
    def type1_bytes(self, i):
        """A_i: bytes of chunk i's Type-1 tensors."""
        s = self.L.chunk_len(i)
        tot = 0
        for n in TYPE1 + STATS:
            shape, dt = self._t1_shape(n, s)
            numel = 1
            for e in shape:
                numel *= e
            tot += numel * (2 if dt == torch.bfloat16 else 4)
        return tot

    def _host_buf(self, key, nbytes):
        if key not in self._host:
            self._host[key] = (self.ctx.host_alloc(nbytes), nbytes)
        return self._host[key][0]

    def free_host(self):
        for ptr, _ in self._host.values():
            self.ctx.host_free(ptr)
        self._host.clear()

    def step_offload(self, x, dz, alpha, stream=None, depth: int = 2, poison: bool = False, mark=None):
        """Forward + backward with the alpha_i-prefix of every Type-1 tensor of
        chunk i offloaded after fwd(i) and prefetched before bwd(i).  pool mode:
        the offloaded device memory is released once its D2H completes (see the
        module docstring).  ``poison`` (resident mode): the offloaded device bytes
        are overwritten once the D2H completes, proving the backward reads the
        prefetched bytes.  Returns bytes moved per direction."""
        strm = stream or torch.cuda.current_stream()
        with torch.cuda.stream(strm):  # torch-side allocations / suffix copies ordered on strm
            return self._step_offload(x, dz, alpha, strm, depth, poison, mark)

    def _step_offload(self, x, dz, alpha, strm, depth, poison, mark):
        self._zero()
        moved = {"d2h": 0, "h2d": 0}
        plan, done = {}, {}
        # pool: per offloaded chunk, (its last D2H event, its device tensors).  The
        # host enqueues far ahead of the GPU, so completed copies cannot be found by
        # polling alone: with more than `inflight` chunks pending the host waits for
        # the oldest one's D2H (the GPU still has the chunks enqueued since then).
        pending = []

        def reap(block=False, inflight=2):
            while pending and (block or len(pending) > inflight or pending[0][0].query()):
                pending[0][0].synchronize()
                pending.pop(0)

        for i in range(self.N):
            self.forward_chunk(i, x, strm)
            a = float(alpha[i])
            if a <= 0.0:
                continue
            parts = {}
            held = []
            T = self.T[i]
            for name in TYPE1 + STATS:
                t = T[name]
                nb = t.numel() * t.element_size()
                host = self._host_buf((name, i), nb)
                ev = torch.cuda.Event()
                n = self.ctx.kv_offload(i, t, host, nb, alpha=(a if name in TYPE1 else 1.0), producer=strm, done=ev)
                moved["d2h"] += n
                suffix = None
                if self.pool:
                    if n < nb:  # keep the resident suffix compactly (device copy, ordered after fwd(i))
                        suffix = t.reshape(-1).view(torch.uint8)[n:].clone()
                    held.append(t)
                    T[name] = None
                elif poison:
                    strm.wait_event(ev)
                    t.reshape(-1).view(torch.uint8)[:n].fill_(0xFF)
                parts[name] = (host, n, nb, suffix, ev)
            plan[i] = parts
            if self.pool:
                self.T[i] = None
                pending.append((ev, held))  # ev: this chunk's last D2H (the D2H stream is in order)
                del T, t, held
                reap()
        if mark is not None:
            mark.record(strm)
        issued = set()

        def prefetch(i):
            if i < 0 or i in issued or i not in plan:
                return
            issued.add(i)
            T = self._t1_set(i) if self.pool else self.T[i]
            evs = []
            for name, (host, n, nb, suffix, ev) in plan[i].items():
                t = T[name]
                strm.wait_event(ev)  # the bytes reached the host (its D2H completed)
                pe = torch.cuda.Event()
                # ordered after the work already on strm (the fresh allocation's previous users)
                self.ctx.kv_prefetch(i, host, t, n, consumer=strm, done=pe, flags=sppo.SPPO_COPY_DEFER_WAIT)
                moved["h2d"] += n
                if suffix is not None:
                    t.reshape(-1).view(torch.uint8)[n:].copy_(suffix)
                evs.append(pe)
            if self.pool:
                self.T[i] = T
            done[i] = evs
            plan[i] = {}  # drop the suffix copies (released after the restores enqueued above)

        for i in range(self.N - 1, -1, -1):
            for dd in range(depth):
                prefetch(i - dd)
            for pe in done.get(i, []):
                strm.wait_event(pe)
            self.backward_chunk(i, x, dz, strm)
            if self.pool:
                reap()
        reap(block=True)
        return moved

    def alpha_plan(self, fwd_ms, bw_d2h_gbs):
        """Sequence-aware alpha from measured per-chunk forward
        times: alpha_i = min(1, BW_D2H * T_fwd(i+1) / A_i), alpha_{N-1} = 0."""
        A = [float(self.type1_bytes(i)) for i in range(self.N)]
        M = [bw_d2h_gbs * 1e9 * (fwd_ms[i + 1] * 1e-3) if i + 1 < self.N else 0.0 for i in range(self.N)]
        return sppo.offload_alpha(A, M, last=0.0)
