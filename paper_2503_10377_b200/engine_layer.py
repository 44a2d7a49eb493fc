"""Chunk-loop orchestration of one GPT transformer layer over the C ABI
(include/sppo.h + include/sppo_layer.h).

One step = the layer forward over chunks i = 0..N-1, then its backward over
i = N-1..0 (reading L11).  Per chunk i (token rows [c_i, c_{i+1})):

  forward   a = LN1(x)                       sppo_layernorm_fwd
            [q k v] = a W_qkv^T + b_qkv      sppo_gemm (C split into Q | K | V)
            o = attention(q; K, V of 0..i)   sppo_attn_fwd  (ChunkedAttention)
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
(Type-0); the Type-1 tensors of chunk i — a, q, o, y, b, u, g (13 h bf16 per
token) plus LSE and the LayerNorm statistics — leave after fwd(i) as the
alpha_i-prefix of each token-major buffer on the ctx D2H stream (overlapping
fwd(i+1)) and come back on the H2D stream before bwd(i), at most
``depth`` chunks ahead.  alpha_i = min(1, BW_D2H * T_fwd(i+1) / A_i),
alpha_{N-1} = 0 (reading L9).  This module allocates buffers and
sequences ABI calls; every arithmetic step runs in libsppo's kernels.
"""

from __future__ import annotations

import torch

from . import sppo
from .engine import ChunkedAttention

PARAM_NAMES = ("ln1_g", "ln1_b", "w_qkv", "b_qkv", "w_o", "b_o", "ln2_g", "ln2_b", "w_1", "b_1", "w_2", "b_2")
TYPE1 = ("a", "q", "o", "y", "b", "u", "g")  # token-major bf16 activations offloaded with alpha
STATS = ("mu1", "rstd1", "mu2", "rstd2")     # fp32 [S] per-token LayerNorm statistics (offloaded whole)
LN_EPS = 1e-5


class ChunkedLayer:
    def __init__(self, ctx: sppo.Context, hidden: int, heads: int, offsets, params: dict, device="cuda",
                 timing: bool = False):
        self.ctx = ctx
        self.H, self.heads = hidden, heads
        self.d = hidden // heads
        self.L = sppo.Layout(heads, self.d, offsets, dtype=sppo.SPPO_BF16)
        self.N = self.L.num_chunks
        self.S = S = self.L.offsets[-1]
        self.device = torch.device(device)
        self.p = params
        self.timing = timing
        H = hidden
        bf = dict(dtype=torch.bfloat16, device=self.device)
        f32 = dict(dtype=torch.float32, device=self.device)
        self.att = ChunkedAttention(ctx, self.L, device=device, fwd_streams=1)
        # saved activations (whole sequence, token-major; chunk i = rows [c_i, c_{i+1}))
        self.a = torch.empty((S, H), **bf)
        self.q = torch.empty((S, H), **bf)
        self.k = torch.empty((S, H), **bf)
        self.v = torch.empty((S, H), **bf)
        self.o = self.att.o.view(S, H)
        self.y = torch.empty((S, H), **bf)
        self.b = torch.empty((S, H), **bf)
        self.u = torch.empty((S, 4 * H), **bf)
        self.g = torch.empty((S, 4 * H), **bf)
        self.z = torch.empty((S, H), **bf)
        for n in STATS:
            setattr(self, n, torch.empty((S,), **f32))
        # backward: outputs and per-chunk scratch (longest chunk)
        smax = max(self.L.chunk_len(i) for i in range(self.N))
        self.dx = torch.empty((S, H), **bf)
        self.d_o = torch.empty((S, H), **bf)
        self.du = torch.empty((smax, 4 * H), **bf)
        self.dbn = torch.empty((smax, H), **bf)
        self.dy = torch.empty((smax, H), **bf)
        self.da = torch.empty((smax, H), **bf)
        self.grads = {n: torch.zeros(tuple(params[n].shape), **f32) for n in PARAM_NAMES}
        self.launches = 0
        self.events = {"fwd": [], "bwd": []}
        self.gemm_events = None  # list: (start, end, FLOPs) of every GEMM call (bench instrumentation)
        self._host = {}

    # ------------------------------------------------------------------ helpers
    def rows(self, t, i):
        c = self.L.offsets
        return t[c[i]:c[i + 1]]

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

    # ------------------------------------------------------------------ forward of chunk i
    def forward_chunk(self, i, x, strm):
        p, H, s = self.p, self.H, self.L.chunk_len(i)
        end = self._ev("fwd", strm)
        r = lambda t: self.rows(t, i)  # noqa: E731
        self.ctx.layernorm_fwd(r(x), p["ln1_g"], p["ln1_b"], r(self.a), r(self.mu1), r(self.rstd1), eps=LN_EPS,
                               stream=strm)
        self._gemm(s, 3 * H, H, r(self.a), p["w_qkv"], [r(self.q), r(self.k), r(self.v)], bias=p["b_qkv"],
                   stream=strm)
        S = self.S
        self.att.forward_chunk(i, self.q.view(S, self.heads, self.d), self.k.view(S, self.heads, self.d),
                               self.v.view(S, self.heads, self.d), strm)
        self._gemm(s, H, H, r(self.o), p["w_o"], r(self.y), bias=p["b_o"], residual=r(x), stream=strm)
        self.ctx.layernorm_fwd(r(self.y), p["ln2_g"], p["ln2_b"], r(self.b), r(self.mu2), r(self.rstd2),
                               eps=LN_EPS, stream=strm)
        self._gemm(s, 4 * H, H, r(self.b), p["w_1"], r(self.g), bias=p["b_1"], aux_out=r(self.u),
                   epilogue=sppo.SPPO_EPI_GELU, stream=strm)
        self._gemm(s, H, 4 * H, r(self.g), p["w_2"], r(self.z), bias=p["b_2"], residual=r(self.y), stream=strm)
        self.launches += 3
        if end is not None:
            end.record(strm)

    # ------------------------------------------------------------------ backward of chunk i
    def backward_chunk(self, i, x, dz, strm):
        p, gr, H, s = self.p, self.grads, self.H, self.L.chunk_len(i)
        end = self._ev("bwd", strm)
        r = lambda t: self.rows(t, i)  # noqa: E731
        ctx = self.ctx
        du, dbn, dy, da = self.du[:s], self.dbn[:s], self.dy[:s], self.da[:s]
        dzi = r(dz)
        acc = sppo.SPPO_EPI_ACC_F32
        # MLP: fc2 then fc1
        self._gemm(s, 4 * H, H, dzi, p["w_2"], du, b_mn=1, aux_in=r(self.u), epilogue=sppo.SPPO_EPI_DGELU,
                   stream=strm)
        self._gemm(H, 4 * H, s, dzi, r(self.g), gr["w_2"], a_mn=1, b_mn=1, epilogue=acc, stream=strm)
        ctx.col_reduce(dzi, s, H, gr["b_2"], stream=strm)
        self._gemm(s, H, 4 * H, du, p["w_1"], dbn, b_mn=1, stream=strm)
        self._gemm(4 * H, H, s, du, r(self.b), gr["w_1"], a_mn=1, b_mn=1, epilogue=acc, stream=strm)
        ctx.col_reduce(du, s, 4 * H, gr["b_1"], stream=strm)
        # LN2 (+ residual stream gradient dz)
        ctx.layernorm_bwd(dbn, r(self.y), p["ln2_g"], r(self.mu2), r(self.rstd2), dy, dres=dzi, stream=strm)
        ctx.col_reduce(dbn, s, H, gr["ln2_b"], x=r(self.y), mean=r(self.mu2), rstd=r(self.rstd2),
                       prod_acc=gr["ln2_g"], stream=strm)
        # out-proj
        self._gemm(s, H, H, dy, p["w_o"], r(self.d_o), b_mn=1, stream=strm)
        self._gemm(H, H, s, dy, r(self.o), gr["w_o"], a_mn=1, b_mn=1, epilogue=acc, stream=strm)
        ctx.col_reduce(dy, s, H, gr["b_o"], stream=strm)
        # attention of chunk i against K/V of chunks 0..i; dK_i, dV_i final afterwards (L11)
        S, hd = self.S, (self.S, self.heads, self.d)
        self.att.backward_chunk(i, self.q.view(*hd), self.k.view(*hd), self.v.view(*hd), self.d_o.view(*hd), strm)
        dq, dk, dv = (r(t.view(S, H)) for t in (self.att.dq, self.att.dk, self.att.dv))
        # QKV projection from the three gradient parts, then LN1 (+ dy)
        self._gemm(s, H, 3 * H, [dq, dk, dv], p["w_qkv"], da, b_mn=1, stream=strm)
        self._gemm(3 * H, H, s, [dq, dk, dv], r(self.a), gr["w_qkv"], a_mn=1, b_mn=1, epilogue=acc, stream=strm)
        ctx.col_reduce([dq, dk, dv], s, 3 * H, gr["b_qkv"], stream=strm)
        ctx.layernorm_bwd(da, r(x), p["ln1_g"], r(self.mu1), r(self.rstd1), r(self.dx), dres=dy, stream=strm)
        ctx.col_reduce(da, s, H, gr["ln1_b"], x=r(x), mean=r(self.mu1), rstd=r(self.rstd1), prod_acc=gr["ln1_g"],
                       stream=strm)
        self.launches += 8
        if end is not None:
            end.record(strm)

    def _zero(self):
        for t in self.grads.values():
            t.zero_()
        self.att.dk_acc.zero_()
        self.att.dv_acc.zero_()

    # ------------------------------------------------------------------ one step, resident
    def step(self, x, dz, stream=None, mark=None):
        """Forward over chunks 0..N-1 then backward over N-1..0, all resident."""
        strm = stream or torch.cuda.current_stream()
        self._zero()
        for i in range(self.N):
            self.forward_chunk(i, x, strm)
        if mark is not None:
            mark.record(strm)
        for i in range(self.N - 1, -1, -1):
            self.backward_chunk(i, x, dz, strm)
        return dict(z=self.z, dx=self.dx, grads=self.grads)

    # ------------------------------------------------------------------ Type-1 offload with alpha
    def type1_tensors(self, i):
        """(name, chunk view, alpha applies) of chunk i's Type-1 tensors."""
        out = [(n, self.rows(getattr(self, n), i), True) for n in TYPE1]
        out.append(("lse", self.att.lse_view(i), False))
        out += [(n, self.rows(getattr(self, n), i), False) for n in STATS]
        return out

    def type1_bytes(self, i):
        """A_i: bytes of chunk i's Type-1 tensors."""
        return sum(t.numel() * t.element_size() for _, t, _ in self.type1_tensors(i))

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
        chunk i offloaded after fwd(i) and prefetched before bwd(i).  With
        ``poison`` the offloaded device bytes are overwritten (NaN pattern) once
        the D2H completes, proving the backward reads the prefetched bytes.
        Returns bytes moved per direction."""
        strm = stream or torch.cuda.current_stream()
        self._zero()
        moved = {"d2h": 0, "h2d": 0}
        plan, done = {}, {}
        for i in range(self.N):
            self.forward_chunk(i, x, strm)
            a = float(alpha[i])
            if a <= 0.0:
                continue
            parts = []
            for name, t, scaled in self.type1_tensors(i):
                nb = t.numel() * t.element_size()
                host = self._host_buf((name, i), nb)
                ev = torch.cuda.Event()
                n = self.ctx.kv_offload(i, t, host, nb, alpha=(a if scaled else 1.0), producer=strm, done=ev)
                moved["d2h"] += n
                parts.append((t, host, n, ev))
            plan[i] = parts
            if poison:
                for t, _, n, ev in parts:
                    strm.wait_event(ev)
                    t.reshape(-1).view(torch.uint8)[:n].fill_(0xFF)
        if mark is not None:
            mark.record(strm)
        issued = set()

        def prefetch(i):
            if i < 0 or i in issued or i not in plan:
                return
            issued.add(i)
            evs = []
            for t, host, n, ev in plan[i]:
                strm.wait_event(ev)  # the bytes reached the host (its D2H completed)
                pe = torch.cuda.Event()
                self.ctx.kv_prefetch(i, host, t, n, consumer=strm, done=pe, flags=sppo.SPPO_COPY_DEFER_WAIT)
                moved["h2d"] += n
                evs.append(pe)
            done[i] = evs

        for i in range(self.N - 1, -1, -1):
            for dd in range(depth):
                prefetch(i - dd)
            for pe in done.get(i, []):
                strm.wait_event(pe)
            self.backward_chunk(i, x, dz, strm)
        return moved

    def alpha_plan(self, fwd_ms, bw_d2h_gbs):
        """Sequence-aware alpha from measured per-chunk forward
        times: alpha_i = min(1, BW_D2H * T_fwd(i+1) / A_i), alpha_{N-1} = 0."""
        A = [float(self.type1_bytes(i)) for i in range(self.N)]
        M = [bw_d2h_gbs * 1e9 * (fwd_ms[i + 1] * 1e-3) if i + 1 < self.N else 0.0 for i in range(self.N)]
        return sppo.offload_alpha(A, M, last=0.0)
