"""Chunk-loop orchestration of one SPPO attention step over the C ABI.

One step = forward over chunks i = 0..N-1 (ascending) then backward over
i = N-1..0 (reading L11), each chunk's prior-KV set 0..i visited in windows of
at most ``window`` chunks (FIRST/LAST carry).  Every compute
step is a call into libsppo (sppo_attn_fwd / sppo_attn_bwd) and every copy a
call to sppo_kv_offload / sppo_kv_prefetch; this module only allocates buffers
(torch device memory, pinned host memory from sppo_host_alloc) and sequences
the calls.

Two-level activation management (P:356 [§5.1], P:369-377 [§5.2]):
  * level 1 (GPU): K_j, V_j of every chunk stay resident (Type-0);
  * level 2 (host): the Type-1 tensors of chunk i (Q_i, O_i, LSE_i — used once
    in forward, once in backward) are offloaded with ratio alpha_i right after
    fwd(i) on the D2H stream, overlapping fwd(i+1), and prefetched on
    the H2D stream before bwd(i), at most ``depth`` chunks ahead.
    alpha_i = min(1, BW_D2H * T_fwd(i+1) / A_i), alpha_{N-1} = 0 (reading L9).

Buffer layout in HBM: full-sequence token-major tensors
[S, h, d] whose chunk i is the contiguous row range [c_i, c_{i+1}); LSE stored
chunk after chunk, each chunk head-major [h, s_i]; fp32 dK/dV accumulators for
the whole sequence; per-chunk fp32 scratch (dQ accumulator, Delta, fwd carry)
sized for the longest chunk and reused.
"""

from __future__ import annotations

import functools
import os
import inspect

import torch

from . import sppo


def _on_step_stream(fn):
    """Runs a step method with torch's current stream set to its ``stream``
    argument, so the torch-side work inside it (accumulator zeroing, poison
    fills, allocations) is ordered with the ABI calls enqueued on that stream."""
    sig = inspect.signature(fn)

    @functools.wraps(fn)
    def run(self, *args, **kwargs):
        b = sig.bind(self, *args, **kwargs)
        strm = b.arguments.get("stream") or torch.cuda.current_stream()
        b.arguments["stream"] = strm
        with torch.cuda.stream(strm):
            return fn(*b.args, **b.kwargs)
    return run

DTYPES = {sppo.SPPO_BF16: torch.bfloat16, sppo.SPPO_FP32: torch.float32}
DTYPE_BYTES = {sppo.SPPO_BF16: 2, sppo.SPPO_FP32: 4}


class ChunkedAttention:
    def __init__(self, ctx: sppo.Context, layout: sppo.Layout, device="cuda", window: int | None = None,
                 timing: bool = False, fwd_streams: int | None = None, fwd_group: int | None = None):
        self.ctx, self.L = ctx, layout
        # resident step(): forward chunks are independent (chunk i reads only inputs), so
        # consecutive forward launches may alternate between two streams and the next one
        # fills the SMs the previous one's last wave leaves idle.  Measured: worth it
        # when a launch is a few waves and its K/V sweep is short (C2 per-GPU shares at
        # 2-8 GPUs: +5 %), harmful when two concurrent kernels sweep long, different K/V
        # ranges (C3, 14 waves, 17 GB of K/V: -11 % forward; the C5 per-GPU share,
        # 3.5 waves but 17 GB: -10 %, profiles/r02).  Default: two streams below 8
        # waves of CTAs per launch and at most 4 GB of K/V behind the last chunk.
        # Grouped KV streaming shares ONE window between the concurrent launches, so
        # there the wave count alone decides (C5 share: -2 % step time).
        smax = max(layout.chunk_len(i) for i in range(layout.num_chunks))
        ctas = -(-smax // 256) * layout.heads  # fwd_kernel: 2 Q tiles of 128 rows per CTA
        sms = torch.cuda.get_device_properties(torch.device(device)).multi_processor_count \
            if torch.cuda.is_available() else 148
        self._few_waves = ctas < 8 * sms
        if fwd_streams is None:
            kv_bytes = layout.offsets[-1] * layout.heads * layout.head_dim * 2 * \
                torch.tensor([], dtype=DTYPES[layout.dtype]).element_size()
            fwd_streams = 2 if (self._few_waves and kv_bytes <= 4e9) else 1
        self.fwd_streams = fwd_streams
        # resident step(): all forward chunks in ONE launch (sppo_attn_fwd_chunks, bf16,
        # single window per chunk), longest chunks first — no per-launch wave tails or
        # launch gaps, and the CTAs of all chunks sweep the shared K/V together
        # — while one head's K/V sweep stays moderate.  The CTAs of different chunks start
        # at different times, so with several GB per head they stream it out of step
        # (C5 per-GPU share, 2 GB of K/V per head: forward 977.6 in one launch vs 1000.1
        # per chunk; C3, 0.5 GB per head: 1126.7 in one launch); there the launches take
        # groups of consecutive chunks (nearly the same key range) of >= 8 waves, so a
        # group's CTAs stay together and the per-chunk launches' last-wave tails go
        # (C5 share: a 16K chunk is 512 CTAs = 3.5 waves)
        kv_head = layout.offsets[-1] * layout.head_dim * 2 * DTYPE_BYTES.get(layout.dtype, 4)
        self.fwd_multi = (layout.dtype == sppo.SPPO_BF16 and layout.num_chunks <= 256
                          and os.environ.get("SPPO_FWD_MULTI", "1") != "0")
        if fwd_group is None and os.environ.get("SPPO_FWD_GROUP"):
            fwd_group = int(os.environ["SPPO_FWD_GROUP"])
        if fwd_group is None:
            # >= 8 waves per launch (choosing the group whose last wave is fullest instead,
            # 4 chunks = 13.84 waves at the C5 share, measured fwd 1013.0 vs 1022.4)
            fwd_group = layout.num_chunks if kv_head <= 1 << 30 else -(-8 * sms // max(1, ctas))
        self.fwd_group = max(1, min(fwd_group, layout.num_chunks))
        self._side = None
        # instrumentation (tools/offload_timeline.py): when a list, every compute call
        # and every copy appends {kind, chunk, bytes, events}; see _tl_begin/_tl_end
        self.timeline = None
        self._copy_streams = None
        self.device = torch.device(device)
        self.window = window if window else 10**9
        self.timing = timing
        self.launches = 0
        self.events = {"fwd": [], "bwd": []}
        h, d = layout.heads, layout.head_dim
        S = layout.offsets[-1]
        smax = max(layout.chunk_len(i) for i in range(layout.num_chunks))
        dt = DTYPES[layout.dtype]
        self.elem = torch.tensor([], dtype=dt).element_size()
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
        self._host = {}

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

    def _ev(self, kind, stream):
        if not self.timing:
            return None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        self.events[kind].append((e0, e1))
        return e1

    def _tl_begin(self, kind, i, stream, nbytes=0, copy=None):
        """copy=None: a compute call on `stream` (start event).  copy='d2h'/'h2d': an
        event on that ctx copy stream before the call plus one on `stream` (the
        producer / consumer): the copy starts at the later of the two."""
        if self.timeline is None:
            return None
        ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
        rec = {"kind": kind, "chunk": i, "bytes": nbytes}
        if copy is None:
            rec["e0"] = ev()
            rec["e0"].record(stream)
        else:
            if self._copy_streams is None:
                d2h, h2d = self.ctx.copy_streams()
                self._copy_streams = {"d2h": torch.cuda.ExternalStream(d2h), "h2d": torch.cuda.ExternalStream(h2d)}
            rec["cs"] = self._copy_streams[copy]
            rec["eb"], rec["ep"] = ev(), ev()
            rec["eb"].record(rec["cs"])
            rec["ep"].record(stream)
        return rec

    def _tl_end(self, rec, stream=None):
        if rec is None:
            return
        rec["e1"] = torch.cuda.Event(enable_timing=True)
        rec["e1"].record(rec.get("cs", stream))
        self.timeline.append(rec)

    def kernel_ms(self, kind):
        """Sum of CUDA-event durations of the recorded calls (after a sync)."""
        return sum(a.elapsed_time(b) for a, b in self.events[kind])

    # forward / backward of one chunk ----------------------------------------
    def forward_chunk(self, i, q, k, v, stream=None):
        L = self.L
        s = L.chunk_len(i)
        h = L.heads
        wins = self.windows(i)
        state = (self.o_acc[:s], self.m[:s * h], self.l[:s * h])
        strm = stream or torch.cuda.current_stream()
        end = self._ev("fwd", strm)
        tl = self._tl_begin("fwd", i, strm)
        for n, ids in enumerate(wins):
            flags = (sppo.SPPO_FIRST if n == 0 else 0) | (sppo.SPPO_LAST if n == len(wins) - 1 else 0)
            self.ctx.attn_fwd(L, i, self.rows(q, i), ids, [self.rows(k, j) for j in ids],
                              [self.rows(v, j) for j in ids], flags=flags,
                              state=None if len(wins) == 1 else state,
                              o=self.rows(self.o, i), lse=self.lse_view(i), stream=strm)
            self.launches += 1
        self._tl_end(tl, strm)
        if end is not None:
            end.record(strm)

    def backward_chunk(self, i, q, k, v, do, stream=None):
        L = self.L
        s = L.chunk_len(i)
        h = L.heads
        wins = self.windows(i)
        strm = stream or torch.cuda.current_stream()
        end = self._ev("bwd", strm)
        tl = self._tl_begin("bwd", i, strm)
        for n, ids in enumerate(wins):
            flags = (sppo.SPPO_FIRST if n == 0 else 0) | (sppo.SPPO_LAST if n == len(wins) - 1 else 0)
            has_i = i in ids
            self.ctx.attn_bwd(L, i, self.rows(q, i), ids, [self.rows(k, j) for j in ids],
                              [self.rows(v, j) for j in ids], self.rows(self.o, i), self.lse_view(i),
                              self.rows(do, i), self.delta[:s * h], self.dq_acc[:s],
                              [self.rows(self.dk_acc, j) for j in ids], [self.rows(self.dv_acc, j) for j in ids],
                              dq=self.rows(self.dq, i), dk=self.rows(self.dk, i) if has_i else None,
                              dv=self.rows(self.dv, i) if has_i else None, flags=flags, stream=strm)
            # main kernel + Delta preprocess on FIRST + dQ cast on LAST
            self.launches += 1 + (flags & sppo.SPPO_FIRST != 0) + (flags & sppo.SPPO_LAST != 0)
        self._tl_end(tl, strm)
        if end is not None:
            end.record(strm)

    # one step, all activations resident ---------------------------------------
    @_on_step_stream
    def step(self, q, k, v, do, stream=None, mark=None):
        """Full forward + backward over all chunks (resident policy).  ``mark``
        (a torch.cuda.Event) is recorded between the forward and backward phases."""
        N = self.L.num_chunks
        strm = stream or torch.cuda.current_stream()
        self.dk_acc.zero_()
        self.dv_acc.zero_()
        if self.fwd_multi and self.window >= N and not self.timing and self.timeline is None:
            L, G = self.L, self.fwd_group
            ks, vs = [self.rows(k, j) for j in range(N)], [self.rows(v, j) for j in range(N)]
            for i0 in range(0, N, G):
                i1 = min(N, i0 + G)
                self.ctx.attn_fwd_chunks(L, i0, i1, [self.rows(q, i) for i in range(i0, i1)], ks[:i1], vs[:i1],
                                         [self.rows(self.o, i) for i in range(i0, i1)],
                                         [self.lse_view(i) for i in range(i0, i1)], stream=strm)
                self.launches += 1
            if mark is not None:
                mark.record(strm)
            for i in range(N - 1, -1, -1):
                self.backward_chunk(i, q, k, v, do, stream)
            return dict(o=self.o, lse=self.lse, dq=self.dq, dk=self.dk, dv=self.dv)
        # two forward streams only without split windows (those share the carry scratch)
        two = self.fwd_streams > 1 and N > 1 and self.window >= N
        if two:
            if self._side is None:
                self._side = torch.cuda.Stream(device=self.device)
            fork = torch.cuda.Event()
            fork.record(strm)
            self._side.wait_event(fork)
        for i in range(N):
            self.forward_chunk(i, q, k, v, self._side if (two and i % 2) else strm)
        if two:
            join = torch.cuda.Event()
            join.record(self._side)
            strm.wait_event(join)
        if mark is not None:
            mark.record(strm)
        for i in range(N - 1, -1, -1):
            self.backward_chunk(i, q, k, v, do, stream)
        return dict(o=self.o, lse=self.lse, dq=self.dq, dk=self.dk, dv=self.dv)

    # one step with Type-1 offload (two-level activation management) ----------
    def type1_bytes(self, i):
        """A_i: bytes of chunk i's Type-1 tensors (Q_i, O_i, LSE_i)."""
        s, h, d = self.L.chunk_len(i), self.L.heads, self.L.head_dim
        return 2 * s * h * d * self.elem + 4 * s * h

    def _host_buf(self, key, nbytes):
        if key not in self._host:
            self._host[key] = (self.ctx.host_alloc(nbytes), nbytes)
        return self._host[key][0]

    def free_host(self):
        for ptr, _ in self._host.values():
            self.ctx.host_free(ptr)
        self._host.clear()

    @_on_step_stream
    def step_offload(self, q, k, v, do, alpha, stream=None, depth: int = 2, poison: bool = False, mark=None):
        """Forward + backward where Q_i, O_i and LSE_i leave the GPU after fwd(i)
        (alpha_i-prefix of each token-major buffer, LSE whole when alpha_i > 0)
        and come back before bwd(i).  With ``poison`` the device copies are
        overwritten with NaN after the offload completes, proving that the
        backward reads the prefetched bytes.  Returns copy statistics."""
        L = self.L
        N = L.num_chunks
        strm = stream or torch.cuda.current_stream()
        self.dk_acc.zero_()
        self.dv_acc.zero_()
        moved = {"d2h": 0, "h2d": 0}
        plan = {}
        done = {}
        for i in range(N):
            self.forward_chunk(i, q, k, v, strm)
            a = float(alpha[i])
            if a <= 0.0:
                continue
            parts = []
            for name, t in (("q", self.rows(q, i)), ("o", self.rows(self.o, i)), ("lse", self.lse_view(i))):
                nb = t.numel() * t.element_size()
                host = self._host_buf((name, i), nb)
                ev = torch.cuda.Event()
                tl = self._tl_begin("d2h", i, strm, copy="d2h")
                n = self.ctx.kv_offload(i, t, host, nb, alpha=(a if name != "lse" else 1.0), producer=strm,
                                        done=ev)
                if tl is not None:
                    tl["bytes"] = n
                self._tl_end(tl)
                moved["d2h"] += n
                parts.append((name, t, host, n, ev))
            plan[i] = parts
            if poison:
                for _, t, _, n, ev in parts:
                    strm.wait_event(ev)
                    t.reshape(-1).view(torch.uint8)[:n].fill_(0xFF)  # first n BYTES: NaN pattern in bf16/fp32
        if mark is not None:
            mark.record(strm)
        issued = set()

        def prefetch(i):
            if i < 0 or i in issued or i not in plan:
                return
            issued.add(i)
            evs = []
            for name, t, host, n, ev in plan[i]:
                # bytes must have reached the host first (D2H of the offload)
                strm.wait_event(ev)
                pe = torch.cuda.Event()
                tl = self._tl_begin("h2d", i, strm, n, copy="h2d")
                self.ctx.kv_prefetch(i, host, t, n, consumer=strm, done=pe,
                                     flags=sppo.SPPO_COPY_DEFER_WAIT)
                self._tl_end(tl)
                moved["h2d"] += n
                evs.append(pe)
            done[i] = evs

        for i in range(N - 1, -1, -1):
            for dd in range(depth):
                prefetch(i - dd)
            for pe in done.get(i, []):
                strm.wait_event(pe)
            self.backward_chunk(i, q, k, v, do, strm)
        return moved

    # one step with KV streaming (hot prefix resident, cold chunks on host) -----
    @_on_step_stream
    def step_kv_stream(self, q, k, v, do, hot: int, window: int, stream=None, poison: bool = False):
        """Forward + backward with the KV residency policy of SURVEY §8(c):
        K_j, V_j of the hot prefix j < ``hot`` stay on the GPU (the most-accessed
        Type-0 tensors); every colder chunk is written back to pinned host
        memory after its forward (D2H overlapping fwd(j+1)) and streamed
        back in windows of ``window`` chunks through a 2-slot device ring for
        every later fwd(i) / bwd(i) (prefetch of window n+1 overlaps compute of
        window n).  Windows of one chunk are chained with FIRST/LAST (the online
        softmax carry, a2).  With ``poison`` the full-sequence device K/V of cold
        chunks are overwritten with NaN once offloaded, proving that only the
        streamed copies are read.  Returns copy statistics."""
        L = self.L
        N = L.num_chunks
        h, d = L.heads, L.head_dim
        strm = stream or torch.cuda.current_stream()
        smax = max(L.chunk_len(i) for i in range(N))
        key = ("ring", window, smax)
        if getattr(self, "_ring_key", None) != key:
            self._ring = torch.empty((2, window, 2, smax, h, d), dtype=self.o.dtype, device=self.device)
            self._ring_key = key
        ring = self._ring
        stats = {"d2h": 0, "h2d": 0, "windows": 0}
        off_done = {}

        def host_of(j):
            nb = L.chunk_len(j) * h * d * self.elem
            return self._host_buf(("k", j), nb), self._host_buf(("v", j), nb), nb

        # flat schedule of (kind, chunk, windows); a window is a list of (j, where)
        def windows_for(i, kind):
            hot_ids = [j for j in range(min(hot, i + 1))]
            if kind == "fwd":
                cold = [j for j in range(hot, i - 1)]           # i-1 and i still on device
                dev_ids = hot_ids + [j for j in (i - 1, i) if j >= hot and j >= 0]
            else:
                cold = [j for j in range(hot, i + 1)]
                dev_ids = hot_ids
            wins = [[(j, "dev") for j in dev_ids]] if dev_ids else []
            wins += [[(j, "ring") for j in cold[a:a + window]] for a in range(0, len(cold), window)]
            return wins

        sched = [("fwd", i, windows_for(i, "fwd")) for i in range(N)] + \
                [("bwd", i, windows_for(i, "bwd")) for i in range(N - 1, -1, -1)]
        ring_windows = [(si, wi) for si, (_, _, ws) in enumerate(sched) for wi, w in enumerate(ws) if w[0][1] == "ring"]
        ring_slot = {rw: n % 2 for n, rw in enumerate(ring_windows)}
        ready = {}

        offloaded = set(range(min(hot, N)))  # chunks whose host copy has been issued (hot ones never stream)

        def prefetch(n, must=False):
            if n >= len(ring_windows) or n in ready:
                return
            si, wi = ring_windows[n]
            if not all(j in offloaded for j, _ in sched[si][2][wi]):
                assert not must, "window streamed before its chunks were written back"
                return  # a chunk of this window has not been offloaded yet: issue later
            slot = n % 2
            evs = []
            for c, (j, _) in enumerate(sched[si][2][wi]):
                if j in off_done:
                    strm.wait_event(off_done.pop(j))  # its D2H must have landed before reading the host copy
                hk, hv, nb = host_of(j)
                for which, hp in ((0, hk), (1, hv)):
                    dst = ring[slot, c, which, :L.chunk_len(j)]
                    ev = torch.cuda.Event()
                    # ordered after the compute work enqueued so far (the ring slot's last reader)
                    self.ctx.kv_prefetch(j, hp, dst, nb, consumer=strm, done=ev, flags=sppo.SPPO_COPY_DEFER_WAIT)
                    stats["h2d"] += nb
                    evs.append(ev)
            ready[n] = evs

        self.dk_acc.zero_()
        self.dv_acc.zero_()
        n_ring = 0
        prefetch(0)
        for si, (kind, i, wins) in enumerate(sched):
            s = L.chunk_len(i)
            for wi, w in enumerate(wins):
                flags = (sppo.SPPO_FIRST if wi == 0 else 0) | (sppo.SPPO_LAST if wi == len(wins) - 1 else 0)
                ids = [j for j, _ in w]
                if w[0][1] == "ring":
                    prefetch(n_ring, must=True)  # no-op when already issued one window ahead
                    prefetch(n_ring + 1)  # next window's copy overlaps this window's compute
                    for ev in ready.pop(n_ring):
                        strm.wait_event(ev)
                    slot = n_ring % 2
                    ks = [ring[slot, c, 0, :L.chunk_len(j)] for c, j in enumerate(ids)]
                    vs = [ring[slot, c, 1, :L.chunk_len(j)] for c, j in enumerate(ids)]
                    n_ring += 1
                else:
                    ks = [self.rows(k, j) for j in ids]
                    vs = [self.rows(v, j) for j in ids]
                stats["windows"] += 1
                if kind == "fwd":
                    self.ctx.attn_fwd(L, i, self.rows(q, i), ids, ks, vs, flags=flags,
                                      state=None if len(wins) == 1 else (self.o_acc[:s], self.m[:s * h], self.l[:s * h]),
                                      o=self.rows(self.o, i), lse=self.lse_view(i), stream=strm)
                    self.launches += 1
                else:
                    has_i = i in ids
                    self.ctx.attn_bwd(L, i, self.rows(q, i), ids, ks, vs, self.rows(self.o, i), self.lse_view(i),
                                      self.rows(do, i), self.delta[:s * h], self.dq_acc[:s],
                                      [self.rows(self.dk_acc, j) for j in ids],
                                      [self.rows(self.dv_acc, j) for j in ids],
                                      dq=self.rows(self.dq, i), dk=self.rows(self.dk, i) if has_i else None,
                                      dv=self.rows(self.dv, i) if has_i else None, flags=flags, stream=strm)
                    self.launches += 1 + (flags & sppo.SPPO_FIRST != 0) + (flags & sppo.SPPO_LAST != 0)
            if kind == "fwd" and i >= hot:
                # write K_i, V_i back to the host arena (Type-0 demoted by the policy); overlaps fwd(i+1)
                hk, hv, nb = host_of(i)
                ev = torch.cuda.Event()
                stats["d2h"] += self.ctx.kv_offload(i, self.rows(k, i), hk, nb, 1.0, producer=strm)
                stats["d2h"] += self.ctx.kv_offload(i, self.rows(v, i), hv, nb, 1.0, producer=strm, done=ev)
                off_done[i] = ev
                offloaded.add(i)
                poison_ev = ev
            if poison and kind == "fwd" and i - 1 >= hot:
                # chunk i-1 has left the GPU for good (fwd(i+1) streams it): poison its device copy
                strm.wait_event(self._last_off_ev)
                self.rows(k, i - 1).view(torch.uint8).fill_(0xFF)
                self.rows(v, i - 1).view(torch.uint8).fill_(0xFF)
            if kind == "fwd" and i >= hot:
                self._last_off_ev = poison_ev
        return stats

    @_on_step_stream
    def step_kv_stream_grouped(self, q, k, v, do, hot: int, window: int, group: int = 2, stream=None,
                               poison: bool = False):
        """KV streaming (step_kv_stream's policy, L10) with the cold windows shared
        by ``group`` consecutive chunks: each streamed window of K_j, V_j is applied
        to the forwards of chunks i..i+G-1 (each with its own FIRST/LAST carry) or
        to the backwards of chunks i..i-G+1 (descending, so a chunk's final dK/dV
        is written after every later chunk's contribution) before the ring slot is
        refilled — the host->device KV volume drops by ~G.  Chunk j only ever sees
        ids <= j, so the results equal the ungrouped step up to fp32 accumulation
        order.  Trade-off: a group's chunks finish together (coarser sequence
        pipelining granularity).  Returns copy statistics."""
        L = self.L
        N = L.num_chunks
        h, d = L.heads, L.head_dim
        strm = stream or torch.cuda.current_stream()
        smax = max(L.chunk_len(i) for i in range(N))
        G = max(1, int(group))
        key = ("ring", window, smax)
        if getattr(self, "_ring_key", None) != key:
            self._ring = torch.empty((2, window, 2, smax, h, d), dtype=self.o.dtype, device=self.device)
            self._ring_key = key
        ring = self._ring
        gkey = ("grp", G, smax)
        if getattr(self, "_grp_key", None) != gkey:
            f32 = dict(dtype=torch.float32, device=self.device)
            self._grp = [dict(o_acc=torch.empty((smax, h, d), **f32), m=torch.empty((smax * h,), **f32),
                              l=torch.empty((smax * h,), **f32), delta=torch.empty((smax * h,), **f32),
                              dq_acc=torch.empty((smax, h, d), **f32)) for _ in range(G)]
            self._grp_key = gkey
        scr = self._grp
        stats = {"d2h": 0, "h2d": 0, "windows": 0, "group": G}
        off_done = {}

        def host_of(j):
            nb = L.chunk_len(j) * h * d * self.elem
            return self._host_buf(("k", j), nb), self._host_buf(("v", j), nb), nb

        # steps: (kind, chunks of the group in processing order, windows); a window = (ids, where)
        steps = []
        for a in range(0, N, G):
            C = list(range(a, min(N, a + G)))
            dev_ids = [j for j in range(min(hot, C[-1] + 1))] + [j for j in range(max(hot, a - 1), C[-1] + 1)]
            cold = list(range(hot, a - 1))
            wins = [(dev_ids, "dev")] + [(cold[x:x + window], "ring") for x in range(0, len(cold), window)]
            steps.append(("fwd", C, wins))
        for b in range(N - 1, -1, -G):
            C = list(range(b, max(-1, b - G), -1))
            dev_ids = list(range(min(hot, b + 1)))
            cold = list(range(hot, b + 1))
            wins = ([(dev_ids, "dev")] if dev_ids else []) + \
                [(cold[x:x + window], "ring") for x in range(0, len(cold), window)]
            steps.append(("bwd", C, wins))
        ring_windows = [(si, wi) for si, (_, _, ws) in enumerate(steps) for wi, w in enumerate(ws) if w[1] == "ring"]
        ready = {}
        offloaded = set(range(min(hot, N)))

        def prefetch(n, must=False):
            if n >= len(ring_windows) or n in ready:
                return
            si, wi = ring_windows[n]
            ids = steps[si][2][wi][0]
            if not all(j in offloaded for j in ids):
                assert not must, "window streamed before its chunks were written back"
                return
            slot = n % 2
            evs = []
            for c, j in enumerate(ids):
                if j in off_done:
                    strm.wait_event(off_done.pop(j))
                hk, hv, nb = host_of(j)
                for which, hp in ((0, hk), (1, hv)):
                    ev = torch.cuda.Event()
                    self.ctx.kv_prefetch(j, hp, ring[slot, c, which, :L.chunk_len(j)], nb, consumer=strm, done=ev,
                                         flags=sppo.SPPO_COPY_DEFER_WAIT)
                    stats["h2d"] += nb
                    evs.append(ev)
            ready[n] = evs

        self.dk_acc.zero_()
        self.dv_acc.zero_()
        n_ring = 0
        prefetch(0)
        for si, (kind, C, wins) in enumerate(steps):
            # per chunk: its windows restricted to ids <= chunk, for FIRST / LAST
            mine = {i: [wi for wi, (ids, _) in enumerate(wins) if any(j <= i for j in ids)] for i in C}
            for wi, (ids, where) in enumerate(wins):
                if where == "ring":
                    prefetch(n_ring, must=True)
                    prefetch(n_ring + 1)
                    for ev in ready.pop(n_ring):
                        strm.wait_event(ev)
                    slot = n_ring % 2
                    ks_all = [ring[slot, c, 0, :L.chunk_len(j)] for c, j in enumerate(ids)]
                    vs_all = [ring[slot, c, 1, :L.chunk_len(j)] for c, j in enumerate(ids)]
                    n_ring += 1
                else:
                    ks_all = [self.rows(k, j) for j in ids]
                    vs_all = [self.rows(v, j) for j in ids]
                stats["windows"] += 1
                # the group's forwards of one window are independent (own Q, carry and
                # outputs; shared K/V window): with few waves per launch they alternate
                # between two streams so one launch fills the other's last wave; the
                # side stream joins back before the window's ring slot is reused
                two = kind == "fwd" and len(C) > 1 and self._few_waves
                if two:
                    if self._side is None:
                        self._side = torch.cuda.Stream(device=self.device)
                    fork = torch.cuda.Event()
                    fork.record(strm)
                    self._side.wait_event(fork)
                for gi, i in enumerate(C):
                    sel = [c for c, j in enumerate(ids) if j <= i]
                    if not sel:
                        continue
                    my = mine[i]
                    flags = (sppo.SPPO_FIRST if wi == my[0] else 0) | (sppo.SPPO_LAST if wi == my[-1] else 0)
                    wids = [ids[c] for c in sel]
                    ks, vs = [ks_all[c] for c in sel], [vs_all[c] for c in sel]
                    s = L.chunk_len(i)
                    sc = scr[gi]
                    if kind == "fwd":
                        self.ctx.attn_fwd(L, i, self.rows(q, i), wids, ks, vs, flags=flags,
                                          state=None if len(my) == 1 else (sc["o_acc"][:s], sc["m"][:s * h], sc["l"][:s * h]),
                                          o=self.rows(self.o, i), lse=self.lse_view(i),
                                          stream=self._side if (two and gi % 2) else strm)
                        self.launches += 1
                    else:
                        has_i = i in wids
                        self.ctx.attn_bwd(L, i, self.rows(q, i), wids, ks, vs, self.rows(self.o, i), self.lse_view(i),
                                          self.rows(do, i), sc["delta"][:s * h], sc["dq_acc"][:s],
                                          [self.rows(self.dk_acc, j) for j in wids],
                                          [self.rows(self.dv_acc, j) for j in wids],
                                          dq=self.rows(self.dq, i), dk=self.rows(self.dk, i) if has_i else None,
                                          dv=self.rows(self.dv, i) if has_i else None, flags=flags, stream=strm)
                        self.launches += 1 + (flags & sppo.SPPO_FIRST != 0) + (flags & sppo.SPPO_LAST != 0)
                if two:
                    join = torch.cuda.Event()
                    join.record(self._side)
                    strm.wait_event(join)
            if kind == "fwd":
                last_ev = None
                for i in C:
                    if i < hot:
                        continue
                    hk, hv, nb = host_of(i)
                    ev = torch.cuda.Event()
                    stats["d2h"] += self.ctx.kv_offload(i, self.rows(k, i), hk, nb, 1.0, producer=strm)
                    stats["d2h"] += self.ctx.kv_offload(i, self.rows(v, i), hv, nb, 1.0, producer=strm, done=ev)
                    off_done[i] = ev
                    offloaded.add(i)
                    last_ev = ev
                if poison:
                    # chunks < C[-1] are never read from the device again (the next group's
                    # device window starts at C[-1]); poison those whose host copy is complete
                    for j in range(max(hot, C[0] - 1), C[-1]):
                        if j in off_done:
                            strm.wait_event(off_done[j])
                        self.rows(k, j).view(torch.uint8).fill_(0xFF)
                        self.rows(v, j).view(torch.uint8).fill_(0xFF)
        return stats

    # end-to-end step through host buffers --------------------------------------
    @_on_step_stream
    def step_host_io(self, host_in, host_out, dev_in, stream=None):
        """One step whose inputs start in pinned host memory and whose results end
        there: chunk-wise H2D of Q_i, K_i, V_i, dO_i (sppo_kv_prefetch, deferred
        wait) overlapped with compute, D2H of O_i after fwd(i) and of dQ_i, dK_i,
        dV_i after bwd(i) (sppo_kv_offload).  Returns (h2d_bytes, d2h_bytes,
        last_done_event)."""
        L = self.L
        N = L.num_chunks
        strm = stream or torch.cuda.current_stream()
        h2d = d2h = 0
        # Issue order = consumption order on the single H2D stream: Q,K,V chunk by
        # chunk for the forward, then dO from the last chunk down for the
        # backward (which runs N-1 .. 0), so no copy queues behind one needed later.
        ready = [[None] * 4 for _ in range(N)]
        order = [(i, j, name) for i in range(N) for j, name in enumerate(("q", "k", "v"))]
        order += [(i, 3, "do") for i in range(N - 1, -1, -1)]
        for i, j, name in order:
            t = self.rows(dev_in[name], i)
            nb = t.numel() * t.element_size()
            off = L.offsets[i] * L.heads * L.head_dim * self.elem
            ev = torch.cuda.Event()
            # ordered after the work already on `strm` (a previous step still reading the
            # device inputs); nothing of this step is enqueued yet, so the copies of this
            # step do not wait for each other's consumers
            self.ctx.kv_prefetch(i, host_in[name] + off, t, nb, consumer=strm, done=ev,
                                 flags=sppo.SPPO_COPY_DEFER_WAIT)
            h2d += nb
            ready[i][j] = ev
        self.dk_acc.zero_()
        self.dv_acc.zero_()
        # the device result rows of chunk i are rewritten only after the previous
        # call's D2H of those rows has completed (WAR on o / dq / dk / dv)
        prev = getattr(self, "_io_prev", {})
        self._io_prev = cur = {}
        last = None
        for i in range(N):
            for ev in ready[i][:3]:
                strm.wait_event(ev)
            if ("o", i) in prev:
                strm.wait_event(prev[("o", i)])
            self.forward_chunk(i, dev_in["q"], dev_in["k"], dev_in["v"], strm)
            t = self.rows(self.o, i)
            nb = t.numel() * t.element_size()
            off = L.offsets[i] * L.heads * L.head_dim * self.elem
            last = torch.cuda.Event()
            d2h += self.ctx.kv_offload(i, t, host_out["o"] + off, nb, 1.0, producer=strm, done=last)
            cur[("o", i)] = last
        for i in range(N - 1, -1, -1):
            strm.wait_event(ready[i][3])
            if ("g", i) in prev:
                strm.wait_event(prev[("g", i)])
            self.backward_chunk(i, dev_in["q"], dev_in["k"], dev_in["v"], dev_in["do"], strm)
            for name, t in (("dq", self.rows(self.dq, i)), ("dk", self.rows(self.dk, i)), ("dv", self.rows(self.dv, i))):
                nb = t.numel() * t.element_size()
                off = L.offsets[i] * L.heads * L.head_dim * self.elem
                last = torch.cuda.Event()
                d2h += self.ctx.kv_offload(i, t, host_out[name] + off, nb, 1.0, producer=strm, done=last)
            cur[("g", i)] = last  # the copies run in order on the D2H stream: the last covers all three
        return h2d, d2h, last

    def lse_heads_major(self):
        """[h, S] view assembled from per-chunk [h, s_i] blocks (for checks)."""
        parts = [self.lse_view(i).view(self.L.heads, -1) for i in range(self.L.num_chunks)]
        return torch.cat(parts, dim=1)
