"""Multiplexed sequence partitioning (MSP) execution across pipeline stages
(P:420-461 [§6.2, Definitions 1-2, Table P:386-404];
P:322 [§4]).

PP stages, one process (GPU) per stage, one transformer layer (or a list) per
stage, N subsequences (chunks).  In the plain subsequence pipeline
(pipeline.py) stage s is idle while the first chunks travel down the pipe and
again while the last ones drain.  MSP fills those bubbles: per Definition 1
(reading L18, sppo_msp_phases) stage s splits its chunks into

    Left   {0 .. PP-2-s}      run on the GPUs {s .. PP-1}  (Left-SP range)
    Steady {PP-1-s .. N-1-s}  run on GPU s alone (adaptive offloading)
    Right  {N-s .. N-1}       run on the GPUs {0 .. s}     (Right-SP range)

where "run on a range" means Megatron-style tensor/sequence parallelism of the
stage's layer over that range ("the traditional Megatron sequence
parallelism"; the heads — and the MLP columns — are split, the partial sums
all-reduced: engine_layer's tp mode), so a bubble-adjacent chunk finishes
|range| times sooner and later stages (Left) or earlier ones (Right) start or
finish that much earlier.

Reading L20: the backward, "similar yet asymmetric" and
otherwise unspecified, runs every (stage, chunk) on the SAME GPU range as its
forward.  Both bubbles line up: in the backward, stage s processes its Right
chunks first, while stages < s wait for its dx (so GPUs 0..s are free), and
its Left chunks last, after stages > s have finished (GPUs s..PP-1 free); and
every activation a range produced in the forward is still on that range —
nothing is re-partitioned for the backward except the K/V gradient
accumulators below.

K/V across phases.  Chunk i's attention needs K_j, V_j of every j <= i,
and dK_j, dV_j accumulate over every later chunk.  The layer state moves at
the four phase boundaries of stage s (owner = GPU s):
    forward  Left -> Steady : the owner gathers the Left chunks' K/V head
                              shards from the Left range            (gather)
             Steady -> Right: every member of the Right range gets its head
                              shard of K/V rows [0, c_{N-s})        (scatter)
    backward Right -> Steady: the Right range's dK/dV contributions to rows
                              [0, c_{N-s}) are added into the owner's
                              accumulators                          (reduce)
             Steady -> Left : the Left range gets its head shards of the
                              accumulated dK/dV rows [0, c_{PP-1-s}) (scatter)
Inter-stage activations (z rows forward, dx rows backward) travel from the
producing stage's owner to the members of the consuming range that did not
take part in producing them.

Execution order.  Every rank walks ONE global task list (same on all ranks)
and performs the tasks it takes part in; transfers are non-blocking sends and
blocking receives, group collectives run inside the tasks.  The earliest
unfinished task always has all its participants available, so the walk cannot
deadlock.  The list is ordered by a list-scheduling simulation of the plan
(cost of a task = its chunk's work / |range|), which is also the MSP makespan
model (`MSPPlan.makespan`).

Every arithmetic step runs in libsppo's kernels (engine_layer); this module
only builds the plan, moves rows between ranks and sequences the ABI calls.
Transfers: NCCL point-to-point on device tensors when the default group is
NCCL, host-staged over gloo otherwise (tests: several ranks sharing one GPU).
"""

from __future__ import annotations

import contextlib

import torch
import torch.distributed as dist

from . import engine_layer, sppo


# ============================================================================ plan
class MSPPlan:
    """The phase map of every stage, the GPU range of every (stage, chunk), and the
    global task order.  t_fwd[i] / t_bwd[i] = one GPU's time for chunk i of a
    stage (default: its attention pairs plus a per-token linear term, backward
    twice the forward)."""

    def __init__(self, PP: int, N: int, offsets, t_fwd=None, t_bwd=None, msp: bool = True):
        self.PP, self.N = PP, N
        self.offsets = [int(x) for x in offsets]
        self.msp = msp
        self.ph = [sppo.msp_phases(PP, N, s) for s in range(PP)]
        if t_fwd is None:
            c = self.offsets
            t_fwd = [(c[i + 1] * (c[i + 1] + 1) - c[i] * (c[i] + 1)) / 2 + 4096.0 * (c[i + 1] - c[i])
                     for i in range(N)]
        # a list (one GPU's time per chunk; a range of g GPUs takes 1/g of it) or a
        # dict {g: list} of per-chunk times measured for a g-way tensor-parallel shard
        norm = lambda t: {int(g): [float(w) for w in v] for g, v in t.items()} if isinstance(t, dict) else [
            float(w) for w in t]
        self.t_fwd = norm(t_fwd)
        if t_bwd is None:
            t_bwd = ({g: [2.0 * w for w in v] for g, v in self.t_fwd.items()} if isinstance(self.t_fwd, dict)
                     else [2.0 * w for w in self.t_fwd])
        self.t_bwd = norm(t_bwd)
        self.tasks = self._order()

    # ---- phase queries
    def kind(self, s: int, i: int) -> str:
        if not self.msp:
            return "steady"
        p = self.ph[s]
        return "left" if i in p["left"] else ("right" if i in p["right"] else "steady")

    def group(self, s: int, i: int):
        k = self.kind(s, i)
        return tuple(self.ph[s]["left_sp"]) if k == "left" else (
            tuple(self.ph[s]["right_sp"]) if k == "right" else (s,))

    def n_left(self, s: int) -> int:
        return len(self.ph[s]["left"]) if self.msp else 0

    def first_right(self, s: int) -> int:
        return self.N - len(self.ph[s]["right"]) if self.msp else self.N

    # ---- tasks: (kind, stage, chunk); participants; cost
    def participants(self, task):
        kind, s, i = task
        PP = self.PP
        if kind in ("F", "B"):
            g = set(self.group(s, i))
            src = s - 1 if kind == "F" else s + 1
            if 0 <= src < PP:
                g.add(src)
            return tuple(sorted(g))
        if kind in ("LS", "SL"):
            return tuple(self.ph[s]["left_sp"])
        if kind in ("SR", "RS"):
            return tuple(self.ph[s]["right_sp"])
        if kind == "G":  # final gradient / output assembly of stage s
            return tuple(sorted(set(self.ph[s]["left_sp"]) | set(self.ph[s]["right_sp"]) | {s}))
        raise ValueError(kind)

    def _deps(self):
        """Dependency edges of the task graph (predecessors per task)."""
        PP, N = self.PP, self.N
        deps = {}
        for s in range(PP):
            nL, fR = self.n_left(s), self.first_right(s)
            for i in range(N):
                d = []
                if s > 0:
                    d.append(("F", s - 1, i))
                if i > 0:
                    d.append(("F", s, i - 1))
                if self.msp and nL > 0 and i == nL:
                    d.append(("LS", s, -1))
                if self.msp and fR < N and i == fR:
                    d.append(("SR", s, -1))
                deps[("F", s, i)] = d
            if self.msp and nL > 0:
                deps[("LS", s, -1)] = [("F", s, nL - 1)]
            if self.msp and fR < N:
                deps[("SR", s, -1)] = [("F", s, fR - 1)]
            for i in range(N - 1, -1, -1):
                d = [("F", s, N - 1)] if i == N - 1 else [("B", s, i + 1)]
                if s < PP - 1:
                    d.append(("B", s + 1, i))
                if self.msp and fR < N and i == fR - 1:
                    d.append(("RS", s, -1))
                if self.msp and nL > 0 and i == nL - 1:
                    d.append(("SL", s, -1))
                deps[("B", s, i)] = d
            if self.msp and fR < N:
                deps[("RS", s, -1)] = [("B", s, fR)]
            if self.msp and nL > 0:
                deps[("SL", s, -1)] = [("B", s, nL)]
            deps[("G", s, -1)] = [("B", s, 0)]
        return deps

    def cost(self, task) -> float:
        """A chunk on a range of g GPUs takes its measured g-way shard time, or 1/g
        of its one-GPU time (perfect split); the range's all-reduces and the
        phase-boundary moves are not modeled (cost 0)."""
        kind, s, i = task
        if kind not in ("F", "B"):
            return 0.0
        tab, g = (self.t_fwd if kind == "F" else self.t_bwd), len(self.group(s, i))
        return tab[g][i] if isinstance(tab, dict) else tab[i] / g

    def busy(self, task):
        """Ranks a task occupies in the schedule model: the range computing it (the
        producing stage's owner only sends, non-blocking)."""
        return self.group(task[1], task[2]) if task[0] in ("F", "B") else self.participants(task)

    def _order(self):
        """List scheduling of the task graph: repeatedly take the ready task of
        highest priority and start it as early as its predecessors and the ranks it
        occupies allow.  Three priority rules are tried — critical path (longest
        remaining path to the end), earliest feasible start, and pipeline order
        (forward: lower stage first; backward: higher stage first) — and the
        schedule with the smallest makespan is kept (deterministic: every rank
        computes the same one).  The walk order is the tasks sorted by start
        (scheduling sequence for ties, which respects every dependency)."""
        deps = self._deps()
        succ = {t: [] for t in deps}
        for t, d in deps.items():
            for u in d:
                succ[u].append(t)
        indeg0 = {t: len(d) for t, d in deps.items()}
        # bottom levels (longest path to exit, including the task itself)
        topo, stack, cnt = [], [t for t, n in indeg0.items() if n == 0], dict(indeg0)
        while stack:
            t = stack.pop()
            topo.append(t)
            for u in succ[t]:
                cnt[u] -= 1
                if cnt[u] == 0:
                    stack.append(u)
        assert len(topo) == len(deps), "task graph has a cycle"
        level = {}
        for t in reversed(topo):
            level[t] = self.cost(t) + max([level[u] for u in succ[t]] + [0.0])
        kind_rank = lambda u: "FLSRBSLRSG".find(u[0])  # noqa: E731

        def schedule(rule):
            indeg = dict(indeg0)
            end, free, start, seq = {}, [0.0] * self.PP, {}, []
            ready = [t for t, n in indeg.items() if n == 0]

            def est(u):
                return max([end[v] for v in deps[u]] + [free[r] for r in self.busy(u)] + [0.0])
            while ready:
                if rule == "critical":
                    t = max(ready, key=lambda u: (level[u], -u[1] if u[0] == "F" else u[1], -kind_rank(u), -u[2]))
                elif rule == "earliest":
                    t = min(ready, key=lambda u: (est(u), -level[u], kind_rank(u), u[1], u[2]))
                else:  # pipeline order
                    t = min(ready, key=lambda u: (0 if u[0] in ("F", "LS", "SR") else 1,
                                                  u[1] if u[0] in ("F", "LS", "SR") else -u[1],
                                                  u[2] if u[0] in ("F", "LS", "SR") else -u[2], kind_rank(u)))
                ready.remove(t)
                st = est(t)
                start[t], end[t] = st, st + self.cost(t)
                for r in self.busy(t):
                    free[r] = end[t]
                seq.append(t)
                for u in succ[t]:
                    indeg[u] -= 1
                    if indeg[u] == 0:
                        ready.append(u)
            return max(end.values()), start, end, seq

        best = None
        for rule in ("critical", "earliest", "pipeline"):
            res = schedule(rule)
            if best is None or res[0] < best[0] - 1e-12:
                best = res + (rule,)
        _, self.start, self.end, seq, self.rule = best
        pos = {t: n for n, t in enumerate(seq)}
        return sorted(seq, key=lambda t: (self.start[t], pos[t]))

    @property
    def makespan(self) -> float:
        return max(self.end.values())


def msp_makespan(PP: int, N: int, offsets, t_fwd, t_bwd, msp: bool = True) -> float:
    """Makespan of one fwd+bwd pass from per-chunk times of ONE GPU's full-stage
    work (any unit), under the MSP plan (msp=True) or the plain subsequence
    pipeline (msp=False)."""
    return MSPPlan(PP, N, offsets, t_fwd=t_fwd, t_bwd=t_bwd, msp=msp).makespan


# ============================================================================ execution
class _Xfer:
    """Point-to-point rows between global ranks: NCCL on device tensors, or
    host-staged over gloo."""

    def __init__(self):
        self.nccl = dist.get_backend() == "nccl"
        self.pending = []

    def send(self, t, dst):
        if self.nccl:
            self.pending.append((dist.isend(t.contiguous(), dst), t))
        else:
            h = t.detach().to("cpu", copy=True).contiguous()
            self.pending.append((dist.isend(h, dst), h))

    def recv(self, shape, dtype, device, src):
        if self.nccl:
            t = torch.empty(shape, dtype=dtype, device=device)
            dist.recv(t, src)
            return t
        h = torch.empty(shape, dtype=dtype)
        dist.recv(h, src)
        return h.to(device)

    def flush(self):
        for w, _ in self.pending:
            w.wait()
        self.pending.clear()


class MSPExecutor:
    """This rank's part of an MSP pipeline of PP single-layer stages.

    `stage_params[s]` is stage s's full parameter dict (any device; every rank
    gets all of them and keeps only what its ranges need: the full layer of its
    own stage, tensor-parallel shards of the stages whose Left/Right ranges
    include it).  `msp=False` runs the plain subsequence pipeline through the
    same machinery (every chunk on its stage's own GPU)."""

    def __init__(self, ctx: sppo.Context, rank: int, PP: int, hidden: int, heads: int, offsets, stage_params,
                 device="cuda", msp: bool = True, t_fwd=None, t_bwd=None, make_layer=None, shard=None,
                 unshard=None):
        """make_layer(params, tp) / shard(params, j, g) / unshard(shards) default to
        engine_layer.ChunkedLayer / shard_params / unshard_params (other layer
        objects with the same interface are accepted: host-logic tests)."""
        assert dist.is_initialized() and dist.get_world_size() == PP
        self.ctx, self.rank, self.PP = ctx, rank, PP
        off_ = [int(x) for x in offsets]
        self.make_layer = make_layer or (lambda prm, tp: engine_layer.ChunkedLayer(
            ctx, hidden, heads, off_, prm, tp=tp))
        self.shard = shard or (lambda prm, j, g: engine_layer.shard_params(prm, hidden, heads, j, g))
        self.unshard = unshard or (lambda shards: unshard_params(shards, hidden, heads))
        self.H, self.heads = hidden, heads
        self.plan = MSPPlan(PP, len(offsets) - 1, offsets, t_fwd=t_fwd, t_bwd=t_bwd, msp=msp)
        self.N = self.plan.N
        self.S = self.plan.offsets[-1]
        self.device = torch.device(device)
        self.xf = _Xfer()
        # process groups of every SP range (created by all ranks, same order)
        self.pg = {}
        for s in range(PP):
            for key in ("left_sp", "right_sp"):
                rg = tuple(self.plan.ph[s][key])
                if msp and len(rg) > 1 and rg not in self.pg:
                    self.pg[rg] = dist.new_group(list(rg))
        # layer instances: (stage, kind) -> ChunkedLayer; kind in full / left / right
        self.inst = {}
        for s in range(PP):
            p = stage_params[s]
            if rank == s:
                self.inst[(s, "steady")] = self.make_layer({k: v.to(self.device) for k, v in p.items()}, None)
            for kind, key in (("left", "left_sp"), ("right", "right_sp")):
                rg = tuple(self.plan.ph[s][key])
                if msp and rank in rg and len(rg) > 0 and self._has(s, kind):
                    j = rg.index(rank)
                    sh = self.shard(p, j, len(rg))
                    self.inst[(s, kind)] = self.make_layer({k: v.to(self.device) for k, v in sh.items()},
                                                           (j, len(rg), self.pg[rg]))
        some = next(iter(self.inst.values()))
        bf = dict(dtype=some.z.dtype, device=self.device)
        # per-stage input rows (forward x, backward dz) for the stages this rank computes
        self.X = {s: torch.zeros((self.S, hidden), **bf) for s in range(PP) if self._computes(s)}
        self.DZ = {s: torch.zeros((self.S, hidden), **bf) for s in range(PP) if self._computes(s)}
        self.log = []

    def _has(self, s, kind):
        ph = self.plan.ph[s]
        return bool(ph["left"]) if kind == "left" else bool(ph["right"])

    def _computes(self, s):
        return any(k[0] == s for k in self.inst)

    def layer(self, s, i):
        return self.inst[(s, self.plan.kind(s, i))]

    def rows(self, t, i):
        c = self.plan.offsets
        return t[c[i]:c[i + 1]]

    def _col(self, s, kind, j):
        """Hidden-column slice of member j's heads in the range of (s, kind)."""
        rg = self.plan.ph[s]["left_sp" if kind == "left" else "right_sp"]
        w = self.H // len(rg)
        return slice(j * w, (j + 1) * w)

    # ------------------------------------------------------------------ one step
    def step(self, x, dz, stream=None):
        """Forward of every stage over chunks 0..N-1 and backward over N-1..0 under
        the MSP plan.  x: model input [S, H] (used by stage 0's ranges), dz: the
        upstream gradient of the last stage's output (used by stage PP-1's).
        Returns, for the stage this rank owns: dict(x, z, dz, dx, grads) with
        every chunk's rows assembled on the owner."""
        cuda = self.device.type == "cuda"
        strm = stream or (torch.cuda.current_stream() if cuda else None)
        for lay in self.inst.values():
            lay._zero()
        with (torch.cuda.stream(strm) if cuda else contextlib.nullcontext()):
            for task in self.plan.tasks:
                if self.rank in self.plan.participants(task):
                    getattr(self, "_t_" + task[0])(task, x, dz, strm)
                    self.log.append(task)
            self.xf.flush()
        return self.result

    # ---- forward / backward of one chunk on its range
    def _route(self, s, i, src_stage, get_rows, bufs):
        """Rows of chunk i produced by stage `src_stage` (its range G') into this
        rank's `buf` rows for stage s (range G): members of G ∩ G' copy their own
        rows, the others receive them from the producing stage's owner."""
        G = self.plan.group(s, i)
        Gp = self.plan.group(src_stage, i)
        r = self.rank
        if r == src_stage:
            for m in G:
                if m not in Gp:
                    self.xf.send(get_rows(src_stage, i), m)
        if r in G:
            buf = bufs[s]
            if r in Gp:
                self.rows(buf, i).copy_(get_rows(src_stage, i))
            else:
                t = self.xf.recv(self.rows(buf, i).shape, buf.dtype, self.device, src_stage)
                self.rows(buf, i).copy_(t)

    def _t_F(self, task, x, dz, strm):
        _, s, i = task
        if s > 0:
            self._route(s, i, s - 1, lambda st, ii: self.rows(self.layer(st, ii).z, ii), self.X)
        elif self.rank in self.plan.group(s, i):
            self.rows(self.X[0], i).copy_(self.rows(x, i))
        if self.rank in self.plan.group(s, i):
            self.layer(s, i).forward_chunk(i, self.X[s], strm)

    def _t_B(self, task, x, dz, strm):
        _, s, i = task
        if s < self.PP - 1:
            self._route(s, i, s + 1, lambda st, ii: self.rows(self.layer(st, ii).dx, ii), self.DZ)
        elif self.rank in self.plan.group(s, i):
            self.rows(self.DZ[s], i).copy_(self.rows(dz, i))
        if self.rank in self.plan.group(s, i):
            self.layer(s, i).backward_chunk(i, self.X[s], self.DZ[s], strm)

    # ---- phase boundaries
    def _gather_cols(self, s, kind, rows, names, add):
        """Owner <- members: each member's `names` tensors (rows [0, rows)) into the
        owner's steady instance at the member's hidden columns (copy or +=)."""
        rg = self.plan.ph[s]["left_sp" if kind == "left" else "right_sp"]
        own, part = self.inst.get((s, "steady")), self.inst[(s, kind)]
        if self.rank != s:
            for n in names:
                self.xf.send(getattr(part, n)[:rows], s)
            return
        for j, m in enumerate(rg):
            for n in names:
                src = getattr(part, n)[:rows] if m == s else self.xf.recv(
                    (rows, getattr(part, n).shape[1]), getattr(part, n).dtype, self.device, m)
                dst = getattr(own, n)[:rows, self._col(s, kind, j)]
                if add:
                    dst.add_(src)
                else:
                    dst.copy_(src)

    def _scatter_cols(self, s, kind, rows, names):
        """Owner -> members: the owner's `names` rows [0, rows) at member j's hidden
        columns into member j's instance of (s, kind)."""
        rg = self.plan.ph[s]["left_sp" if kind == "left" else "right_sp"]
        part = self.inst[(s, kind)]
        if self.rank == s:
            own = self.inst[(s, "steady")]
            for j, m in enumerate(rg):
                for n in names:
                    sl = getattr(own, n)[:rows, self._col(s, kind, j)]
                    if m == s:
                        getattr(part, n)[:rows].copy_(sl)
                    else:
                        self.xf.send(sl.contiguous(), m)
        else:
            for n in names:
                t = getattr(part, n)
                t[:rows].copy_(self.xf.recv((rows, t.shape[1]), t.dtype, self.device, s))

    def _t_LS(self, task, x, dz, strm):
        s = task[1]
        self._gather_cols(s, "left", self.plan.offsets[self.plan.n_left(s)], ("k", "v"), add=False)

    def _t_SR(self, task, x, dz, strm):
        s = task[1]
        self._scatter_cols(s, "right", self.plan.offsets[self.plan.first_right(s)], ("k", "v"))

    def _t_RS(self, task, x, dz, strm):
        s = task[1]
        self._gather_cols(s, "right", self.plan.offsets[self.plan.first_right(s)], ("dk_acc", "dv_acc"), add=True)

    def _t_SL(self, task, x, dz, strm):
        s = task[1]
        self._scatter_cols(s, "left", self.plan.offsets[self.plan.n_left(s)], ("dk_acc", "dv_acc"))

    # ---- final assembly on the owner: outputs of every chunk and the stage's gradients
    def _t_G(self, task, x, dz, strm):
        s = task[1]
        if self.rank == s:
            own = self.inst[(s, "steady")]
            z, dx = torch.empty_like(own.z), torch.empty_like(own.dx)
            for i in range(self.N):
                lay = self.layer(s, i)
                self.rows(z, i).copy_(self.rows(lay.z, i))
                self.rows(dx, i).copy_(self.rows(lay.dx, i))
            grads = {k: v.clone() for k, v in own.grads.items()}
        for kind in ("left", "right"):
            if not (self.plan.msp and self._has(s, kind)):
                continue
            rg = self.plan.ph[s]["left_sp" if kind == "left" else "right_sp"]
            if self.rank not in rg:
                continue
            part = self.inst[(s, kind)]
            names = sorted(part.grads)
            if self.rank != s:
                for k in names:
                    self.xf.send(part.grads[k], s)
                continue
            shards = []
            for m in rg:
                shards.append({k: (part.grads[k] if m == self.rank else self.xf.recv(
                    tuple(part.grads[k].shape), part.grads[k].dtype, self.device, m)) for k in names})
            full = self.unshard(shards)
            for k in grads:
                grads[k] += full[k]
        if self.rank == s:
            self.result = dict(x=self.X[s], z=z, dz=self.DZ[s], dx=dx, grads=grads)

    result = None


def unshard_params(shards, hidden: int, heads: int) -> dict:
    """Inverse of engine_layer.shard_params for gradient shards: column/row-parallel
    parts concatenated in rank order; replicated parameters (LayerNorms, b_o, b_2)
    are identical on every rank (their inputs are all-reduced), rank 0's is taken."""
    size = len(shards)
    H, Hl = hidden, hidden // size
    out = dict(shards[0])
    q = [torch.cat([sh[name][k * Hl:(k + 1) * Hl] for sh in shards]) for name in ("w_qkv",) for k in range(3)]
    out["w_qkv"] = torch.cat(q)
    out["b_qkv"] = torch.cat([torch.cat([sh["b_qkv"][k * Hl:(k + 1) * Hl] for sh in shards]) for k in range(3)])
    out["w_o"] = torch.cat([sh["w_o"] for sh in shards], dim=1)
    out["w_1"] = torch.cat([sh["w_1"] for sh in shards])
    out["b_1"] = torch.cat([sh["b_1"] for sh in shards])
    out["w_2"] = torch.cat([sh["w_2"] for sh in shards], dim=1)
    return out
