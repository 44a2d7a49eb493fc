"""Benchmark of the SPPO hot path on B200: chunked causal attention fwd+bwd.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One step = one pass of the whole hot path over one synthetic batch: partition
(a0) -> forward of chunks 0..N-1 (a1) -> backward of chunks N-1..0 (a5-a7),
all through the C ABI (libsppo.so).  Workload at N=1: configs[1] (C2, GPT-7B
attention layer: h=32, d=128, S=128K, 16 chunks).  For N>1 (torchrun) the
heads are sharded over the ranks (Ulysses-style head parallelism without the
all-to-all); no collective inside the step; one NCCL all-gather
of O after timing (not timed).  Rank 0 prints one JSON line.

Besides the resident step the line carries: the end-to-end step from/to pinned
host memory (e2e), the Type-1 alpha offload policy (exposed %, split by phase),
optionally KV streaming (--kv-hot / --device-budget, --kv-group G: windows
shared by G chunks), the bwd kernel's roofline object and the oracle's CPU
baseline.  Other modes: --parallel cp (sequence ring,
paper_2503_10377_b200/cp.py), --shard-of G (rank 0's share of a G-GPU head split
on one GPU), --partition balanced | layer-balanced, --impl reference (the
oracle), --workload layer (the full GPT layer per chunk, with
--layer-pool for activation offload that frees device memory and
--layer-streams 2; its line reports the layer GEMMs' roofline, the Type-1
offload exposure for sequence-aware vs fixed alpha, and a PP pipeline model).

FLOP convention: 4d per causal pair forward, 10d backward.
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

CONFIGS = {
    "C1": dict(heads=1, d=64, S=1024, N=4, dtype="fp32",
               workload="configs[0] tiny: 1 head, d=64, S=1024, N=4, fp32"),
    "C2": dict(heads=32, d=128, S=131072, N=16, dtype="bf16",
               workload="configs[1] GPT-7B attention layer: 32 heads, d=128, S=128K, N=16, bf16"),
    "C3": dict(heads=32, d=128, S=1048576, N=64, dtype="bf16",
               workload="configs[2] GPT-7B shape: 32 heads, d=128, S=1M, N=64, bf16"),
    "C4": dict(heads=40, d=128, S=524288, N=32, dtype="bf16",
               workload="configs[3] GPT-13B shape: 40 heads, d=128, S=512K, N=32, bf16"),
    "C5": dict(heads=64, d=128, S=4194304, N=256, dtype="bf16",
               workload="configs[4] GPT-65B shape: 64 heads, d=128, S=4M, N=256, bf16"),
}
METRIC = "chunked attn fwd+bwd TFLOP/s per B200 (% BF16 peak), tokens/s at 1/2/4/8 GPU"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(burst=d.get("bf16_tflops", 1590.0), sustained=d.get("bf16_tflops_sustained", 1400.0),
                    hbm=d.get("hbm_gbs", 6650.0), source="MEASURED_PEAKS.json (measured)")
    return dict(burst=1590.0, sustained=1400.0, hbm=6650.0, source="B200_PROFILING.md fallback")


def ncu_traffic(kernel):
    """DRAM bytes (read + write) per launch of `kernel` from the committed ncu
    --set full capture (profiles/r02/ncu_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "r02", "ncu_traffic.json")
    try:
        d = json.load(open(p))[kernel]
        return {"bytes": d["dram_read_bytes"] + d["dram_write_bytes"], "launch": d["launch"],
                "source": "profiles/r02/ncu_traffic.json (ncu --set full, one launch)"}
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) > 8 and r[1].strip().replace(".", "").isdigit()]
        if not sm:
            return None
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for n, v in zip(names, r[5:9]):
                if v.strip() == "Active":
                    reasons.add(n)
        load = [s for s in sm if s > 500] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": float(rows[0][2]), "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(float(r[3]) for r in rows if r[3].strip()[:1].isdigit())}


CLOCK_REJECT = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}


def flops_of(offsets, heads, d, part="fwd+bwd"):
    from paper_2503_10377_b200 import sppo
    pairs = sppo.causal_pairs(offsets)  # product's own host helper (a0 / FLOP accounting)
    per = {"fwd": 4, "bwd": 10, "fwd+bwd": 14}[part] * d
    return heads * per * pairs


# ------------------------------------------------------------------ CPU baseline (oracle)
def cpu_oracle_sample(seconds_target=12.0):
    """The fp64 oracle as it stands, on a bounded sample of the C2 workload: one
    head, the first S_s tokens as 2 chunks of C2's 8192-token chunk length.
    Returns dict(value TFLOP/s, cores, sample, seconds)."""
    import numpy as np

    import oracle
    from synth import make_inputs
    try:
        from threadpoolctl import threadpool_info
        cores = max([t.get("num_threads", 1) for t in threadpool_info()] or [1])
    except Exception:
        cores = os.cpu_count()
    S_s, N_s = 16384, 2
    x = make_inputs(S_s, [0], 128, seed=0, dtype=torch.bfloat16)
    xn = {k: v.double().numpy() for k, v in x.items()}
    off = [0, 8192, 16384]
    t0 = time.perf_counter()
    o, lse = oracle.chunked_attention_fwd(xn["q"], xn["k"], xn["v"], off)
    oracle.chunked_attention_bwd(xn["q"], xn["k"], xn["v"], o, lse, xn["do"], off)
    dt = time.perf_counter() - t0
    fl = 14 * 128 * (S_s * (S_s + 1) // 2)
    model = platform.processor()
    try:
        model = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name"))
    except (OSError, StopIteration):
        pass
    return dict(value=fl / dt / 1e12, cores=int(cores), seconds=dt, cpu_model=model,
                sample=f"oracle fp64 chunked fwd+bwd, 1 head x {S_s} tokens in {N_s} chunks of 8192 (C2 chunk length), "
                       f"{fl:.3e} FLOP in {dt:.1f}s")


# ------------------------------------------------------------------ distributed
def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test-only overrides: run several ranks on one GPU (SPPO_BENCH_DEVICE=0) over gloo
    # (SPPO_DIST_BACKEND=gloo) to exercise the multi-rank path where only one GPU exists
    if "SPPO_BENCH_DEVICE" in os.environ:
        local = int(os.environ["SPPO_BENCH_DEVICE"])
    if ws > 1:
        import torch.distributed as dist
        backend = os.environ.get("SPPO_DIST_BACKEND", "nccl" if torch.cuda.is_available() else "gloo")
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return ws, rank, local


def bind_numa(local):
    """P:472 [§7] "bind the NUMA node": pin this rank's host threads to the CPUs of
    its GPU's NUMA node (sysfs), so the offload copies' host side and the pinned
    arena (sppo_host_alloc, NUMA-local) sit on the same socket.  Returns a dict
    for the JSON line."""
    if not torch.cuda.is_available():
        return None
    try:
        p = torch.cuda.get_device_properties(local)
        bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        node = int(open(f"/sys/bus/pci/devices/{bus}/numa_node").read().strip())
    except Exception as e:
        return {"node": None, "note": f"NUMA node unknown ({type(e).__name__})"}
    if node < 0:
        return {"node": node, "note": "GPU reports no NUMA affinity (single-node host)"}
    try:
        cpus = set()
        for part in open(f"/sys/devices/system/node/node{node}/cpulist").read().strip().split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        cpus &= os.sched_getaffinity(0) or cpus
        if cpus:
            os.sched_setaffinity(0, cpus)
        return {"node": node, "cpus": len(cpus)}
    except Exception as e:
        return {"node": node, "note": f"affinity not set ({type(e).__name__})"}


def head_range(heads, ws, rank):
    from paper_2503_10377_b200.dist import head_range as hr
    return hr(heads, ws, rank)


def max_over_ranks(x, ws):
    from paper_2503_10377_b200.dist import max_over_ranks as mx
    return mx(x, ws, device="cuda" if torch.cuda.is_available() else "cpu")


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


# ------------------------------------------------------------------ our implementation
def run_ours(args, cfg, ws, rank, local):
    from paper_2503_10377_b200 import engine, sppo
    from synth import make_tensor

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    # --shard-of G: run rank 0's share of a G-GPU head split on this one GPU (per-GPU
    # measurement of a config that needs G GPUs; value is then per GPU, not aggregate)
    shard = args.shard_of if ws == 1 else ws
    heads = head_range(cfg["heads"], shard, rank)
    h, d, S, N = len(heads), cfg["d"], cfg["S"], cfg["N"]
    dtype = sppo.SPPO_BF16 if cfg["dtype"] == "bf16" else sppo.SPPO_FP32
    tdt = torch.bfloat16 if dtype == sppo.SPPO_BF16 else torch.float32
    ctx = sppo.Context(local)
    # a0, in the product's C helpers: equal (configs) or FLOPs-balanced
    offsets = sppo.partition_balanced(S, N) if args.partition == "balanced" else sppo.partition_equal(S, N)
    L = sppo.Layout(h, d, offsets, dtype=dtype)
    x = {t: make_tensor(t, S, heads, d, seed=0, dtype=tdt, device=dev) for t in ("q", "k", "v", "do")}
    eng = engine.ChunkedAttention(ctx, L, device=dev, timing=True, fwd_streams=args.fwd_streams)
    stream = torch.cuda.current_stream()

    for _ in range(args.warmup):
        eng.step(x["q"], x["k"], x["v"], x["do"], stream)
    torch.cuda.synchronize()
    eng.events = {"fwd": [], "bwd": []}
    eng.timing = False  # per-call events are not used for the timed steps (phase marks are)
    remeasured = None
    for attempt in range(2):
        phase = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        eng.launches = 0
        barrier(ws)
        torch.cuda.synchronize()
        clk = ClockSampler(local)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        t0.record(stream)
        for st in range(args.steps):
            marks[st].record(stream)  # step start; eng.step records the fwd/bwd boundary in phase[st]
            eng.step(x["q"], x["k"], x["v"], x["do"], stream, mark=phase[st])
        marks[args.steps].record(stream)
        t1.record(stream)
        torch.cuda.synchronize()
        clocks = clk.stop()
        barrier(ws)
        # timing rules: a run that saw a hardware / thermal slowdown is re-measured once
        bad = sorted(set((clocks or {}).get("reasons", [])) & CLOCK_REJECT)
        if not bad or attempt == 1:
            break
        remeasured = {"first_attempt_reasons": bad, "first_attempt_ms_per_step": t0.elapsed_time(t1) / args.steps}
    if clocks is not None and remeasured is not None:
        clocks["remeasured"] = remeasured
    ms_local = t0.elapsed_time(t1) / args.steps
    ms = max_over_ranks(ms_local, ws)
    launches = eng.launches // args.steps
    # phase times: forward = step start -> boundary (the two forward streams overlap, so
    # per-call events would double count), backward = boundary -> next step start
    fwd_ms = sum(marks[st].elapsed_time(phase[st]) for st in range(args.steps)) / args.steps
    bwd_ms = sum(phase[st].elapsed_time(marks[st + 1]) for st in range(args.steps)) / args.steps

    fl_dev = flops_of(offsets, h, d)
    fl_total = flops_of(offsets, cfg["heads"] if args.shard_of == 1 else len(heads), d)
    peaks = load_peaks()
    tflops = fl_total / (ms * 1e-3) / 1e12
    per_gpu = tflops / ws
    bwd_fl = flops_of(offsets, h, d, "bwd")
    fwd_fl = flops_of(offsets, h, d, "fwd")
    ach_bwd = bwd_fl / (bwd_ms * 1e-3) / 1e12
    ach_fwd = fwd_fl / (fwd_ms * 1e-3) / 1e12

    # ---- end to end through host buffers (pinned), same metric
    e2e = None
    if not args.no_e2e:
        nb = S * h * d * eng.elem
        host_in = {t: ctx.host_alloc(nb) for t in ("q", "k", "v", "do")}
        host_out = {t: ctx.host_alloc(nb) for t in ("o", "dq", "dk", "dv")}
        for t in ("q", "k", "v", "do"):  # stage the synthetic inputs in host memory once (outside timing)
            ctx.kv_offload(0, x[t], host_in[t], nb, 1.0, producer=stream)
        ctx.sync()
        res = []
        for rep in range(1 + max(1, args.steps // 2)):
            torch.cuda.synchronize()
            barrier(ws)
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            h2d, d2h, last = eng.step_host_io(host_in, host_out, x, stream)
            # end of step = the last D2H of a result has landed in host memory
            e1 = torch.cuda.Event(enable_timing=True)
            stream.wait_event(last)
            e1.record(stream)
            torch.cuda.synchronize()
            if rep > 0:  # first rep is a warm-up
                res.append(e0.elapsed_time(e1))
        e2e_ms = max_over_ranks(statistics.median(res), ws)
        e2e = {"value": round(fl_total / (e2e_ms * 1e-3) / 1e12, 2), "unit": "TFLOP/s",
               "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": h2d * ws, "d2h_bytes_per_step": d2h * ws,
               "path": "pinned host Q,K,V,dO -> chunk-wise sppo_kv_prefetch overlapped with compute; "
                       "O, dQ, dK, dV -> sppo_kv_offload after each chunk"}
        for p in list(host_in.values()) + list(host_out.values()):
            ctx.host_free(p)

    # ---- Type-1 offload policy (alpha) : exposed offload time vs resident
    offload = None
    if not args.no_offload:
        bw = 56e9  # pinned D2H GB/s measured on this pool (tools/box_probe.py, gpurun_out/box_probe.json)
        eng.events = {"fwd": [], "bwd": []}
        fs_default = eng.fwd_streams
        eng.timing, eng.fwd_streams = True, 1  # per-chunk forward times, one stream
        eng.step(x["q"], x["k"], x["v"], x["do"], stream)
        torch.cuda.synchronize()
        eng.fwd_streams = fs_default
        t_fwd = [a.elapsed_time(b) * 1e-3 for a, b in eng.events["fwd"]]
        A = [eng.type1_bytes(i) for i in range(N)]
        thr = [bw * (t_fwd[i + 1] if i + 1 < N else 0.0) for i in range(N)]
        alpha = sppo.offload_alpha(A, thr, 0.0)  # sequence-aware (reading L9)
        eng.timing = False

        def time_offload(al):
            """median step ms and its forward / backward phases (ms); al=None: resident"""
            res, moved = [], None
            for rep in range(1 + max(1, args.steps // 2)):
                torch.cuda.synchronize()
                e0, em, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                e0.record(stream)
                if al is None:
                    eng.step(x["q"], x["k"], x["v"], x["do"], stream, mark=em)
                else:
                    moved = eng.step_offload(x["q"], x["k"], x["v"], x["do"], al, stream, mark=em)
                e1.record(stream)
                torch.cuda.synchronize()
                if rep > 0:
                    res.append((e0.elapsed_time(e1), e0.elapsed_time(em), em.elapsed_time(e1)))
            med = [max_over_ranks(statistics.median(r[j] for r in res), ws) for j in range(3)]
            return med, moved

        (res_ms, res_f, res_b), _ = time_offload(None)  # resident, same session, phase-split
        (off_ms, off_f, off_b), moved = time_offload(alpha)
        (fix_ms, _, _), fix_moved = time_offload([1.0] * (N - 1) + [0.0])  # fixed full offload (P:250 baseline)
        offload = {"policy": "type1-alpha (Q,O,LSE offloaded after fwd(i), prefetched depth 2 before bwd(i))",
                   "ms_per_step": round(off_ms, 3), "resident_ms_per_step": round(ms, 3),
                   "exposed_pct": round(100.0 * (off_ms - ms) / ms, 2),
                   "exposed_split_pct": {"fwd": round(100.0 * (off_f - res_f) / res_ms, 2),
                                         "bwd": round(100.0 * (off_b - res_b) / res_ms, 2),
                                         "resident_ms_this_run": round(res_ms, 3),
                                         "note": "phase times vs a resident step timed in the same loop"},
                   "d2h_bytes": moved["d2h"], "h2d_bytes": moved["h2d"],
                   "alpha": [round(a, 3) for a in alpha], "bw_d2h_gbs_assumed": bw / 1e9,
                   "fixed_alpha1": {"ms_per_step": round(fix_ms, 3), "exposed_pct": round(100.0 * (fix_ms - ms) / ms, 2),
                                    "d2h_bytes": fix_moved["d2h"]},
                   "fwd_ms_per_chunk": [round(t * 1e3, 3) for t in t_fwd],
                   "d2h_ms_per_chunk_alpha1": [round(a / bw * 1e3, 3) for a in A]}
        eng.free_host()

    # ---- KV streaming policy (hot prefix resident, colder chunks streamed from host)
    kvs = None
    budget = None
    if args.device_budget > 0:
        # SURVEY §8(a) note / reading L10: the largest hot prefix P whose resident bytes fit
        # the budget; everything but K/V of chunks >= P stays resident, plus a 2-slot ring
        # of W-chunk windows for the streamed K/V
        el = eng.elem
        tok = h * d
        non_kv = S * tok * (6 * el + 2 * 4) + S * h * 4 * 2 + max(L.chunk_len(i) for i in range(N)) * tok * 8
        ring = 2 * args.kv_window * max(L.chunk_len(i) for i in range(N)) * tok * 2 * el
        kv_of = [L.chunk_len(i) * tok * 2 * el for i in range(N)]
        room = args.device_budget * 1e9 - non_kv - ring
        P = 0
        while P < N and sum(kv_of[:P + 1]) <= room:
            P += 1
        if room < 0:
            raise SystemExit(f"--device-budget {args.device_budget} GB is below the non-KV working set")
        args.kv_hot = P
        budget = {"device_budget_gb": args.device_budget, "hot_prefix_chosen": P,
                  "resident_bytes": int(non_kv + ring + sum(kv_of[:P])),
                  "all_resident_bytes": int(non_kv + sum(kv_of))}
    if args.kv_hot >= 0:
        res = []
        st = None
        for rep in range(1 + max(1, args.steps // 2)):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            if args.kv_group > 1:
                st = eng.step_kv_stream_grouped(x["q"], x["k"], x["v"], x["do"], hot=args.kv_hot,
                                                window=args.kv_window, group=args.kv_group, stream=stream)
            else:
                st = eng.step_kv_stream(x["q"], x["k"], x["v"], x["do"], hot=args.kv_hot, window=args.kv_window,
                                        stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            if rep > 0:
                res.append(e0.elapsed_time(e1))
        kv_ms = max_over_ranks(statistics.median(res), ws)
        kvs = {"policy": f"kv hot-prefix P={args.kv_hot} resident, chunks >= P streamed H2D in windows of "
                         f"{args.kv_window} (2-slot ring) for every later fwd/bwd"
                         + (f", each window shared by {args.kv_group} consecutive chunks" if args.kv_group > 1 else "")
                         + "; Type-1 resident", "group": args.kv_group,
               "ms_per_step": round(kv_ms, 3), "resident_ms_per_step": round(ms, 3),
               "exposed_pct": round(100.0 * (kv_ms - ms) / ms, 2), "h2d_bytes": st["h2d"], "d2h_bytes": st["d2h"],
               "h2d_gbs_achieved": round(st["h2d"] / (kv_ms * 1e-3) / 1e9, 1), "windows": st["windows"],
               "budget": budget}
        eng.free_host()

    # ---- final gather of O over NCCL (multi-GPU only, not timed in value)
    gather = None
    full = eng.o
    if ws > 1:
        from paper_2503_10377_b200.dist import gather_heads
        g0 = time.perf_counter()
        full = gather_heads(eng.o, ws)
        torch.cuda.synchronize()
        import torch.distributed as dist
        gather = {"op": f"all_gather O over {dist.get_backend()}", "ms": round((time.perf_counter() - g0) * 1e3, 2),
                  "bytes": full.numel() * full.element_size()}
    o_digest = None
    if args.o_digest:  # forward is bitwise deterministic per head: sharded and unsharded runs must agree
        import hashlib
        o_digest = hashlib.sha256(full.contiguous().view(torch.uint8).cpu().numpy().tobytes()).hexdigest()

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        c = cpu_oracle_sample()
        cpu = {"value": round(c["value"], 6), "unit": "TFLOP/s", "cores": c["cores"], "kind": "oracle",
               "sample": c["sample"], "cpu_model": c["cpu_model"],
               "full_oracle_hours_extrapolated": round(fl_total / (c["value"] * 1e12) / 3600, 1),
               "more": "tools/oracle_timing.py -> profiles/r01/oracle_timing.json (C1 full, 1 thread)"}

    ctx.close()
    if rank != 0:
        return None
    line = {
        "metric": METRIC, "value": round(tflops, 2), "unit": "TFLOP/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": cfg["dtype"], "data": "synthetic",
        "config": {"workload": cfg["workload"], "heads": cfg["heads"], "heads_per_gpu": h, "head_dim": d,
                   "seq_len": S, "chunks": N, "chunk_len": S // N if args.partition == "equal" else "balanced",
                   "partition": args.partition, "policy": "resident (KV + activations on GPU)",
                   "parallelism": (f"heads sharded over {ws} GPU(s), no collective in step" if args.shard_of == 1 else
                                   f"rank 0's share of a {args.shard_of}-GPU head split, run on 1 GPU "
                                   f"(value = per-GPU TFLOP/s of that config)"),
                   "l2": f"inputs {4 * S * h * d * eng.elem / 2**30:.1f} GiB per GPU > 126 MB L2 (no flush needed)"},
        "per_gpu_tflops": round(per_gpu, 2),
        "pct_bf16_peak": {"burst": round(100 * per_gpu / peaks["burst"], 1),
                          "sustained": round(100 * per_gpu / peaks["sustained"], 1),
                          "datasheet_2250": round(100 * per_gpu / 2250.0, 1), "source": peaks["source"]},
        "tokens_per_s": round(S / (ms * 1e-3), 1), "tgs": round(S / (ms * 1e-3) / ws, 1),
        "fwd_tflops": round(ach_fwd, 2), "bwd_tflops": round(ach_bwd, 2),
        "roofline": {"bound": "tensor", "kernel": "bwd_kernel (sppo_attn_bwd calls, incl. Delta/cast helpers)",
                     "achieved": round(ach_bwd, 2), "peak": peaks["sustained"], "unit": "TFLOP/s",
                     "frac": round(ach_bwd / peaks["sustained"], 3), "traffic": ncu_traffic("bwd_kernel"),
                     "peak_kind": "sustained bf16 (kernel timed inside a long step), " + peaks["source"],
                     "share_of_step": round(bwd_ms / ms, 3)},
        "e2e": e2e, "gpu_launches": launches, "clocks": clocks, "offload": offload, "kv_stream": kvs,
        "gather": gather, "numa": args.numa,
        "cpu_baseline": cpu,
    }
    if o_digest:
        line["o_sha256"] = o_digest
    if (args.config == "C2" and ws == 1 and args.shard_of == 1 and not args.no_c3 and args.partition == "equal"
            and not (args.heads or args.seq_len or args.chunks)):
        # the north-star target workload (1M tokens on 1 GPU) on the same clock as the line
        del eng, x, full
        torch.cuda.empty_cache()
        line["target_c3"] = resident_sub("C3", local)
    return line


def resident_sub(name, local, steps=2, warmup=1):
    """Bounded resident fwd+bwd measurement of another config on this GPU (BASELINE.json
    north_star target: >= 60 % of dense bf16 peak at 1M tokens on 1 GPU): `warmup`
    untimed steps (each ~30 s at C3), `steps` timed with CUDA events on the launching
    stream, clocks sampled during the timed region."""
    from paper_2503_10377_b200 import engine, sppo
    from synth import make_tensor
    cfg = CONFIGS[name]
    dev = torch.device("cuda", local)
    heads = list(range(cfg["heads"]))
    h, d, S, N = len(heads), cfg["d"], cfg["S"], cfg["N"]
    ctx = sppo.Context(local)
    offsets = sppo.partition_equal(S, N)
    L = sppo.Layout(h, d, offsets)
    x = {t: make_tensor(t, S, heads, d, seed=0, dtype=torch.bfloat16, device=dev) for t in ("q", "k", "v", "do")}
    eng = engine.ChunkedAttention(ctx, L, device=dev)
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        eng.step(x["q"], x["k"], x["v"], x["do"], stream)
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    phase = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    for st in range(steps):
        marks[st].record(stream)
        eng.step(x["q"], x["k"], x["v"], x["do"], stream, mark=phase[st])
    marks[steps].record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = marks[0].elapsed_time(marks[steps]) / steps
    fwd_ms = sum(marks[i].elapsed_time(phase[i]) for i in range(steps)) / steps
    bwd_ms = sum(phase[i].elapsed_time(marks[i + 1]) for i in range(steps)) / steps
    fl = flops_of(offsets, h, d)
    tf = fl / (ms * 1e-3) / 1e12
    peaks = load_peaks()
    ctx.close()
    del eng, x
    torch.cuda.empty_cache()
    return {"workload": cfg["workload"], "value": round(tf, 2), "unit": "TFLOP/s", "ms_per_step": round(ms, 1),
            "steps": steps, "warmup": warmup, "fwd_tflops": round(flops_of(offsets, h, d, "fwd") / (fwd_ms * 1e-3) / 1e12, 2),
            "bwd_tflops": round(flops_of(offsets, h, d, "bwd") / (bwd_ms * 1e-3) / 1e12, 2),
            "pct_bf16_peak": {"burst": round(100 * tf / peaks["burst"], 1),
                              "sustained": round(100 * tf / peaks["sustained"], 1), "source": peaks["source"]},
            "target": ">= 60 % of dense bf16 peak at 1M tokens on 1 GPU (BASELINE.json north_star)",
            "clocks": clocks}


# ------------------------------------------------------------------ context parallelism
def run_cp(args, cfg, ws, rank, local):
    """--parallel cp: the sequence sharded over the ranks (zigzag chunks), all heads
    on every rank, K/V (and dK/dV accumulators) rotated around the ring
    (paper_2503_10377_b200.cp).  value = whole-problem FLOPs / max-over-ranks time."""
    from paper_2503_10377_b200 import cp, sppo
    from synth import make_tensor

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    h, d, S, N = cfg["heads"], cfg["d"], cfg["S"], cfg["N"]
    dtype = sppo.SPPO_BF16 if cfg["dtype"] == "bf16" else sppo.SPPO_FP32
    tdt = torch.bfloat16 if dtype == sppo.SPPO_BF16 else torch.float32
    ctx = sppo.Context(local)
    offsets = sppo.partition_equal(S, N)
    L = sppo.Layout(h, d, offsets, dtype=dtype)
    own = cp.owned_chunks(N, ws, rank)
    x = {}
    for t in ("q", "k", "v", "do"):  # this rank's own tokens only (seeds per global head)
        full = make_tensor(t, S, range(h), d, seed=0, dtype=tdt, device=dev)
        x[t] = torch.cat([full[offsets[i]:offsets[i + 1]] for i in own]).contiguous()
        del full
    ra = cp.RingAttention(ctx, L, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        ra.forward(x["q"], x["k"], x["v"], stream)
        ra.backward(x["q"], x["k"], x["v"], x["do"], stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(ws)
    clk = ClockSampler(local)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    barrier(ws)
    ms = max_over_ranks(t0.elapsed_time(t1) / args.steps, ws)
    fl = flops_of(offsets, h, d)
    peaks = load_peaks()
    ctx.close()
    if rank != 0:
        return None
    tflops = fl / (ms * 1e-3) / 1e12
    return {"metric": METRIC, "value": round(tflops, 2), "unit": "TFLOP/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": cfg["dtype"], "data": "synthetic",
            "config": {"workload": cfg["workload"], "heads": h, "head_dim": d, "seq_len": S, "chunks": N,
                       "parallelism": f"context parallel: sequence zigzag-sharded over {ws} GPU(s), K/V ring "
                                      f"(P2P), all heads per GPU",
                       "l2": "inputs > 126 MB L2 (no flush needed)"},
            "per_gpu_tflops": round(tflops / ws, 2),
            "pct_bf16_peak": {"burst": round(100 * tflops / ws / peaks["burst"], 1), "source": peaks["source"]},
            "tokens_per_s": round(S / (ms * 1e-3), 1), "clocks": clocks, "gpu_launches": None,
            "note": "kernel roofline / e2e / offload / cpu_baseline: see the default (--parallel heads) line"}


# ------------------------------------------------------------------ full layer per chunk
LAYER_METRIC = "chunked GPT layer fwd+bwd TFLOP/s per B200 (GEMMs + chunked attention), tokens/s"


def cpu_oracle_layer_sample(H, heads):
    """The fp64 layer oracle as it stands on a bounded sample: 512 tokens of the
    layer (hidden H, `heads` heads) in 2 chunks, forward + reverse-order backward."""
    import oracle.layer as OL
    import synth
    try:
        from threadpoolctl import threadpool_info
        cores = max([t.get("num_threads", 1) for t in threadpool_info()] or [1])
    except Exception:
        cores = os.cpu_count()
    S_s = 512
    p = {k: v.double().numpy() for k, v in synth.make_layer_params(H, 0).items()}
    io = synth.make_layer_io(S_s, H, 0)
    t0 = time.perf_counter()
    z, cache = OL.layer_fwd(io["x"].double().numpy(), p, heads, offsets=[0, 256, 512])
    OL.chunked_layer_bwd(io["dz"].double().numpy(), cache, p)
    dt = time.perf_counter() - t0
    f = OL.layer_flops(S_s, H, d=H // heads)
    fl = sum(f.values())
    return dict(value=fl / dt / 1e12, cores=int(cores), seconds=dt,
                sample=f"oracle fp64 layer fwd+bwd, {S_s} tokens (2 chunks), H={H}, {fl:.3e} FLOP in {dt:.1f}s")


def layer_offsets(args, S, N, H):
    """a0 for the layer: equal, attention-balanced (pairs only) or layer-balanced
    (pairs + the token-wise GEMM work: 72 h^2 s + 14 h pairs FLOPs -> lin = 36 h / 7)."""
    from paper_2503_10377_b200 import sppo
    if args.partition == "balanced":
        return sppo.partition_balanced(S, N)
    if args.partition == "layer-balanced":
        return sppo.partition_balanced(S, N, 36 * H // 7)
    return sppo.partition_equal(S, N)


def run_layer(args, cfg, ws, rank, local):
    """One step = the GPT layer (hidden = heads*d of the config) forward over the
    N chunks then backward in reverse (engine_layer.ChunkedLayer).  N > 1 ranks
    partition the heads (tensor parallelism: column / row-parallel projections,
    NCCL all-reduce of the partial sums, engine_layer tp=...): the total work is
    fixed (strong scaling), value = the whole layer's FLOPs / max-over-ranks time."""
    from paper_2503_10377_b200 import engine_layer, msp, sppo
    import synth

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    heads, d, S, N = cfg["heads"], cfg["d"], cfg["S"], cfg["N"]
    H = heads * d
    ctx = sppo.Context(local)
    offsets = layer_offsets(args, S, N, H)
    params = synth.make_layer_params(H, 0, device=dev)
    if ws > 1:
        params = engine_layer.shard_params(params, H, heads, rank, ws)
    io = synth.make_layer_io(S, H, 0, device=dev)
    lay = engine_layer.ChunkedLayer(ctx, H, heads, offsets, params, device=dev, streams=args.layer_streams,
                                    tp=(rank, ws, None) if ws > 1 else None)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        lay.step(io["x"], io["dz"], stream)
    torch.cuda.synchronize()
    lay.launches = 0
    barrier(ws)
    clk = ClockSampler(local)
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    phase = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for st in range(args.steps):
        marks[st].record(stream)
        lay.step(io["x"], io["dz"], stream, mark=phase[st])
    marks[args.steps].record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    launches = lay.launches // args.steps
    barrier(ws)
    ms = max_over_ranks(marks[0].elapsed_time(marks[args.steps]) / args.steps, ws)
    fwd_ms = sum(marks[i].elapsed_time(phase[i]) for i in range(args.steps)) / args.steps
    bwd_ms = sum(phase[i].elapsed_time(marks[i + 1]) for i in range(args.steps)) / args.steps
    pairs = sppo.causal_pairs(offsets)
    f_gemm_fwd, f_attn_fwd = 24 * H * H * S, 4 * d * heads * pairs
    f_fwd = f_gemm_fwd + f_attn_fwd
    f_bwd = 2 * f_gemm_fwd + 10 * d * heads * pairs
    fl = f_fwd + f_bwd
    peaks = load_peaks()
    tflops = fl / (ms * 1e-3) / 1e12

    # per-kernel-class device time in one instrumented step (events around each call)
    lay.timing = True
    lay.events = {"fwd": [], "bwd": []}
    lay.gemm_events, lay.attn_events = [], []
    lay.step(io["x"], io["dz"], stream)
    torch.cuda.synchronize()
    gemm_ms = sum(a.elapsed_time(b) for a, b, _ in lay.gemm_events)
    gemm_fl = sum(f for _, _, f in lay.gemm_events)
    attn_ms = sum(a.elapsed_time(b) for a, b in lay.attn_events)
    t_fwd = lay.chunk_ms("fwd")
    t_bwd = list(reversed(lay.chunk_ms("bwd")))  # recorded N-1..0 -> index by chunk
    lay.timing = False
    lay.attn_events = None
    # subsequence pipeline model: PP stages of one such layer each, the
    # measured per-chunk times on every stage; makespan from sppo_pipeline_makespan
    F = sum(t_fwd) + sum(t_bwd)
    pipe = {"note": "MODEL from this run's measured per-chunk layer fwd/bwd times (1 layer per stage); "
                    "multi-GPU execution not measured (one GPU in this environment)",
            "F_ms": round(F, 3)}
    # MSP: bubble-adjacent chunks tensor-parallel over the
    # stage's Left-SP / Right-SP range (msp.py).  Per-rank times of a g-way shard of
    # this layer (heads / g, MLP columns / g) are MEASURED here for g | heads (one
    # rank's compute; the range's all-reduces not included); other g: t_1 / g.
    shard = {}
    if ws == 1 and not args.no_msp:
        for g in (2, 4, 8):
            if heads % g:
                continue
            sl = engine_layer.ChunkedLayer(ctx, H, heads, offsets, engine_layer.shard_params(params, H, heads, 0, g),
                                           device=dev, tp=(0, g, False))
            sl.step(io["x"], io["dz"], stream)
            sl.timing, sl.events = True, {"fwd": [], "bwd": []}
            sl.step(io["x"], io["dz"], stream)
            torch.cuda.synchronize()
            shard[g] = (sl.chunk_ms("fwd"), list(reversed(sl.chunk_ms("bwd"))))
            del sl
    for pp in (2, 4, 8):
        T = sppo.pipeline_makespan(pp, t_fwd, t_bwd)
        pipe[f"pp{pp}"] = {"makespan_ms": round(T, 3), "bubble_ratio": round((T - F) / F, 4),
                           "uniform_formula": round(sppo.pipeline_bubble(pp, N), 4)}
        if shard:
            tf = {1: t_fwd, **{g: (shard[g][0] if g in shard else [x / g for x in t_fwd]) for g in range(2, pp + 1)}}
            tb = {1: t_bwd, **{g: (shard[g][1] if g in shard else [x / g for x in t_bwd]) for g in range(2, pp + 1)}}
            Tm = msp.msp_makespan(pp, N, offsets, tf, tb, msp=True)
            Ti = msp.msp_makespan(pp, N, offsets, t_fwd, t_bwd, msp=True)
            pipe[f"pp{pp}"]["msp"] = {"makespan_ms": round(Tm, 3), "bubble_ratio": round((Tm - F) / F, 4),
                                      "speedup_vs_plain": round(T / Tm, 4),
                                      "makespan_perfect_split_ms": round(Ti, 3)}
    if shard:
        pipe["shard_efficiency"] = {f"g{g}": round(F / (g * (sum(f) + sum(b))), 4) for g, (f, b) in shard.items()}
        pipe["msp_note"] = ("MSP plan (msp.MSPPlan list schedule) with this run's per-chunk times; a range of g GPUs "
                            "takes the measured per-rank time of a g-way shard (g | heads) or t_1 / g; "
                            "all-reduces and phase-boundary K/V moves not modeled")
    lay.gemm_events = None

    # Type-1 activation offload with sequence-aware alpha vs the paper's fixed full offload
    offload = None
    if not args.no_offload:
        bw = 56.0  # GB/s pinned D2H measured on this pool (profiles/r01/box_probe.json)
        alpha = lay.alpha_plan(t_fwd, bw)

        def timed(al):
            res, moved = [], None
            for rep in range(3):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                if al is None:
                    lay.step(io["x"], io["dz"], stream)
                else:
                    moved = lay.step_offload(io["x"], io["dz"], al, stream)
                e1.record(stream)
                torch.cuda.synchronize()
                if rep > 0:
                    res.append(e0.elapsed_time(e1))
            return statistics.median(res), moved

        res_ms, _ = timed(None)
        off_ms, moved = timed(alpha)
        fix_ms, fix_moved = timed([1.0] * (N - 1) + [0.0])
        A = [lay.type1_bytes(i) for i in range(N)]
        offload = {"policy": "type1-alpha: a,q,o,y,b,u,g (alpha-prefix) + LSE, LN stats after fwd(i); "
                             "prefetch depth 2 before bwd(i); K,V resident (Type-0)",
                   "resident_ms": round(res_ms, 3), "alpha_ms": round(off_ms, 3),
                   "exposed_pct": round(100 * (off_ms - res_ms) / res_ms, 2),
                   "d2h_bytes": moved["d2h"], "alpha": [round(a, 3) for a in alpha],
                   "fixed_alpha1": {"ms": round(fix_ms, 3), "exposed_pct": round(100 * (fix_ms - res_ms) / res_ms, 2),
                                    "d2h_bytes": fix_moved["d2h"]},
                   "type1_bytes_per_chunk": A[0], "fwd_ms_per_chunk": [round(t, 3) for t in t_fwd],
                   "d2h_ms_per_chunk_alpha1": [round(a / bw / 1e6, 3) for a in A], "bw_d2h_gbs_assumed": bw}
        lay.free_host()

    # e2e: x, dz from pinned host memory in (chunk by chunk, overlapped), z, dx back after each chunk
    e2e = None
    if not args.no_e2e:
        nb = S * H * 2
        hin = {t: ctx.host_alloc(nb) for t in ("x", "dz")}
        hout = {t: ctx.host_alloc(nb) for t in ("z", "dx")}
        for t in ("x", "dz"):
            ctx.kv_offload(0, io[t], hin[t], nb, 1.0, producer=stream)
        ctx.sync()
        xin = {t: torch.empty_like(io[t]) for t in ("x", "dz")}
        res = []
        h2d = d2h = 0
        for rep in range(3):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            h2d, d2h, last = lay.step_host_io(hin["x"], hin["dz"], hout["z"], hout["dx"], xin["x"], xin["dz"], stream)
            stream.wait_event(last)
            e1.record(stream)
            torch.cuda.synchronize()
            if rep > 0:
                res.append(e0.elapsed_time(e1))
        e2e_ms = max_over_ranks(statistics.median(res), ws)
        e2e = {"value": round(fl / (e2e_ms * 1e-3) / 1e12, 2), "unit": "TFLOP/s", "ms_per_step": round(e2e_ms, 3),
               "h2d_bytes_per_step": h2d * ws, "d2h_bytes_per_step": d2h * ws,
               "path": "pinned host x (forward order), dz (backward order) -> chunk-wise sppo_kv_prefetch overlapped "
                       "with compute; z after fwd(i), dx after bwd(i) -> sppo_kv_offload"}
        for ptr in list(hin.values()) + list(hout.values()):
            ctx.host_free(ptr)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        c = cpu_oracle_layer_sample(H, heads)
        cpu = {"value": round(c["value"], 6), "unit": "TFLOP/s", "cores": c["cores"], "kind": "oracle",
               "sample": c["sample"]}
    gemm_tf = gemm_fl / (gemm_ms * 1e-3) / 1e12
    line = {"metric": LAYER_METRIC, "value": round(tflops, 2), "unit": "TFLOP/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": cfg["workload"].replace("attention layer", "layer") + " -- full GPT layer "
                                   f"(hidden {H}, MLP 4x, LayerNorm, GELU) per chunk",
                       "hidden": H, "heads": heads, "seq_len": S, "chunks": N, "partition": args.partition,
                       "streams": args.layer_streams,
                       "parallelism": f"tensor parallel: heads over {ws} GPUs" if ws > 1 else "single GPU",
                       "l2": "inputs larger than L2 (activations GBs per step)"},
            "tokens_per_s": round(S / (ms * 1e-3), 1), "pct_of_bf16_peak": round(100 * tflops / ws / peaks["burst"], 2),
            "fwd_tflops": round(f_fwd / (fwd_ms * 1e-3) / 1e12, 1), "bwd_tflops": round(f_bwd / (bwd_ms * 1e-3) / 1e12, 1),
            "breakdown": {"gemm_ms": round(gemm_ms, 3), "gemm_tflops": round(gemm_tf, 1),
                          "attention_ms": round(attn_ms, 3),
                          "attention_tflops": round((f_attn_fwd * 3.5) / ws / (attn_ms * 1e-3) / 1e12, 1),
                          "gemm_flop_share": round(3 * f_gemm_fwd / fl, 3)},
            "gpu_launches": launches,
            "roofline": {"bound": "tensor", "kernel": "gemm_kernel (all layer GEMMs, event-timed in one step)",
                         "achieved": round(gemm_tf, 1), "peak": peaks["burst"], "unit": "TFLOP/s",
                         "frac": round(gemm_tf / peaks["burst"], 3), "traffic": None,
                         "peak_source": peaks["source"] + " bf16 burst"},
            "clocks": clocks, "offload": offload, "pipeline_model": pipe, "e2e": e2e, "cpu_baseline": cpu}
    ctx.close()
    return line if rank == 0 else None


def run_layer_pool(args, cfg, ws, rank, local):
    """The layer step with two-level activation management that actually frees
    memory (engine_layer pool mode): every chunk's Type-1 set leaves the GPU as
    its alpha-prefix after fwd(i) and is rebuilt before bwd(i).  Needed where the
    all-resident step does not fit (e.g. C3's 1M tokens at hidden 4096).  Warm-up
    steps 1-2 run alpha = 1, step 2 measures the per-chunk forward times; alpha is then
    the sequence-aware plan.  value = FLOPs / offloaded step time."""
    from paper_2503_10377_b200 import engine_layer, msp, sppo
    import synth

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    heads, d, S, N = cfg["heads"], cfg["d"], cfg["S"], cfg["N"]
    H = heads * d
    ctx = sppo.Context(local)
    offsets = layer_offsets(args, S, N, H)
    params = synth.make_layer_params(H, 0, device=dev)
    io = synth.make_layer_io(S, H, 0, device=dev)
    lay = engine_layer.ChunkedLayer(ctx, H, heads, offsets, params, device=dev, pool=True)
    stream = torch.cuda.current_stream()
    bw = 56.0  # GB/s pinned D2H measured on this pool (profiles/r01/box_probe.json)
    full = [1.0] * (N - 1) + [0.0]
    lay.step_offload(io["x"], io["dz"], full, stream)  # warm-up (allocator, pinned host buffers)
    lay.timing = True
    lay.events = {"fwd": [], "bwd": []}
    lay.step_offload(io["x"], io["dz"], full, stream)
    torch.cuda.synchronize()
    t_fwd = lay.chunk_ms("fwd")
    lay.timing = False
    alpha = lay.alpha_plan(t_fwd, bw)
    for _ in range(max(0, args.warmup - 2)):
        lay.step_offload(io["x"], io["dz"], alpha, stream)
    torch.cuda.synchronize()
    lay.launches = 0
    torch.cuda.reset_peak_memory_stats(dev)
    barrier(ws)
    clk = ClockSampler(local)
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    phase = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    moved = None
    for st in range(args.steps):
        marks[st].record(stream)
        moved = lay.step_offload(io["x"], io["dz"], alpha, stream, mark=phase[st])
    marks[args.steps].record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    launches = lay.launches // args.steps
    peak = torch.cuda.max_memory_allocated(dev)
    barrier(ws)
    ms = max_over_ranks(marks[0].elapsed_time(marks[args.steps]) / args.steps, ws)
    fwd_ms = sum(marks[i].elapsed_time(phase[i]) for i in range(args.steps)) / args.steps
    bwd_ms = sum(phase[i].elapsed_time(marks[i + 1]) for i in range(args.steps)) / args.steps
    pairs = sppo.causal_pairs(offsets)
    f_gemm_fwd, f_attn_fwd = 24 * H * H * S, 4 * d * heads * pairs
    f_fwd = f_gemm_fwd + f_attn_fwd
    f_bwd = 2 * f_gemm_fwd + 10 * d * heads * pairs
    fl = f_fwd + f_bwd
    peaks = load_peaks()
    tflops = fl / (ms * 1e-3) / 1e12
    # one instrumented step: GEMM / attention device time
    lay.gemm_events, lay.attn_events = [], []
    lay.step_offload(io["x"], io["dz"], alpha, stream)
    torch.cuda.synchronize()
    gemm_ms = sum(a.elapsed_time(b) for a, b, _ in lay.gemm_events)
    gemm_fl = sum(f for _, _, f in lay.gemm_events)
    attn_ms = sum(a.elapsed_time(b) for a, b in lay.attn_events)
    lay.gemm_events = lay.attn_events = None
    # the paper's fixed alpha = 1 (every chunk's activations fully offloaded) for comparison
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    fix_moved = lay.step_offload(io["x"], io["dz"], full, stream)
    e1.record(stream)
    torch.cuda.synchronize()
    fix_ms = e0.elapsed_time(e1)
    lay.free_host()
    A = [lay.type1_bytes(i) for i in range(N)]
    total_mem = torch.cuda.get_device_properties(dev).total_memory
    # device bytes an all-resident step would need on top of what this one keeps: every
    # chunk's Type-1 set at once (the pool step keeps only suffixes + in-flight sets)
    resident_need = peak + sum(A) - max(A) * 3
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        c = cpu_oracle_layer_sample(H, heads)
        cpu = {"value": round(c["value"], 6), "unit": "TFLOP/s", "cores": c["cores"], "kind": "oracle",
               "sample": c["sample"]}
    gemm_tf = gemm_fl / (gemm_ms * 1e-3) / 1e12
    line = {"metric": LAYER_METRIC, "value": round(tflops * ws, 2), "unit": "TFLOP/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": cfg["workload"].replace("shape", "layer") + " -- full GPT layer (hidden "
                                   f"{H}) per chunk, Type-1 activations offloaded (pool: device copies freed)",
                       "hidden": H, "heads": heads, "seq_len": S, "chunks": N, "partition": args.partition,
                       "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU",
                       "l2": "inputs larger than L2"},
            "tokens_per_s": round(S * ws / (ms * 1e-3), 1), "pct_of_bf16_peak": round(100 * tflops / peaks["burst"], 2),
            "fwd_tflops": round(f_fwd / (fwd_ms * 1e-3) / 1e12, 1), "bwd_tflops": round(f_bwd / (bwd_ms * 1e-3) / 1e12, 1),
            "breakdown": {"gemm_ms": round(gemm_ms, 3), "gemm_tflops": round(gemm_tf, 1),
                          "attention_ms": round(attn_ms, 3),
                          "attention_tflops": round((f_attn_fwd * 3.5) / (attn_ms * 1e-3) / 1e12, 1)},
            "memory": {"peak_allocated_gb": round(peak / 1e9, 2), "device_total_gb": round(total_mem / 1e9, 2),
                       "type1_bytes_all_chunks_gb": round(sum(A) / 1e9, 2),
                       "all_resident_estimate_gb": round(resident_need / 1e9, 2),
                       "fits_without_offload": bool(resident_need < total_mem)},
            "offload": {"alpha": [round(a, 3) for a in alpha], "d2h_bytes": moved["d2h"], "h2d_bytes": moved["h2d"],
                        "fixed_alpha1": {"ms": round(fix_ms, 3), "slowdown_pct": round(100 * (fix_ms - ms) / ms, 2),
                                         "d2h_bytes": fix_moved["d2h"]},
                        "fwd_ms_per_chunk_calibration": [round(t, 3) for t in t_fwd], "bw_d2h_gbs_assumed": bw},
            "gpu_launches": launches,
            "roofline": {"bound": "tensor", "kernel": "gemm_kernel (all layer GEMMs, event-timed in one step)",
                         "achieved": round(gemm_tf, 1), "peak": peaks["burst"], "unit": "TFLOP/s",
                         "frac": round(gemm_tf / peaks["burst"], 3), "traffic": None,
                         "peak_source": peaks["source"] + " bf16 burst"},
            "clocks": clocks, "e2e": None, "cpu_baseline": cpu}
    ctx.close()
    return line if rank == 0 else None


# ------------------------------------------------------------------ reference arm (the oracle)
def run_reference(args, cfg, ws, rank):
    if rank != 0:
        return None
    res = []
    c = None
    layer = args.workload == "layer"
    for it in range(args.warmup + args.steps):
        c = cpu_oracle_layer_sample(cfg["heads"] * cfg["d"], cfg["heads"]) if layer else cpu_oracle_sample()
        if it >= args.warmup:
            res.append(c)
    secs = statistics.median([r["seconds"] for r in res])
    val = statistics.median([r["value"] for r in res])
    return {"metric": LAYER_METRIC if layer else METRIC, "value": round(val, 6), "unit": "TFLOP/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(secs * 1e3, 1), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": cfg["workload"] + " -- bounded oracle sample per step", "sample": c["sample"]},
            "cpu_baseline": {"value": round(val, 6), "unit": "TFLOP/s", "cores": c["cores"], "kind": "oracle",
                             "sample": c["sample"]},
            "e2e": {"value": round(val, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-offload", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--kv-hot", type=int, default=-1, help="also time KV streaming with this hot prefix (-1: skip)")
    ap.add_argument("--kv-window", type=int, default=4)
    ap.add_argument("--kv-group", type=int, default=1, help="KV streaming: chunks sharing each streamed window")
    ap.add_argument("--fwd-streams", type=int, default=None, choices=[1, 2],
                    help="resident step: forward launches alternate over this many streams (default: by launch size)")
    ap.add_argument("--device-budget", type=float, default=0.0,
                    help="GB of device memory for the step: picks the KV hot prefix that fits (0: off)")
    ap.add_argument("--partition", default="equal", choices=["equal", "balanced", "layer-balanced"])
    ap.add_argument("--shard-of", type=int, default=1, help="1 GPU: run rank 0's heads of a G-GPU split")
    ap.add_argument("--layer-streams", type=int, default=1, choices=[1, 2],
                    help="layer workload: 2 = token-wise halves of chunk i overlap chunk i+1's attention phase")
    ap.add_argument("--layer-pool", action="store_true",
                    help="layer workload with activation sets freed after offload (fits C3's 1M tokens)")
    ap.add_argument("--workload", default="attention", choices=["attention", "layer"],
                    help="attention: the chunked attention hot path (headline); layer: full GPT layer per chunk")
    ap.add_argument("--parallel", default="heads", choices=["heads", "cp"],
                    help="multi-GPU split: heads (no collective in the step) or context-parallel ring")
    ap.add_argument("--heads", type=int, default=0, help="override the config's head count (tests)")
    ap.add_argument("--seq-len", type=int, default=0, help="override the config's S (tests)")
    ap.add_argument("--chunks", type=int, default=0, help="override the config's N (tests)")
    ap.add_argument("--o-digest", action="store_true",
                    help="add sha256 of the (gathered) forward output O to the line (sharded == unsharded check)")
    ap.add_argument("--no-msp", action="store_true", help="layer workload: skip the MSP shard timings")
    ap.add_argument("--no-c3", action="store_true",
                    help="skip the bounded C3 (1M tokens, the north-star target) sub-measurement of the C2 line")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: warmup < 3 violates the timing rules", file=sys.stderr)
    os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator / NVLS lines in the log (rank count evidence)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # plain `python bench.py --gpus N`: launch the N ranks ourselves (one process per GPU)
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    ws_env = int(os.environ.get("WORLD_SIZE", "1"))
    if ws_env != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws_env}; launch with torchrun --nproc-per-node "
              f"{args.gpus} or without torchrun", file=sys.stderr)
        sys.exit(2)
    ws, rank, local = dist_setup()
    numa = bind_numa(local) if args.impl == "ours" else None
    cfg = dict(CONFIGS[args.config])
    if args.heads or args.seq_len or args.chunks:  # test-size overrides: the line names the changed workload
        cfg.update({k: v for k, v in (("heads", args.heads), ("S", args.seq_len), ("N", args.chunks)) if v})
        cfg["workload"] = (f"{args.config} override (tests): {cfg['heads']} heads, d={cfg['d']}, S={cfg['S']}, "
                           f"N={cfg['N']}, {cfg['dtype']}")
    args.numa = numa
    if args.impl == "reference":
        line = run_reference(args, cfg, ws, rank)
    elif args.workload == "layer":
        line = (run_layer_pool if args.layer_pool else run_layer)(args, cfg, ws, rank, local)
    elif args.parallel == "cp":
        line = run_cp(args, cfg, ws, rank, local)
    else:
        line = run_ours(args, cfg, ws, rank, local)
    if line is not None:
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
