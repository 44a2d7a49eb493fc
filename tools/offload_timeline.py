"""Overlap timeline of one C2 step with the Type-1 alpha offload policy
(compute-stream idle gaps, host-link GB/s over copy-stream busy
time).  CUDA events around every fwd/bwd call on the compute stream and around
every copy on the ctx's D2H / H2D streams (sppo_ctx_streams); a copy starts at
the later of "its copy stream got there" and "the compute-side event it waits
on".  usage: python tools/offload_timeline.py [--fixed] > profiles/r01/offload_timeline.json"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_10377_b200 import engine, sppo  # noqa: E402
from synth import make_tensor  # noqa: E402

S, h, d, N = 131072, 32, 128, 16
BW = 56e9  # pinned D2H bytes/s on this pool (tools/box_probe.py)


def union(iv):
    out = []
    for a, b in sorted(iv):
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def overlap(a, b):
    tot, j = 0.0, 0
    for x0, x1 in a:
        for y0, y1 in b:
            tot += max(0.0, min(x1, y1) - max(x0, y0))
    return tot


def main():
    ctx = sppo.Context(0)
    off = sppo.partition_equal(S, N)
    eng = engine.ChunkedAttention(ctx, sppo.Layout(h, d, off), timing=True, fwd_streams=1)
    x = {t: make_tensor(t, S, range(h), d, seed=0, device="cuda") for t in ("q", "k", "v", "do")}
    strm = torch.cuda.current_stream()
    for _ in range(2):
        eng.step(x["q"], x["k"], x["v"], x["do"], strm)
    torch.cuda.synchronize()
    t_fwd = [a.elapsed_time(b) * 1e-3 for a, b in eng.events["fwd"][-N:]]
    A = [eng.type1_bytes(i) for i in range(N)]
    if "--fixed" in sys.argv:
        alpha = [1.0] * (N - 1) + [0.0]
    else:
        alpha = sppo.offload_alpha(A, [BW * (t_fwd[i + 1] if i + 1 < N else 0.0) for i in range(N)], 0.0)
    eng.timing = False
    q = x["q"].clone()
    eng.step_offload(q, x["k"], x["v"], x["do"], alpha, strm)  # warm-up (host buffers, descriptors)
    torch.cuda.synchronize()
    eng.timeline = []
    ref = torch.cuda.Event(enable_timing=True)
    ref.record(strm)
    eng.step_offload(q, x["k"], x["v"], x["do"], alpha, strm)
    end = torch.cuda.Event(enable_timing=True)
    end.record(strm)
    torch.cuda.synchronize()
    t = lambda e: ref.elapsed_time(e)  # noqa: E731  ms since step start
    comp, d2h, h2d, rows = [], [], [], []
    for r in eng.timeline:
        if r["kind"] in ("fwd", "bwd"):
            iv = (t(r["e0"]), t(r["e1"]))
            comp.append(iv)
        else:
            iv = (max(t(r["eb"]), t(r["ep"])), t(r["e1"]))
            (d2h if r["kind"] == "d2h" else h2d).append((iv, r["bytes"]))
        rows.append({"kind": r["kind"], "chunk": r["chunk"], "start_ms": round(iv[0], 3), "end_ms": round(iv[1], 3),
                     "bytes": r["bytes"]})
    step_ms = t(end)
    cu = union(comp)
    gaps = [round(b[0] - a[1], 3) for a, b in zip(cu, cu[1:]) if b[0] - a[1] > 1e-3]
    res = {"config": "C2 (32 heads, S=128K, N=16, bf16), Type-1 offload " + ("alpha=1 (fixed)" if "--fixed" in sys.argv
                                                                             else "sequence-aware alpha"),
           "alpha": [round(a, 3) for a in alpha], "step_ms": round(step_ms, 3),
           "compute_busy_ms": round(sum(b - a for a, b in cu), 3),
           "compute_idle_gaps_ms": gaps, "compute_idle_total_ms": round(sum(gaps), 3)}
    for name, lst in (("d2h", d2h), ("h2d", h2d)):
        u = union([iv for iv, _ in lst])
        busy = sum(b - a for a, b in u)
        nbytes = sum(n for _, n in lst)
        res[name] = {"copies": len(lst), "bytes": nbytes, "busy_ms": round(busy, 3),
                     "achieved_gbs": round(nbytes / (busy * 1e-3) / 1e9, 1) if busy > 0 else None,
                     "overlapped_with_compute_pct": round(100 * overlap(u, cu) / busy, 1) if busy > 0 else None}
    res["events"] = rows
    print(json.dumps(res, indent=1))
    eng.free_host()
    ctx.close()


if __name__ == "__main__":
    main()
