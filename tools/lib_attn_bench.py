"""Context measurement (not a bench line): library causal attention on this box.

Times torch SDPA on the cuDNN backend (cuDNN's sm_100 fused attention) for one
causal self-attention of S tokens, h heads, d = 128, bf16 — forward alone and
forward + backward — with the FLOP convention of BASELINE.md (forward 4d, backward
10d per causal pair per head).  The SPPO kernels compute the same pairs chunk by
chunk; this says what a vendor kernel reaches on the same box and clocks.

  python tools/lib_attn_bench.py [--seq 131072] [--heads 32] [--reps 3]
  python tools/lib_attn_bench.py --impl sppo --chunks 16   # the SPPO engine, same metric
"""

from __future__ import annotations

import argparse
import json

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=131072)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--backend", default="cudnn", choices=["cudnn", "flash", "efficient"])
    ap.add_argument("--impl", default="lib", choices=["lib", "sppo"])
    ap.add_argument("--chunks", type=int, default=1)
    args = ap.parse_args()
    if args.impl == "sppo":
        return run_sppo(args)
    be = {"cudnn": SDPBackend.CUDNN_ATTENTION, "flash": SDPBackend.FLASH_ATTENTION,
          "efficient": SDPBackend.EFFICIENT_ATTENTION}[args.backend]
    S, h, d = args.seq, args.heads, 128
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v, do = (torch.randn(1, h, S, d, device="cuda", dtype=torch.bfloat16, generator=g)
                   for _ in range(4))
    for t in (q, k, v):
        t.requires_grad_(True)
    pairs = S * (S + 1) / 2
    f_fwd, f_bwd = 4 * d * pairs * h, 10 * d * pairs * h
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    out = {"backend": args.backend, "seq": S, "heads": h, "head_dim": d, "dtype": "bf16",
           "cudnn": torch.backends.cudnn.version()}
    with sdpa_kernel(be):
        for i in range(args.reps + 1):
            torch.cuda.synchronize()
            ev[0].record()
            o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
            ev[1].record()
            o.backward(do)
            ev[2].record()
            torch.cuda.synchronize()
            if i == 0:
                continue  # warm-up (plan build)
            tf = ev[0].elapsed_time(ev[1]) * 1e-3
            tb = ev[1].elapsed_time(ev[2]) * 1e-3
            out.setdefault("fwd_tflops", []).append(round(f_fwd / tf / 1e12, 1))
            out.setdefault("bwd_tflops", []).append(round(f_bwd / tb / 1e12, 1))
            out.setdefault("step_tflops", []).append(round((f_fwd + f_bwd) / (tf + tb) / 1e12, 1))
            q.grad = k.grad = v.grad = None
    print(json.dumps(out))


def run_sppo(args):
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2503_10377_b200 import engine, sppo
    from synth import make_tensor
    S, h, d = args.seq, args.heads, 128
    ctx = sppo.Context(0)
    x = {t: make_tensor(t, S, range(h), d, seed=0, device="cuda") for t in ("q", "k", "v", "do")}
    off = sppo.partition_equal(S, args.chunks)
    eng = engine.ChunkedAttention(ctx, sppo.Layout(h, d, off))
    pairs = sppo.causal_pairs(off)
    out = {"impl": "sppo", "seq": S, "heads": h, "head_dim": d, "chunks": args.chunks, "dtype": "bf16"}
    for i in range(args.reps + 1):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        torch.cuda.synchronize()
        ev[0].record()
        eng.step(x["q"], x["k"], x["v"], x["do"], mark=ev[1])
        ev[2].record()
        torch.cuda.synchronize()
        if i == 0:
            continue
        tf, tb = ev[0].elapsed_time(ev[1]) * 1e-3, ev[1].elapsed_time(ev[2]) * 1e-3
        out.setdefault("fwd_tflops", []).append(round(4 * d * h * pairs / tf / 1e12, 1))
        out.setdefault("bwd_tflops", []).append(round(10 * d * h * pairs / tb / 1e12, 1))
        out.setdefault("step_tflops", []).append(round(14 * d * h * pairs / (tf + tb) / 1e12, 1))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
