"""N-sweep at C2 (SURVEY §8(d) "optional N-sweep"): the same S = 128K, 32-head
attention layer split into N = 1 .. 128 chunks, fwd+bwd TFLOP/s per N (the
subsequence-length trade-off of P:276 / P:289-294 for the attention layer:
more chunks = smaller launches, more diagonal-tile waste and tails).
usage: python tools/n_sweep.py > profiles/r02/n_sweep.json"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_10377_b200 import engine, sppo  # noqa: E402
from synth import make_tensor  # noqa: E402

S, h, d = 131072, 32, 128
ctx = sppo.Context(0)
x = {t: make_tensor(t, S, range(h), d, seed=0, device="cuda") for t in ("q", "k", "v", "do")}
res = []
for N in (1, 2, 4, 8, 16, 32, 64, 128):
    off = sppo.partition_equal(S, N)
    eng = engine.ChunkedAttention(ctx, sppo.Layout(h, d, off))
    for _ in range(3):
        eng.step(x["q"], x["k"], x["v"], x["do"])
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
    for r in range(3):
        ev[2 * r].record()
        eng.step(x["q"], x["k"], x["v"], x["do"], mark=ev[2 * r + 1])
    ev[6].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[6]) / 3
    fwd_ms = sum(ev[2 * r].elapsed_time(ev[2 * r + 1]) for r in range(3)) / 3
    pairs = sppo.causal_pairs(off)
    fl = 14 * d * h * pairs
    res.append({"N": N, "chunk_len": S // N, "ms_per_step": round(ms, 2), "tflops": round(fl / ms / 1e9, 1),
                "fwd_tflops": round(4 * d * h * pairs / fwd_ms / 1e9, 1),
                "bwd_tflops": round(10 * d * h * pairs / (ms - fwd_ms) / 1e9, 1),
                "fwd_streams": eng.fwd_streams, "launches_per_step": eng.launches // 6})
    del eng
    torch.cuda.empty_cache()
print(json.dumps({"config": "C2 shape: 32 heads, d=128, S=131072, bf16, resident; 3 warm-up + 3 timed steps",
                  "sweep": res}, indent=1))
