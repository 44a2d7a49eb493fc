"""The paper's subsequence-length trade-off for one transformer layer (P:276-285
[§3.3], Fig. "relationship between subsequence length and overall forward
propagation and bubble time for one transformer layer with a hidden dimension
of 4096 and a fixed sequence length of 128K"): the GPT-7B layer (hidden 4096,
32 heads) at S = 128K split into N = 1 .. 128 equal chunks, measured on one
B200 through engine_layer.ChunkedLayer:
  * forward time of the whole sequence (sum over chunks) and fwd+bwd step time,
  * per-chunk forward time (the pipeline's unit of work),
  * the pipeline bubble for PP = 4 stages of one such layer each, from the
    measured per-chunk times (sppo_pipeline_makespan) and the uniform formula
    (PP-1)/N (sppo_pipeline_bubble).
usage: python tools/layer_n_sweep.py > profiles/r01/layer_n_sweep.json"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2503_10377_b200 import engine_layer, sppo  # noqa: E402

S, H, heads, PP = 131072, 4096, 32, 4
ctx = sppo.Context(0)
params = synth.make_layer_params(H, 0, device="cuda")
io = synth.make_layer_io(S, H, 0, device="cuda")
res = []
for N in (1, 2, 4, 8, 16, 32, 64, 128):
    off = sppo.partition_equal(S, N)
    lay = engine_layer.ChunkedLayer(ctx, H, heads, off, params)
    for _ in range(2):
        lay.step(io["x"], io["dz"])
    torch.cuda.synchronize()
    steps = []
    for _ in range(2):
        e0, em, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        lay.step(io["x"], io["dz"], mark=em)
        e1.record()
        torch.cuda.synchronize()
        steps.append((e0.elapsed_time(em), e0.elapsed_time(e1)))
    fwd_ms = min(s[0] for s in steps)
    step_ms = min(s[1] for s in steps)
    lay.timing = True
    lay.events = {"fwd": [], "bwd": []}
    lay.step(io["x"], io["dz"])
    torch.cuda.synchronize()
    tf, tb = lay.chunk_ms("fwd"), list(reversed(lay.chunk_ms("bwd")))
    F = sum(tf) + sum(tb)
    T = sppo.pipeline_makespan(PP, tf, tb) if N >= PP else None
    fl = 72 * H * H * S + 14 * H * sppo.causal_pairs(off)
    r = {"N": N, "chunk": S // N, "fwd_ms": round(fwd_ms, 3), "step_ms": round(step_ms, 3),
         "tflops": round(fl / (step_ms * 1e-3) / 1e12, 1),
         "fwd_ms_per_chunk_first_last": [round(tf[0], 3), round(tf[-1], 3)],
         f"pp{PP}_bubble_measured_times": round((T - F) / F, 4) if T else None,
         f"pp{PP}_bubble_formula": round(sppo.pipeline_bubble(PP, N), 4) if N >= PP else None,
         f"pp{PP}_makespan_ms": round(T, 3) if T else None}
    res.append(r)
    print(json.dumps(r), file=sys.stderr, flush=True)
    del lay
    torch.cuda.empty_cache()
print(json.dumps({"workload": "GPT-7B layer (hidden 4096, 32 heads), S = 128K, equal chunks, one B200",
                  "sweep": res}, indent=1))
ctx.close()
