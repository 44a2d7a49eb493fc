"""Device-memory timeline of one layer step under the Type-1 offload policies
(the paper's activation-memory-over-time plot, Fig. "System Overview" right
panel, and the recurrence M_i = M_{i-1} + A_i - alpha_{i-1} A_{i-1}):
engine_layer.ChunkedLayer in pool mode (chunk activation sets are separate
allocations released after their D2H), GPT-7B layer, S = 128K, N = 16.
Records torch.cuda.memory_allocated() after each chunk's forward and backward
for: no offload, the paper's fixed alpha = 1, and the sequence-aware alpha.
usage: python tools/layer_memory_timeline.py > profiles/r01/layer_memory_timeline.json"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2503_10377_b200 import engine_layer, sppo  # noqa: E402

S, N, H, heads = 131072, 16, 4096, 32
ctx = sppo.Context(0)
params = synth.make_layer_params(H, 0, device="cuda")
io = synth.make_layer_io(S, H, 0, device="cuda")
lay = engine_layer.ChunkedLayer(ctx, H, heads, sppo.partition_equal(S, N), params, pool=True)
trace = []
fwd0, bwd0 = lay.forward_chunk, lay.backward_chunk


def fwd(i, x, strm):
    fwd0(i, x, strm)
    trace.append(("fwd", i, torch.cuda.memory_allocated()))


def bwd(i, x, dz, strm):
    bwd0(i, x, dz, strm)
    trace.append(("bwd", i, torch.cuda.memory_allocated()))


lay.forward_chunk, lay.backward_chunk = fwd, bwd
full = [1.0] * (N - 1) + [0.0]
lay.step_offload(io["x"], io["dz"], full)  # warm-up (allocator, pinned host buffers)
lay.timing = True
lay.events = {"fwd": [], "bwd": []}
lay.step_offload(io["x"], io["dz"], full)
torch.cuda.synchronize()
t_fwd = lay.chunk_ms("fwd")
lay.timing = False
policies = {"none": [0.0] * N, "fixed_alpha1": full, "sequence_aware": lay.alpha_plan(t_fwd, 56.0)}
torch.cuda.synchronize()
base = torch.cuda.memory_allocated()
out = {"workload": "GPT-7B layer, S = 128K, N = 16, pool mode, one B200", "A_i_bytes": lay.type1_bytes(0),
       "base_bytes_K_V_io_grads_scratch": base, "policies": {}}
for name, alpha in policies.items():
    trace.clear()
    torch.cuda.reset_peak_memory_stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    lay.step_offload(io["x"], io["dz"], alpha)
    e1.record()
    torch.cuda.synchronize()
    out["policies"][name] = {"alpha": [round(a, 3) for a in alpha], "step_ms": round(e0.elapsed_time(e1), 3),
                             "peak_above_base_gb": round((torch.cuda.max_memory_allocated() - base) / 1e9, 3),
                             "timeline_gb": [(k, i, round((m - base) / 1e9, 3)) for k, i, m in trace]}
    print(name, out["policies"][name]["step_ms"], out["policies"][name]["peak_above_base_gb"], file=sys.stderr)
lay.free_host()
print(json.dumps(out, indent=1))
ctx.close()
