"""Small run of every layer kernel for compute-sanitizer (memcheck / racecheck /
synccheck): a 2-chunk layer step with pool offload (GEMMs in all orientations,
single-CTA and CTA-pair kernels, LayerNorm fwd/bwd, column reductions) plus a
forced pair GEMM with MN-major operands.
  compute-sanitizer --tool racecheck python tools/sanitize_layer.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_10377_b200 import engine_layer, sppo  # noqa: E402
import synth  # noqa: E402

ctx = sppo.Context(0)
S, H, heads = 512, 256, 2
params = {k: v.cuda() for k, v in synth.make_layer_params(H, 1).items()}
io = {k: v.cuda() for k, v in synth.make_layer_io(S, H, 1).items()}
lay = engine_layer.ChunkedLayer(ctx, H, heads, [0, 256, 512], params, pool=True)
lay.step_offload(io["x"], io["dz"], [0.5, 0.0])
torch.cuda.synchronize()
a = torch.randn(384, 256, device="cuda").to(torch.bfloat16)
b = torch.randn(384, 512, device="cuda").to(torch.bfloat16)
c = torch.zeros(256, 512, device="cuda")
ctx.gemm(256, 512, 384, a, b, c, a_mn=1, b_mn=1, epilogue=sppo.SPPO_EPI_ACC_F32)
ctx.sync()
lay.free_host()
print("ok")
