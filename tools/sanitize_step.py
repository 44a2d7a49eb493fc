"""Small fwd+bwd steps (bf16 tcgen05 path with split windows + ragged chunks, bf16
with ~5 backward items per CTA pair (the persistent kernel's item hand-over), fp32
path) for compute-sanitizer runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_10377_b200 import engine, sppo  # noqa: E402
from synth import make_inputs  # noqa: E402

ctx = sppo.Context(0)
for dtype, tdt, d, off, win, h in ((sppo.SPPO_BF16, torch.bfloat16, 128, [0, 200, 512, 700], 2, 2),
                                    (sppo.SPPO_BF16, torch.bfloat16, 128, [0, 700, 1500, 2048], None, 40),
                                    (sppo.SPPO_FP32, torch.float32, 64, [0, 100, 256], None, 2)):
    x = {k: v.cuda() for k, v in make_inputs(off[-1], range(h), d, seed=1, dtype=tdt).items()}
    eng = engine.ChunkedAttention(ctx, sppo.Layout(h, d, off, dtype=dtype), window=win)
    eng.step(x["q"], x["k"], x["v"], x["do"])
    ctx.sync()
print("sanitize step ok")
