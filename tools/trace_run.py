"""Run one C2-shaped step with SPPO_TRACE set (kernel event timestamps of CTA
(0,0) of one launch) and print a per-iteration timeline summary."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_10377_b200 import engine, sppo  # noqa: E402
from synth import make_tensor  # noqa: E402

S, N, h = int(os.environ.get("TS", 131072)), int(os.environ.get("TN", 16)), int(os.environ.get("TH", 32))
ctx = sppo.Context(0)
off = sppo.partition_equal(S, N)
L = sppo.Layout(h, 128, off)
x = {t: make_tensor(t, S, range(h), 128, device="cuda") for t in ("q", "k", "v", "do")}
eng = engine.ChunkedAttention(ctx, L)
eng.step(x["q"], x["k"], x["v"], x["do"])
ctx.sync()
path = os.environ["SPPO_TRACE"]
rows = [list(map(int, l.split())) for l in open(path)]
print("iters", len(rows))
names = ["mma_pre", "dP", "dV", "S+1", "dK", "dQdone", "cP0", "pfull", "dpseen", "dsfull0", "cP1", "dsfull1",
         "rdq", "rfree", "r_end", "ldq"]
import statistics
base = rows[0][1]
for r in rows[:6] + rows[len(rows) // 2:len(rows) // 2 + 4]:
    print(r[0], " ".join(f"{n}={(v - base) if v else -1}" for n, v in zip(names, r[1:])))
per = [rows[i + 1][2] - rows[i][2] for i in range(len(rows) - 1) if rows[i + 1][2] and rows[i][2]]
print("median dP-issue period (cycles):", statistics.median(per) if per else None)
def med(a, b):
    d = [r[1 + b] - r[1 + a] for r in rows if r[1 + a] and r[1 + b]]
    return statistics.median(d) if d else None
for a, b in [(1, 2), (2, 3), (3, 4), (4, 5), (0, 1), (6, 7), (8, 9), (12, 13), (1, 8), (4, 9)]:
    print(f"{names[a]}->{names[b]}: {med(a, b)}")
