"""Run one C2-shaped step with SPPO_TRACE set (kernel event timestamps of CTA
(0,0) of one launch, see csrc/*.cu TR(...) points) and print a per-iteration
timeline summary.  Env: SPPO_TRACE=<file> SPPO_TRACE_CHUNK=<i> SPPO_TRACE_KIND=fwd|bwd.
Needs a build with the stamp points compiled in (they cost the forward ~6 % even
untaken): tools/make_variant.sh tr -DSPPO_TRACE_BUILD=1, then run from tmp_tr/."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_10377_b200 import engine, sppo  # noqa: E402
from synth import make_tensor  # noqa: E402

S, N, h = int(os.environ.get("TS", 131072)), int(os.environ.get("TN", 16)), int(os.environ.get("TH", 32))
kind = os.environ.get("SPPO_TRACE_KIND", "bwd")
ctx = sppo.Context(0)
off = sppo.partition_equal(S, N)
L = sppo.Layout(h, 128, off)
x = {t: make_tensor(t, S, range(h), 128, device="cuda") for t in ("q", "k", "v", "do")}
eng = engine.ChunkedAttention(ctx, L)
eng.step(x["q"], x["k"], x["v"], x["do"])
ctx.sync()
if "SPPO_TRACE" not in os.environ:  # plain step (e.g. under ncu)
    sys.exit(0)
rows = [list(map(int, l.split())) for l in open(os.environ["SPPO_TRACE"])]
print(kind, "iters", len(rows))
if kind == "bwd":
    names = ["mma_pre", "dP", "dV", "S+1", "dK", "dQdone", "cP0", "pfull", "dpseen", "dsfull0", "cP1", "dsfull1",
             "rdq", "rfree", "r_end", "ldq"]
    pairs = [(1, 2), (2, 3), (3, 4), (4, 5), (0, 1), (6, 7), (8, 9), (12, 13), (1, 8), (4, 9)]
    period_slot = 2
else:
    names = ["vfull", "PV0", "S0+1", "PV1", "S1+1", "s0seen", "s0max", "p0full", "s1seen", "s1max", "p1full",
             "ldK", "ldV", "s0ld", "s0exp64", "-"]
    pairs = [(5, 6), (6, 7), (8, 9), (9, 10), (1, 2), (3, 4), (7, 2), (10, 4), (2, 5), (4, 8), (5, 13), (13, 14),
             (14, 6)]
    period_slot = 2
base = rows[0][1]
for r in rows[:4] + rows[len(rows) // 2:len(rows) // 2 + 3]:
    print(r[0], " ".join(f"{n}={(v - base) if v else -1}" for n, v in zip(names, r[1:])))
per = [rows[i + 1][period_slot] - rows[i][period_slot] for i in range(len(rows) - 1)
       if rows[i + 1][period_slot] and rows[i][period_slot]]
print("median period (cycles):", statistics.median(per) if per else None)


def med(a, b):
    d = [r[1 + b] - r[1 + a] for r in rows if r[1 + a] and r[1 + b]]
    return statistics.median(d) if d else None


for a, b in pairs:
    print(f"{names[a]}->{names[b]}: {med(a, b)}")
