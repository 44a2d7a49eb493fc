"""Item-boundary view of a persistent bwd trace (SPPO_TRACE, CTA 0's first 512
tiles): per-tile period (dP issue to dP issue) and event offsets for the tiles
around each change of item (a jump in the tile period marks the boundary).
  python tools/trace_boundary.py <trace file> <tiles per item>"""
import statistics
import sys

rows = [list(map(int, l.split())) for l in open(sys.argv[1])]
M = int(sys.argv[2])
t = {r[0]: r[1:] for r in rows}
names = ["mma_top", "dP", "dV", "S+1", "dK", "dKdone", "cS0", "pfull", "dpseen", "dsfull0", "cS1", "dsfull1",
         "rdq", "rfree", "r_end", "lse"]
per = [t[i + 1][1] - t[i][1] for i in range(len(rows) - 1) if i in t and i + 1 in t]
print("median period", statistics.median(per))
for b in range(M, len(rows) - 2, M):
    seg = [t[i + 1][1] - t[i][1] for i in range(b - 2, b + 4) if i in t and i + 1 in t]
    print(f"boundary at tile {b}: periods around it {seg}  excess {sum(seg) - len(seg) * statistics.median(per)}")
b = M
for i in range(b - 1, b + 2):
    r = t[i]
    print(i, " ".join(f"{n}={r[k] - t[b - 1][1]}" for k, n in enumerate(names) if r[k]))
