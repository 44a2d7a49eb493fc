"""Median per-iteration intervals of a bwd trace file (SPPO_TRACE output)."""
import statistics
import sys

names = ["mma_pre", "dP", "dV", "S+1", "dK", "dQdone", "cP0", "pfull", "dpseen", "dsfull0", "cP1", "dsfull1",
         "rdq", "rfree", "r_end", "ldq"]
rows = [list(map(int, l.split()))[1:] for l in open(sys.argv[1])]
rows = rows[2:-2]
def med(a, b, nxt=False):
    v = [(rows[i + 1] if nxt else rows[i])[b] - rows[i][a] for i in range(len(rows) - 1) if rows[i][a] and rows[i][b]]
    return statistics.median(v) if v else None
print("period", med(2, 2, True))
for a, b in [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (6, 7), (7, 8), (8, 9), (1, 8), (9, 4), (12, 13), (5, 12), (13, 14)]:
    print(f"{names[a]:>8} -> {names[b]:<8} {med(a, b)}")
