"""Median per-iteration intervals of a kernel trace file (SPPO_TRACE output).
usage: python tools/trace_stats.py trace.txt [bwd|fwd]"""
import statistics
import sys

kind = sys.argv[2] if len(sys.argv) > 2 else "bwd"
if kind == "bwd":
    names = ["mma_pre", "dP", "dV", "S+1", "dK", "dQdone", "cP0", "pfull", "dpseen", "dsfull0", "cP1", "dsfull1",
             "rdq", "rfree", "r_end", "ldq"]
    pairs = [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (6, 7), (7, 8), (8, 9), (1, 8), (9, 4), (12, 13), (5, 12),
             (13, 14)]
    period_slot = 2
else:
    names = ["vfull", "PV0", "S0+1", "PV1", "S1+1", "s0seen", "s0max", "p0full", "s1seen", "s1max", "p1full",
             "ldK", "ldV", "-", "-", "-"]
    pairs = [(0, 1), (1, 2), (2, 3), (3, 4), (5, 6), (6, 7), (8, 9), (9, 10), (2, 5), (4, 8), (7, 1), (10, 3)]
    period_slot = 1
rows = [list(map(int, l.split()))[1:] for l in open(sys.argv[1])]
rows = rows[2:-2]


def med(a, b, nxt=False):
    v = [(rows[i + 1] if nxt else rows[i])[b] - rows[i][a] for i in range(len(rows) - 1) if rows[i][a] and rows[i][b]]
    return statistics.median(v) if v else None


print("period", med(period_slot, period_slot, True))
for a, b in pairs:
    print(f"{names[a]:>8} -> {names[b]:<8} {med(a, b)}")
# cross-iteration: S_t(n+1) issued (row n) -> s_t seen (row n+1)
for t, (si, ss) in enumerate([(2, 5), (4, 8)]):
    v = [rows[i + 1][ss] - rows[i][si] for i in range(len(rows) - 1) if rows[i][si] and rows[i + 1][ss]]
    if v:
        print(f"S{t}+1 issue -> s{t}seen(next) {statistics.median(v)}")
