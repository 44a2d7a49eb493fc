"""Per-CTA lifetime statistics of one bwd launch (SPPO_TRACE_LIFE=1 with a
-DSPPO_BWD_LIFE=1 build; stamps in kernels_sm100_bwd.cu, layout in internal.h).
Prints the median phase durations of a CTA (cycles), the per-tile period and the
share of SM time outside the Q-tile loop (setup, pipeline fill, drain, epilogue,
teardown, gaps between consecutive CTAs on an SM).
  python tools/life_stats.py <file> [json]"""
import collections
import json
import statistics
import sys

rows = [list(map(int, l.split())) for l in open(sys.argv[1])]
ctas = [r[1:] for r in rows]
ph = collections.defaultdict(list)
by_sm = collections.defaultdict(list)
for s in ctas:
    sm, M = s[7] & 0xffffffff, s[7] >> 32
    if not all(s[:7]) or M == 0:
        continue
    by_sm[sm].append(s)
    ph["setup"].append(s[1] - s[0])
    ph["to_first_S"].append(s[2] - s[1])
    ph["loop"].append(s[3] - s[2])
    ph["period"].append((s[3] - s[2]) / M)
    ph["drain"].append(s[4] - s[3])
    ph["epilogue"].append(s[5] - s[4])
    ph["teardown"].append(s[6] - s[5])
    ph["lifetime"].append(s[6] - s[0])
    ph["M"].append(M)
gaps, busy_loop, span = [], 0, 0
for sm, lst in by_sm.items():
    lst.sort(key=lambda s: s[0])
    span += lst[-1][6] - lst[0][0]
    busy_loop += sum(s[3] - s[2] for s in lst)
    gaps += [b[0] - a[6] for a, b in zip(lst, lst[1:])]
out = {k: round(statistics.median(v), 1) for k, v in ph.items()}
out["gap_between_ctas"] = round(statistics.median(gaps), 1) if gaps else None
out["ctas"] = len(ph["M"])
out["sms"] = len(by_sm)
out["loop_share_of_sm_time"] = round(busy_loop / span, 4) if span else None
out["non_loop_cycles_per_cta"] = round((span - busy_loop) / max(1, len(ph["M"])) * len(by_sm) / len(by_sm), 1)
print(json.dumps(out) if len(sys.argv) > 2 else "\n".join(f"{k:24s} {v}" for k, v in out.items()))
