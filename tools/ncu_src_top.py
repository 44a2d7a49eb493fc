"""Summarise an ncu --page source --csv --print-source sass export: top
instructions by shared-memory wavefronts and by stall samples.
  python tools/ncu_src_top.py file.csv [n]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[1]
recs = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]


def f(r, k):
    try:
        return float(r.get(k, 0) or 0)
    except ValueError:
        return 0.0


tot_w = sum(f(r, "L1 Wavefronts Shared") for r in recs)
tot_s = sum(f(r, "Warp Stall Sampling (All Samples)") for r in recs)
print(f"instructions {len(recs)}, shared wavefronts {tot_w:.3e}, stall samples {tot_s:.0f}")
print("--- top by L1 Wavefronts Shared")
for r in sorted(recs, key=lambda r: -f(r, "L1 Wavefronts Shared"))[:n]:
    print(f"{f(r, 'L1 Wavefronts Shared') / tot_w * 100:6.2f}%  ideal {f(r, 'L1 Wavefronts Shared Ideal'):.3e}  "
          f"exec {f(r, 'Instructions Executed'):.3e}  {r['Address'][-5:]} {r['Source'].strip()[:70]}")
print("--- top by stall samples")
stall_keys = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
for r in sorted(recs, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:n]:
    top = sorted(stall_keys, key=lambda k: -f(r, k))[:2]
    print(f"{f(r, 'Warp Stall Sampling (All Samples)') / tot_s * 100:6.2f}%  {r['Address'][-5:]} "
          f"{r['Source'].strip()[:60]:60s} {top[0][6:]}={f(r, top[0]):.0f} {top[1][6:]}={f(r, top[1]):.0f}")
