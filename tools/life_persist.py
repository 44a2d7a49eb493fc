"""Per-CTA lifetime of a persistent bwd launch (SPPO_TRACE_LIFE=1, -DSPPO_BWD_LIFE=1
build): the spread of CTA end times (load imbalance of the item schedule) and the
effective cycles per Q tile including item boundaries.
  python tools/life_persist.py <file>"""
import statistics
import sys

rows = [list(map(int, l.split())) for l in open(sys.argv[1])]
ends, starts, per_tile, loops = [], [], [], []
for r in rows:
    s = r[1:]
    tiles = s[7] >> 32
    if not s[0] or not s[6] or not tiles:
        continue
    starts.append(s[0]); ends.append(s[6])
    loops.append(s[3] - s[2] if s[3] and s[2] else 0)
    per_tile.append((s[6] - s[0]) / tiles)
life = [e - b for b, e in zip(starts, ends)]
print(f"ctas {len(life)}  lifetime median {statistics.median(life):.0f}  min {min(life)}  max {max(life)}  "
      f"(max/median {max(life) / statistics.median(life):.3f})")
print(f"cycles per tile incl. boundaries: median {statistics.median(per_tile):.0f}  min {min(per_tile):.0f}  max {max(per_tile):.0f}")
