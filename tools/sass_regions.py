"""Group a tools/sass_profile.py listing into runs of equal execution count.

usage: python tools/sass_regions.py listing.txt [min_fraction]
"""
import sys

rows = []
for l in open(sys.argv[1]):
    if l.startswith('#'):
        continue
    p = l.split(None, 5)
    rows.append((p[0], int(p[1]), int(p[2]), p[5].strip() if len(p) > 5 else ""))
minf = float(sys.argv[2]) if len(sys.argv) > 2 else 0.004
grp = []
for r in rows:
    if grp and grp[-1][2] == r[2]:
        g = grp[-1]
        g[1] += r[1]
        g[3] += 1
        g[4] = r[0]
    else:
        grp.append([r[0], r[1], r[2], 1, r[0]])
tot = sum(r[2] for r in rows)
tots = sum(r[1] for r in rows)
for g in grp:
    if g[2] * g[3] > tot * minf or g[1] > tots * minf:
        print(f"{g[0]}-{g[4]} n={g[3]:4d} exec={g[2]:9d} instr={g[2]*g[3]/1e6:7.2f}M ({100*g[2]*g[3]/tot:4.1f}%) "
              f"samples={g[1]} ({100*g[1]/tots:4.1f}%)")
