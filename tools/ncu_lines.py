"""Aggregate ncu source-page stall samples per CUDA source line.

    ncu -i rep --page source --csv --kernel-name regex:K --launch-count 1 --print-source cuda,sass > x.csv
    python tools/ncu_lines.py x.csv [top]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
per_line = collections.Counter()
text = {}
cur_line = None
hdr = None
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5:
        continue
    if r[0]:
        cur_line = int(r[0]) if r[0].isdigit() else cur_line
        text[cur_line] = r[1]
    try:
        v = float(r[4] or 0)
    except ValueError:
        continue
    per_line[cur_line] += v
tot = sum(per_line.values()) or 1
for ln, v in per_line.most_common(top):
    print(f"{v:9.0f} {100 * v / tot:5.1f}%  L{ln}: {text.get(ln, '')[:110]}")
