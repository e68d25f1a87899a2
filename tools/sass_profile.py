"""Condense an ncu source page (SASS view) into addr/instr/samples/executed columns.

usage: python tools/sass_profile.py report.ncu-rep [profiled-kernel-index] > out.txt
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
txt = subprocess.run(cmd, capture_output=True, text=True).stdout
lines = txt.splitlines()
which = int(sys.argv[2]) if len(sys.argv) > 2 else 0
blocks, cur = [], None
for l in lines:
    if l.startswith('"Kernel Name"'):
        cur = []
        blocks.append(cur)
    elif cur is not None:
        cur.append(l)
rows = list(csv.reader(io.StringIO("\n".join(blocks[which]))))
hdr = rows[0]
ia = hdr.index("Address"); isrc = hdr.index("Source"); ism = hdr.index("Warp Stall Sampling (All Samples)")
iex = hdr.index("Instructions Executed"); iwf = hdr.index("L1 Wavefronts Shared"); iwi = hdr.index("L1 Wavefronts Shared Ideal")
tot_s = sum(int(r[ism] or 0) for r in rows[1:] if r[0] != "Address")
tot_e = sum(int(r[iex] or 0) for r in rows[1:] if r[0] != "Address")
print(f"# total samples {tot_s} executed {tot_e}")
for r in rows[1:]:
    if r[0] == "Address":
        continue
    print(f"{r[ia][-5:]} {int(r[ism] or 0):6d} {int(r[iex] or 0):10d} {r[iwf]:>8} {r[iwi]:>8}  {r[isrc].strip()}")
