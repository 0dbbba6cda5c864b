"""Summarise an ncu report's SASS page: instruction mix and stall samples per opcode,
plus the hottest instructions.  Usage: python tools/sass_hist.py report.ncu-rep [kernel-regex]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"]
if len(sys.argv) > 2:
    cmd += ["-k", "regex:" + sys.argv[2]]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
iA, iS = hdr.index("Address"), hdr.index("Source")
iE, iW = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
op, st = collections.Counter(), collections.Counter()
tot = stt = 0
for r in data:
    try:
        e, w = int(r[iE]), int(r[iW])
    except (ValueError, IndexError):
        continue
    t = r[iS].split()
    o = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    op[o] += e
    st[o] += w
    tot += e
    stt += w
print(f"total warp instructions {tot}  stall samples {stt}")
for o, c in op.most_common(18):
    print(f"{o:10s} {c / tot * 100:6.2f}% instr  {st[o] / max(stt, 1) * 100:6.2f}% stall samples")
hot = sorted(((int(r[iW]) if r[iW].isdigit() else 0, r[iA][-5:], r[iS].strip()[:64], r[iE]) for r in data),
             reverse=True)
print("hottest:")
for h in hot[:14]:
    print(*h)
