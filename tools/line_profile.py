"""Per-source-line stall samples and instruction counts for one kernel of an ncu report.

Joins the report's SASS page (per-instruction samples, absolute addresses) with
nvdisasm line info of a -lineinfo cubin of the same source.
Usage: python tools/line_profile.py report.ncu-rep kernel_mangled_name_regex [cubin]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cubin = sys.argv[3] if len(sys.argv) > 3 else "/tmp/lp.cubin"
if len(sys.argv) <= 3:
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
                           "-cubin", "-o", cubin, os.path.join(ROOT, "paper_2108_12050_b200/csrc/mhfd.cu")])
dis = subprocess.run(["nvdisasm", "--print-line-info", "-fun", "dummy", cubin], capture_output=True, text=True)
dis = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True, text=True).stdout
# find the function section
funcs = re.split(r"\n\s*\.section\s+\.text\.", dis)
body = None
for f in funcs:
    name = f.split("\n", 1)[0].split(",")[0].strip()
    if re.search(kre, name):
        body = f
        break
if body is None:
    sys.exit("kernel not found in cubin")
off2line = {}
cur = None
for ln in body.split("\n"):
    m = re.search(r"line (\d+)", ln)
    if "//## File" in ln and m:
        fm = re.search(r'File "([^"]+)"', ln)
        cur = (os.path.basename(fm.group(1)) if fm else "?", int(m.group(1)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        off2line[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
iA, iE, iW = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
STALLS = ["stall_math", "stall_wait", "stall_not_selected", "stall_selected", "stall_short_sb", "stall_barrier",
          "stall_long_sb", "stall_dispatch", "stall_mio", "stall_branch_resolving"]
iS = {k: hdr.index(k) for k in STALLS if k in hdr}
data = [r for r in rows[2:] if len(r) > iW and r[iA].startswith("0x")]
base = int(data[0][iA], 16)
agg_s, agg_e = collections.Counter(), collections.Counter()
agg_r = collections.defaultdict(collections.Counter)
tot = 0
for r in data:
    off = int(r[iA], 16) - base
    key = off2line.get(off, ("?", 0))
    w = int(r[iW]) if r[iW].isdigit() else 0
    e = int(r[iE]) if r[iE].isdigit() else 0
    agg_s[key] += w
    agg_e[key] += e
    for k, i in iS.items():
        agg_r[key][k] += int(r[i]) if r[i].isdigit() else 0
    tot += w
src_cache = {}
print(f"total samples {tot}")
for key, w in agg_s.most_common(int(os.environ.get("TOPN", "30"))):
    fn, line = key
    text = ""
    for cand in (os.path.join(ROOT, "paper_2108_12050_b200/csrc", fn),):
        if os.path.exists(cand):
            src_cache.setdefault(cand, open(cand).read().split("\n"))
            text = src_cache[cand][line - 1].strip()[:80] if 0 < line <= len(src_cache[cand]) else ""
    br = " ".join(f"{k[6:10]}={v * 100 // max(w, 1)}" for k, v in agg_r[key].most_common(4) if v)
    print(f"{w / max(tot, 1) * 100:5.1f}%  {agg_e[key]:>12d}  {fn}:{line}  {text[:56]:56s} [{br}]")
