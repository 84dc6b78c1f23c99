"""Warp-stall samples of one kernel aggregated by CUDA source line.

    ncu -i prof.ncu-rep --page source --csv -k regex:<kernel> > sass.csv
    python tools/stall_lines.py sass.csv <lib.so> <cubin name> <mangled kernel> [N]

Maps each SASS address of the ncu source page to its file:line with
``nvdisasm -g`` on the same build of the library (compiled with -lineinfo).
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

sass_csv, lib, cubin, kern = sys.argv[1:5]
lib = os.path.abspath(lib)
top = int(sys.argv[5]) if len(sys.argv) > 5 else 30
# optional 6th argument: another per-instruction column to aggregate, e.g.
# "Instructions Executed" (default: the warp-stall samples)
column = sys.argv[6] if len(sys.argv) > 6 else "Warp Stall Sampling (All Samples)"
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", cubin, lib], cwd=tmp, check=True, capture_output=True)
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cubin)], capture_output=True,
                     text=True).stdout.split("\n")
start = next(i for i, ln in enumerate(dis) if f".text.{kern}" in ln)
cur, a2l = None, {}
for ln in dis[start + 1:]:
    if ln.startswith("//---------------------"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        a2l[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(sass_csv)))
hdr, data = rows[1], rows[2:]
ia, iss = hdr.index("Address"), hdr.index(column)
base = int(data[0][ia], 16)
agg, tot = collections.Counter(), 0
for r in data:
    try:
        s = int(float(r[iss]))
    except (ValueError, IndexError):
        continue
    agg[a2l.get(int(r[ia], 16) - base, ("?", 0))] += s
    tot += s
srcdir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2109_01158_b200", "csrc")
print("| samples | share | line | source |")
print("|---|---|---|---|")
for (f, ln), s in agg.most_common(top):
    p = os.path.join(srcdir, f)
    txt = open(p).read().split("\n")[ln - 1].strip()[:80] if os.path.exists(p) and ln else ""
    txt = txt.replace("|", "\\|")
    print(f"| {s} | {100 * s / tot:.1f}% | {f}:{ln} | `{txt}` |")
