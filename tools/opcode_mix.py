"""Executed-instruction mix of one kernel from an ncu source page.

    ncu -i prof.ncu-rep --page source --csv -k regex:<kernel> > sass.csv
    python tools/opcode_mix.py sass.csv [elements]

Sums "Instructions Executed" (warp level) by SASS opcode; with the element
count also prints thread-level instructions per element."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
n_el = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
hdr, data = rows[1], rows[2:]
i_src, i_ex = hdr.index("Source"), hdr.index("Instructions Executed")
i_th = hdr.index("Thread Instructions Executed")
agg, th = collections.Counter(), collections.Counter()
seen = set()  # a report with several launches of the kernel lists each address once per launch
i_ad = hdr.index("Address")
for r in data:
    if len(r) <= max(i_src, i_ex, i_th) or r[i_ad] in seen:
        continue
    seen.add(r[i_ad])
    try:
        ex, t = float(r[i_ex] or 0), float(r[i_th] or 0)
    except ValueError:
        continue
    m = re.match(r"\s*(?:@!?U?P\w+\s+)?([A-Z0-9_]+)((?:\.[A-Z0-9_]+)*)", r[i_src])
    if not m:
        continue
    op = m.group(1)
    if op == "IMAD" and ".MOV" in m.group(2):
        op = "IMAD.MOV"
    agg[op] += ex
    th[op] += t
tot, tth = sum(agg.values()), sum(th.values())
print(f"warp instructions {tot / 1e6:.1f} M, thread instructions {tth / 1e9:.2f} G"
      + (f", {tth / n_el:.0f} per element" if n_el else ""))
for op, c in agg.most_common(30):
    line = f"{op:12s} {c / 1e6:9.2f} M  {100 * c / tot:5.1f} %"
    if n_el:
        line += f"  {th[op] / n_el:7.1f} per element"
    print(line)
