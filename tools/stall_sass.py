"""Top warp-stall SASS instructions of one kernel from an ncu source-page CSV,
with their dominant stall reasons and the preceding instructions (context).

    ncu -i prof.ncu-rep --page source --csv -k regex:<kernel> > sass.csv
    python tools/stall_sass.py sass.csv [N]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
hdr, data = rows[1], rows[2:]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iss = hdr.index("Warp Stall Sampling (All Samples)")
seen, first = set(), []
for r in data:  # the first captured launch only
    if r[0] in seen or len(r) <= max(ia if False else 0, 2) or r[0] in ("Kernel Name", "Address"):
        break
    seen.add(r[0])
    first.append(r)
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[iss]) for r in first if r[iss].isdigit())
order = sorted(range(len(first)), key=lambda i: -int(first[i][iss] or 0))
print("| share | instruction | top stall reasons | preceded by |")
print("|---|---|---|---|")
for i in order[:top_n]:
    r = first[i]
    br = sorted(((h[6:], int(r[hdr.index(h)])) for h in reasons if r[hdr.index(h)].isdigit()),
                key=lambda t: -t[1])[:2]
    ctx = " ; ".join(first[j][isrc].strip()[:38] for j in range(max(0, i - 3), i))
    print(f"| {int(r[iss]) / tot * 100:.1f}% | `{r[isrc].strip()[:40]}` | "
          f"{', '.join(f'{k} {v}' for k, v in br)} | `{ctx}` |")
