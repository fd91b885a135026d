"""Group an ncu SASS source page into runs of equal execution count (basic
blocks, roughly) and print the ones holding the stall samples.
python tools/sass_regions.py file.csv [min_share]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
seen, d2 = set(), []
for r in rows[2:]:
    if len(r) != len(hdr) or not r[0].startswith("0x") or r[0] in seen:
        continue
    seen.add(r[0])
    d2.append(r)
d2.sort(key=lambda r: int(r[0], 16))
groups = []
for r in d2:
    ex = int(float(r[ix["Instructions Executed"]] or 0))
    sa = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    t = r[ix["Source"]].strip().split()
    op = (t[1] if t and t[0].startswith("@") else (t[0] if t else "?")).split(".")[0]
    if groups and groups[-1]["ex"] == ex:
        g = groups[-1]
        g["n"] += 1
        g["sa"] += sa
        g["ops"][op] = g["ops"].get(op, 0) + 1
        g["end"] = r[0]
    else:
        groups.append(dict(ex=ex, n=1, sa=sa, ops={op: 1}, start=r[0], end=r[0]))
tot = sum(g["sa"] for g in groups)
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.004
for g in groups:
    if g["sa"] > thr * tot:
        ops = sorted(g["ops"].items(), key=lambda kv: -kv[1])[:5]
        print(f"{g['start'][-5:]}-{g['end'][-5:]} exec {g['ex']:>10d} n {g['n']:4d} samp {100 * g['sa'] / tot:5.1f}%  {ops}")
