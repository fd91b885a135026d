"""Summarise an ncu source page (--page source --csv --print-source sass):
per-opcode executed warp-instructions and stall samples, plus the hottest
instructions.  python tools/sass_profile.py file.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def num(v):
    try:
        return float(v)
    except ValueError:
        return 0.0


by_op = collections.defaultdict(lambda: [0.0, 0.0])
tot_st = collections.Counter()
tot_exec = tot_samp = 0.0
for r in data:
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    ex = num(r[ix["Instructions Executed"]])
    sa = num(r[ix["Warp Stall Sampling (All Samples)"]])
    by_op[op][0] += ex
    by_op[op][1] += sa
    tot_exec += ex
    tot_samp += sa
    for c in stall_cols:
        tot_st[c] += num(r[ix[c]])
print(f"total warp-instructions executed {tot_exec:.3e}, stall samples {tot_samp:.0f}")
for op, (ex, sa) in sorted(by_op.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"  {op:10s} exec {ex:12.0f} ({100*ex/tot_exec:5.1f}%)  samples {sa:8.0f} ({100*sa/max(tot_samp,1):5.1f}%)")
print("stall reasons (all samples):")
for c, v in tot_st.most_common(12):
    print(f"  {c:28s} {v:8.0f} ({100*v/max(tot_samp,1):5.1f}%)")
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print("hottest instructions:")
hot = sorted(data, key=lambda r: -num(r[ix["Warp Stall Sampling (All Samples)"]]))[:top]
for r in hot:
    st = sorted(((num(r[ix[c]]), c) for c in stall_cols), reverse=True)[:3]
    print(f"  {r[ix['Address']][-5:]} {r[ix['Source']].strip()[:60]:60s} samp {r[ix['Warp Stall Sampling (All Samples)']]:>6s} "
          f"exec {r[ix['Instructions Executed']]:>9s} " + " ".join(f"{c[6:]}={v:.0f}" for v, c in st if v))
