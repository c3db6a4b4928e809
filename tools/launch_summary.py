"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv) per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
tail = int(sys.argv[2]) if len(sys.argv) > 2 else len(data)
sel = data[-tail:] if tail else data
agg = collections.defaultdict(lambda: [0, 0.0])
for d in sel:
    k = d["Kernel Name"].split("(")[0][:50]
    agg[k][0] += 1
    agg[k][1] += float(d["Metric Value"])
tot = sum(v[1] for v in agg.values())
print(f"{len(sel)} launches, total {tot/1e3:.1f} us (ns units: {sel[0]['Metric Unit']})")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {k:50s} n={v[0]:5d} total={v[1]/1e3:10.1f}us avg={v[1]/v[0]/1e3:9.2f}us share={v[1]/tot:.3f}")
