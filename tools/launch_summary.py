"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    name = d["Kernel Name"].split("(")[0][:70]
    agg[name][0] += 1
    agg[name][1] += float(d["Metric Value"])
tot = sum(v[1] for v in agg.values())
print(f"{len(data)} launches, {tot/1e3:.1f} us total")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:5d} {t/1e3:10.1f} us total {t/n/1e3:8.2f} us avg {100*t/tot:5.1f}%  {k}")
