"""Per-kernel totals and shares from an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        k = d["Kernel Name"].split("(")[0].replace("void ", "")[:70]
        v = float(d["Metric Value"].replace(",", ""))
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':70s} {'launches':>8s} {'total_us':>12s} {'avg_us':>10s} {'share':>7s}")
for k, (c, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:70s} {c:8d} {s / 1e3:12.1f} {s / 1e3 / c:10.2f} {100 * s / tot:6.2f}%")
print(f"total {tot / 1e3:.1f} us over {sum(v[0] for v in agg.values())} launches")
