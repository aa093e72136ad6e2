"""Aggregate an ncu --metrics gpu__time_duration.sum launch list (csv) per kernel."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h, data = None, []
for r in rows:
    if "Kernel Name" in r and "Metric Value" in r:
        h = r
        continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            v = float(d["Metric Value"].replace(",", ""))
            data.append((d["Kernel Name"][:60], v * {"nsecond": 1e-3, "ns": 1e-3, "msecond": 1e3, "ms": 1e3}.get(d.get("Metric Unit"), 1.0)))
agg = collections.OrderedDict()
for n, v in data:
    a = agg.setdefault(n, [0, 0.0])
    a[0] += 1
    a[1] += v
print(f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'avg_us':>10s}")
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:60s} {c:8d} {t:12.1f} {t / c:10.1f}")
