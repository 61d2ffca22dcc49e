"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h, data = rows[0], rows[1:]
ik, iv, iu, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Metric Name")
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in data:
    if r[im] != "gpu__time_duration.sum":
        continue
    k = r[ik].split("(")[0][:70]
    agg[k][0] += 1
    agg[k][1] += float(r[iv].replace(",", "")) * scale[r[iu]]
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':70s} {'launches':>8s} {'total ms':>10s} {'share':>6s} {'avg ms':>9s}")
for k, (c, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:70s} {c:8d} {ms:10.2f} {100 * ms / tot:5.1f}% {ms / c:9.3f}")
