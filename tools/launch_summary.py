"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list per kernel."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, {}
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[hdr.index("Metric Name")] == "gpu__time_duration.sum":
        k = r[hdr.index("Kernel Name")].split("(")[0]
        v = float(r[hdr.index("Metric Value")].replace(",", ""))
        u = r[hdr.index("Metric Unit")]
        v = v / 1e3 if u in ("nsecond", "ns") else (v * 1e3 if u in ("msecond", "ms") else v)
        a = agg.setdefault(k, [0.0, 0])
        a[0] += v
        a[1] += 1
tot = sum(t for t, _ in agg.values())
for k, (t, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{k[:60]:60s} n={c:4d} total={t:10.1f}us avg={t / c:9.1f}us share={t / tot:6.1%}")
