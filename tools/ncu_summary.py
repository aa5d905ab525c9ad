"""Summarise an ncu launch list (``--metrics gpu__time_duration.sum --csv``) per kernel.

    python tools/ncu_summary.py gpurun_out/launches.csv > profiles/r01_launches.md
"""

import csv
import re
import sys
from collections import OrderedDict


def short(name):
    name = re.sub(r"\(.*", "", name)
    return name.replace("redve::", "")


def main(path):
    rows = []
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        rows.append((short(r["Kernel Name"]), float(r["Metric Value"]), r["Grid Size"],
                     r["Block Size"]))
    agg = OrderedDict()
    for k, ns, g, b in rows:
        a = agg.setdefault(k, [0, 0.0, g, b])
        a[0] += 1
        a[1] += ns
    total = sum(v[1] for v in agg.values())
    print(f"launches: {len(rows)}, total device time {total / 1e6:.3f} ms (serialised, cold-cache)\n")
    print("| kernel | launches | total ms | avg us | share | grid | block |")
    print("|---|---|---|---|---|---|---|")
    for k, (n, ns, g, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {k} | {n} | {ns / 1e6:.3f} | {ns / n / 1e3:.1f} | {100 * ns / total:.1f}% | {g} | {b} |")


if __name__ == "__main__":
    main(sys.argv[1])
