"""Stall samples along the SASS of one kernel in an ncu report (source page).

python tools/ncu_sass_hot.py report.ncu-rep kernel_regex"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--kernel-name",
                      f"regex:{sys.argv[2]}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if "Source" in r and "Address" in r)
data = [r for r in rows if len(r) == len(hdr) and r[0].startswith("0x")]
S = hdr.index("Warp Stall Sampling (All Samples)")
src = hdr.index("Source")


def g(r, k):
    v = r[hdr.index(k)]
    try:
        return int(float(v))
    except ValueError:
        return 0


tot = sum(g(r, hdr[S]) for r in data)
print("total samples", tot, "instructions", len(data))
seg = max(1, len(data) // 16)
for s in range(0, len(data), seg):
    ch = data[s:s + seg]
    n = sum(g(r, hdr[S]) for r in ch)
    print(f"{s:5d} {n:6d} ({n / max(tot, 1):5.1%}) long_sb {sum(g(r, 'stall_long_sb') for r in ch):5d} "
          f"barrier {sum(g(r, 'stall_barrier') for r in ch):5d} short_sb {sum(g(r, 'stall_short_sb') for r in ch):5d}"
          f"  | {ch[0][src].strip()[:50]}")
print("-- hottest")
for k in sorted(range(len(data)), key=lambda k: -g(data[k], hdr[S]))[:20]:
    r = data[k]
    print(f"{k:5d} {g(r, hdr[S]):5d} long_sb {g(r, 'stall_long_sb'):4d} bar {g(r, 'stall_barrier'):4d} | {r[src].strip()[:70]}")
