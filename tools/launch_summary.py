"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv
--log-file): launches, total / mean device time and share per kernel.
Usage: python tools/launch_summary.py launches.csv "<header line>" > out.txt"""
import collections
import csv
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
hdr, data = rows[0], rows[1:]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.OrderedDict()
for r in data:
    name = re.sub(r"^(void )?((sdr::)?<?unnamed>::|sdr::)", "", r[ik])
    m = re.match(r"([A-Za-z0-9_]+(?:<[^(]*>)?)", name)
    nm = m.group(1) if m else name[:60]
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[iu], 1e-3)
    a = agg.setdefault(nm, [0, 0.0])
    a[0] += 1
    a[1] += float(r[iv].replace(",", "")) * scale
tot = sum(a[1] for a in agg.values()) or 1.0
for h in sys.argv[2:]:
    print(h)
print("# kernel, launches, total_us, mean_us, share_of_kernel_time")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:64]:64s} {n:6d} {t:12.1f} {t / n:10.2f} {t / tot:8.3f}")
