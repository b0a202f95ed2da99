"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]) by kernel name."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
idi = hdr.index("ID")
per = defaultdict(dict)
names = {}
for r in rows[hdr_i + 1:]:
    if len(r) <= vi:
        continue
    per[r[idi]][r[mi]] = float(r[vi].replace(",", ""))
    names[r[idi]] = r[ki]
agg = defaultdict(lambda: [0, 0.0, 0.0])
for i, m in per.items():
    n = names[i][:70]
    a = agg[n]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0) / 1e3
    a[2] += (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / 1e6
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':70s} {'n':>4s} {'total us':>9s} {'share':>6s} {'us/launch':>9s} {'MB/launch':>9s}")
for n, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:70s} {a[0]:4d} {a[1]:9.1f} {a[1] / tot * 100:5.1f}% {a[1] / a[0]:9.2f} {a[2] / a[0]:9.1f}")
print(f"sum {tot:.1f} us")
