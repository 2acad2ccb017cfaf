"""Summarise an `ncu --metrics gpu__time_duration.sum,dram__bytes_* --csv` launch list."""
import csv
import re
import sys
from collections import OrderedDict, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
d = OrderedDict()
for r in rows[start + 1:]:
    d.setdefault(int(r[ii]), {"k": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
agg = defaultdict(lambda: [0, 0.0, 0.0])
for v in d.values():
    name = re.sub(r"\(.*", "", v["k"]).replace("(anonymous namespace)::", "").replace("sdb::", "")
    name = name.replace("void ", "").replace("unnamed>::", "")
    a = agg[name]
    a[0] += 1
    a[1] += v.get("gpu__time_duration.sum", 0)
    a[2] += v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)
tot = sum(a[1] for a in agg.values())
print(f"{len(d)} kernels, {tot / 1000:.1f} us total (serialised, ncu)")
for n, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n[:44]:44s} n={a[0]:4d} total={a[1] / 1000:8.1f}us avg={a[1] / a[0] / 1000:7.2f}us "
          f"share={a[1] / tot:.3f} dram={a[2] / max(a[1], 1):.0f} GB/s")
