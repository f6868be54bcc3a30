"""Average time per kernel name of an ncu --metrics gpu__time_duration.sum
CSV launch list: python scripts/launch_avg.py gpurun_out/x.csv [regex]"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[hdr + 1:]:
    if len(r) <= vi or not r[vi]:
        continue
    name = r[ki].split("(")[0][:70]
    if pat and not pat.search(name):
        continue
    t = float(r[vi].replace(",", ""))
    t *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(r[ui], 1e-3)
    tot[name] += t
    cnt[name] += 1
for name in sorted(tot, key=lambda n: -tot[n]):
    print(f"{tot[name] / cnt[name]:10.1f} us avg  x{cnt[name]:<4d} {name}")
