"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: launches, mean
duration and share of the summed time per kernel (cold-cache serialised: compare shares)."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    if r[mi] == "gpu__time_duration.sum":
        v = float(r[vi].replace(",", ""))
        tot[r[ki]] += v
        cnt[r[ki]] += 1
S = sum(tot.values()) or 1
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k[:70]:70s} n={cnt[k]:3d} mean={tot[k] / cnt[k] / 1e3:9.3f} us share={100 * tot[k] / S:5.1f}%")
