"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel total time, share and launch count (profiles/*launches*.txt)."""
import collections
import csv
import sys

rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
hdr = rows[0]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.defaultdict(lambda: [0.0, 0])
for r in rows[1:]:
    v = float(r[iv].replace(",", ""))
    u = r[iu]
    v = v / 1000 if u in ("ns", "nsecond") else (v * 1000 if u in ("ms", "msecond") else v)
    agg[r[ik]][0] += v
    agg[r[ik]][1] += 1
tot = sum(a[0] for a in agg.values())
n = sum(a[1] for a in agg.values())
if len(sys.argv) > 2:
    print("# " + sys.argv[2])
print(f"# {n} launches, sum {tot:.0f} us; per-kernel share of serialized device time")
for k, (t, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{t:12.1f} us {100 * t / tot:5.1f}%  {c:5d}x  {t / c:9.1f} us/launch  {k[:90]}")
