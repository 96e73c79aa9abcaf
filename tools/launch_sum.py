"""Sum an ncu --csv gpu__time_duration launch list by kernel (tools/, not product)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
i = next(j for j, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[i]
kn, mv, mu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[i + 1:]:
    if len(r) <= mv:
        continue
    v = float(r[mv].replace(",", ""))
    unit = r[mu]
    v = v / 1e3 if unit in ("nsecond", "ns") else (v if unit in ("usecond", "us") else v * 1e3)
    name = r[kn].split("(")[0]
    tot[name] += v
    cnt[name] += 1
s = sum(tot.values())
print(f"total {s / 1e3:.3f} ms over {sum(cnt.values())} launches")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:25]:
    print(f"{v / 1e3:9.3f} ms {cnt[k]:6d} x {v / cnt[k]:8.2f} us  {k}")
