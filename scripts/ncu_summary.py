"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import csv, sys, collections, re
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value"); mi = hdr.index("Metric Name")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum": continue
    name = re.sub(r"\(.*", "", r[ki])[:90]
    v = float(r[vi].replace(",", ""))
    agg[name][0] += 1; agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"total {tot/1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches (unit: ns -> ms)")
for k, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{v/1e6:9.3f} ms {100*v/tot:5.1f}%  n={n:5d}  {k}")
