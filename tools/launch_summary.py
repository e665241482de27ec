"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel:
python tools/launch_summary.py launches.csv out.txt"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
kn, mv, mn, mu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name"), h.index("Metric Unit")
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= mv or r[mn] != "gpu__time_duration.sum":
        continue
    v = float(r[mv].replace(",", ""))
    us = {"ns": v / 1e3, "us": v, "ms": v * 1e3}.get(r[mu], v)
    a = agg.setdefault(r[kn].split("(")[0], [0, 0.0])
    a[0] += 1
    a[1] += us
tot = sum(a[1] for a in agg.values())
out = ["# Launch list of `ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 2 --warmup 3 --no-cpu`",
       "# cold-cache, serialised per-launch times (ncu); shares of the summed device time", ""]
for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    out.append(f"{n:60s} launches {c:4d}  mean {t / c:12.1f} us  total {t:12.1f} us  share {100 * t / tot:6.2f} %")
open(sys.argv[2], "w").write("\n".join(out) + "\n")
