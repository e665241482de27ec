"""Analyse one launch of the -DFASTRON_GRAM_PROF Gram build: per-unit start / end (globaltimer)."""
import collections, re, sys
lines = [l for l in open(sys.argv[1]) if l.startswith("gram prof")]
launches, units = [], {}
for l in lines:
    m = re.match(r"gram prof unit (\d+) sm (\d+) start (\d+) first-tile (\d+) end (\d+) rows (\d+) cols (\d+)", l)
    u = int(m.group(1))
    if u in units:
        launches.append(units)
        units = {}
    units[u] = tuple(int(m.group(i)) for i in range(2, 8))
launches.append(units)
units = launches[-2] if len(launches) > 1 else launches[-1]  # a steady-state launch
t0 = min(v[1] for v in units.values())
ends = sorted(v[3] - t0 for v in units.values())
starts = sorted(v[1] - t0 for v in units.values())
per_sm = collections.Counter(v[0] for v in units.values())
print("units", len(units), "sms used", len(per_sm), "ctas/sm histogram", sorted(collections.Counter(per_sm.values()).items()))
print("start ns: min", starts[0], "p50", starts[len(starts) // 2], "p90", starts[int(len(starts) * .9)], "max", starts[-1])
print("end ns:   min", ends[0], "p50", ends[len(ends) // 2], "p90", ends[int(len(ends) * .9)], "max", ends[-1])
print("first-tile ns p50", sorted(v[2] for v in units.values())[len(units) // 2],
      "cols-landed ns p50", sorted(v[5] for v in units.values())[len(units) // 2],
      "max", max(v[5] for v in units.values()))
late = sorted(units.items(), key=lambda kv: -kv[1][3])[:5]
for u, v in late:
    print("late unit", u, "sm", v[0], "start", v[1] - t0, "end", v[3] - t0, "rows", v[4])
