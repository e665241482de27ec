"""Executed-instruction mix per MUFU op of an ncu report (source page): python tools/ncu_opmix.py REP."""
import csv, subprocess, sys, io, collections
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]; data = rows[2:]
ix = {k: i for i, k in enumerate(h)}
c = collections.Counter()
for r in data:
    op = r[1].split()
    if not op: continue
    o = op[0] if not op[0].startswith('@') else op[1]
    c[o.split('.')[0]] += int(r[ix['Instructions Executed']] or 0)
tot = sum(c.values()); mufu = c['MUFU']
for k, v in c.most_common(25): print(f"{k:10s} {v:10d} {v/mufu:6.2f} per MUFU")
print('total', tot, tot/mufu)
