"""Top stall sites of an ncu --set full --import-source report (source page, SASS): python tools/ncu_source_top.py REP [N]."""
import csv, subprocess, sys, io
rep = sys.argv[1]; ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]; data = rows[2:]
ix = {k: i for i, k in enumerate(h)}
S = 'Warp Stall Sampling (All Samples)'
tot = sum(int(r[ix[S]] or 0) for r in data)
cols = [c for c in h if c.startswith('stall_') and '(Not' not in c]
agg = {c: sum(int(r[ix[c]] or 0) for r in data) for c in cols}
print('total samples', tot, sorted(((v, c) for c, v in agg.items()), reverse=True)[:8])
ex = 'Instructions Executed'
tot_ex = sum(int(r[ix[ex]] or 0) for r in data)
mufu = sum(int(r[ix[ex]] or 0) for r in data if 'MUFU' in r[1])
print('executed warp instr', tot_ex, 'MUFU', mufu, 'per MUFU', tot_ex / max(mufu, 1))
top = sorted(data, key=lambda r: -int(r[ix[S]] or 0))[:ntop]
for r in top:
    s = int(r[ix[S]] or 0)
    st = sorted(((int(r[ix[c]] or 0), c[6:]) for c in cols), reverse=True)[:3]
    print(f"{r[0][-5:]} {s:6d} {100*s/tot:5.1f}% {r[1][:50]:50s} {st}")
