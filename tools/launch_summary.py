"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel count, time, share."""
import csv, sys
lines = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
h = rows[0]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
tot = {}
for r in rows[1:]:
    k = r[ik].split("(")[0]
    t = tot.setdefault(k, [0, 0.0])
    t[0] += 1
    t[1] += float(r[iv].replace(",", ""))
s = sum(v[1] for v in tot.values())
print(f"# {sys.argv[2] if len(sys.argv) > 2 else ''}")
for k, (n, t) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print(f"{n:4d} launches  {t / 1e6:10.3f} ms  {100 * t / s:6.2f}%  {k}")
