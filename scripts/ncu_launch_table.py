"""Tabulate an ncu --csv launch list: one line per launch with its metrics."""
import csv, sys
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines)); hdr = rows[0]; idx = {h: i for i, h in enumerate(hdr)}
out = {}
for r in rows[1:]:
    key = (int(r[idx["ID"]]), r[idx["Kernel Name"]].split("(")[0].split("::")[-1])
    out.setdefault(key, {})[r[idx["Metric Name"]]] = r[idx["Metric Value"]]
tot = {}
for (i, k), v in sorted(out.items()):
    t = float(v.get("gpu__time_duration.sum", "0").replace(",", ""))
    tot[k] = tot.get(k, 0.0) + t
    if len(sys.argv) > 2:
        print(i, k, *v.values())
for k, t in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:40s} {t/1e6:9.3f} ms")
