"""Summarise an ncu --csv launch list (gpu__time_duration.sum): time per kernel name and largest launches."""
import csv, sys, collections
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.DictReader(lines))
agg = collections.defaultdict(lambda: [0, 0.0])
launches = []
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0]
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "nsecond")
    us = v / 1e3 if unit.startswith("n") else (v if unit.startswith("u") else (v * 1e3 if unit.startswith("m") else v * 1e6))
    agg[name][0] += 1
    agg[name][1] += us
    launches.append((us, name, r.get("ID"), r.get("Grid Size", "")))
tot = sum(v[1] for v in agg.values())
print(f"total {tot/1e3:.2f} ms over {sum(v[0] for v in agg.values())} launches")
for k, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:40s} {c:6d} launches {us/1e3:9.2f} ms {100*us/tot:5.1f}%")
print("largest launches:")
for us, name, i, g in sorted(launches, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"  {us/1e3:8.3f} ms  {name} id={i} grid={g}")
