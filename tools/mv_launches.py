"""Per-launch time / DRAM bytes / GB/s of the first matvec in an ncu csv (tools/mv_bench.py run)."""
import csv, sys
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
d = {}
for r in csv.DictReader(lines):
    d.setdefault(r['ID'], {'name': r['Kernel Name'][:22], 'grid': r['Grid Size']})[r['Metric Name']] = \
        float(r['Metric Value'].replace(',', ''))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
tot = 0.0
for i in sorted(d, key=int)[:n]:
    x = d[i]; t = x.get('gpu__time_duration.sum', 0); b = x.get('dram__bytes_read.sum', 0); tot += t
    print(i, x['name'], x['grid'], f"{t/1e3:.1f}us", f"{b/1e6:.1f}MB", f"{b/t if t else 0:.0f} GB/s")
print(f"total {tot/1e3:.1f} us")
