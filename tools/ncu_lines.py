"""Per-source-line warp-stall samples of one kernel in an ncu report (needs -lineinfo builds).
usage: python tools/ncu_lines.py report.ncu-rep kernel_regex [launch_skip] [top]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kern}", "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
lines = [l for l in out.splitlines() if l.startswith('"')]
rows = list(csv.reader(io.StringIO("\n".join(lines))))
hdr = next(r for r in rows if r and r[0] == "Line No")
si = hdr.index("Warp Stall Sampling (All Samples)")
ei = hdr.index("Instructions Executed")
data = []
for r in rows:
    if r and r[0].isdigit():
        try:
            data.append((int(r[si] or 0), int(r[ei] or 0), int(r[0]), r[1][:100]))
        except ValueError:
            pass
tot = sum(d[0] for d in data) or 1
print(f"{kern}: {tot} samples, {sum(d[1] for d in data)} warp instructions")
for s, e, ln, src in sorted(data, reverse=True)[:top]:
    print(f"{100*s/tot:5.1f}% ex={e:10d} L{ln:4d} {src}")
