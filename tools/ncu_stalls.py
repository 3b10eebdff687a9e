"""Stall-reason totals of one kernel in an ncu report (source page, SASS level), plus the top SASS
instructions by samples.  usage: python tools/ncu_stalls.py report.ncu-rep kernel_regex [top]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name", f"regex:{kern}", "--launch-count", "1"], capture_output=True, text=True).stdout
lines = [l for l in out.splitlines() if l.startswith('"')]
rows = list(csv.reader(io.StringIO("\n".join(lines))))
hdr = next(r for r in rows if r and r[0] == "Address")
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
si = hdr.index("Warp Stall Sampling (All Samples)")
tot = {hdr[i]: 0 for i in cols}
data = []
for r in rows:
    if r and r[0].startswith("0x"):
        for i in cols:
            tot[hdr[i]] += int(r[i] or 0)
        data.append((int(r[si] or 0), r[1].strip(), {hdr[i]: int(r[i] or 0) for i in cols if int(r[i] or 0)}))
T = sum(tot.values()) or 1
print("stall totals:", {k[6:]: f"{100*v/T:.1f}%" for k, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v})
for s, src, st in sorted(data, key=lambda d: -d[0])[:top]:
    print(f"{100*s/T:5.1f}% {src[:60]:60s} {dict(sorted(st.items(), key=lambda kv: -kv[1])[:3])}")
