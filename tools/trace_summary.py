"""Summarise a chrome trace from h2g_ctx_trace_dump: busy time per stream, gaps, host sync waits."""
import json, sys
ev = json.load(open(sys.argv[1]))["traceEvents"]
dev_all = [e for e in ev if e["pid"] == 0]
dev = [e for e in dev_all if e["name"] in ("gsum", "qr_r", "svd", "norm", "gather")]
sub = [e for e in dev_all if e not in dev]
host = [e for e in ev if e["pid"] == 1]
t_end = max(e["ts"] + e["dur"] for e in ev)
print(f"span {t_end/1e3:.1f} ms, {len(dev)} device intervals, {len(host)} host syncs")
for tid in (0, 1):
    iv = sorted((e["ts"], e["ts"] + e["dur"]) for e in dev if e["tid"] == tid)
    busy = 0.0; cur_s = cur_e = None
    for s, e in iv:
        if cur_e is None or s > cur_e:
            if cur_e is not None: busy += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    if cur_e is not None: busy += cur_e - cur_s
    print(f"stream {tid}: busy {busy/1e3:.1f} ms")
    by = {}
    for e in dev:
        if e["tid"] == tid: by[e["name"]] = by.get(e["name"], 0) + e["dur"]
    print("   ", {k: round(v / 1e3, 1) for k, v in sorted(by.items(), key=lambda kv: -kv[1])})
# union of both streams
iv = sorted((e["ts"], e["ts"] + e["dur"]) for e in dev)
busy = 0.0; cs = ce = None
for s, e in iv:
    if ce is None or s > ce:
        if ce is not None: busy += ce - cs
        cs, ce = s, e
    else: ce = max(ce, e)
if ce is not None: busy += ce - cs
print(f"GPU busy (any stream): {busy/1e3:.1f} ms of {t_end/1e3:.1f} ms")
if len(sys.argv) > 2:   # timeline: per stream, ordered device intervals and host syncs
    tid = int(sys.argv[2])
    evs = sorted([e for e in ev if e["tid"] == tid or e["pid"] == 1], key=lambda e: e["ts"])
    last = 0.0
    for e in evs:
        kind = "HOST" if e["pid"] == 1 else "dev "
        print(f"{kind} {e['ts']/1e3:8.2f} +{e['dur']/1e3:6.2f} ms  gap {max(0, e['ts'] - last)/1e3:5.2f}  {e['name']} tid{e['tid']}")
        if e["pid"] == 0: last = max(last, e["ts"] + e["dur"])
# per stage tag: launches, device ms (per stream), span (first start .. last end)
print("\nper tag (stream: launches, kernel ms, span ms, GFLOP)")
tags = {}
for e in dev:
    a = e.get("args", {})
    key = (a.get("tag", ""), e["tid"])
    t = tags.setdefault(key, [0, 0.0, 1e18, 0.0, 0.0, {}])
    t[0] += 1; t[1] += e["dur"]; t[2] = min(t[2], e["ts"]); t[3] = max(t[3], e["ts"] + e["dur"]); t[4] += a.get("gflop", 0)
    t[5][e["name"]] = t[5].get(e["name"], 0) + e["dur"]
for e in sub:
    key = (e.get("args", {}).get("tag", ""), e["tid"])
    if key in tags: tags[key][5][e["name"]] = tags[key][5].get(e["name"], 0) + e["dur"]
for (tag, tid), t in sorted(tags.items(), key=lambda kv: kv[1][2]):
    print(f"  {tag:14s} s{tid}  n={t[0]:3d}  [{t[2]/1e3:7.1f} .. {t[3]/1e3:7.1f}]  dev {t[1]/1e3:6.2f}  span {(t[3]-t[2])/1e3:6.2f}  {t[4]:7.3f} GF  "
          + " ".join(f"{k}:{v/1e3:.2f}" for k, v in sorted(t[5].items(), key=lambda kv: -kv[1])))
