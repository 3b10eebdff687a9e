"""Summarise a chrome trace from h2g_ctx_trace_dump: busy time per stream, gaps, host sync waits."""
import json, sys
ev = json.load(open(sys.argv[1]))["traceEvents"]
dev = [e for e in ev if e["pid"] == 0]
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
