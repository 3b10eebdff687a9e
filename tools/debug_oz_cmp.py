import sys, numpy as np
a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
worst = {}
for k in a.files:
    x, y = a[k], b[k]
    if k.endswith("xrank"):
        print(k, "equal" if np.array_equal(x, y) else f"DIFF at {np.flatnonzero(x != y)[:10]}")
        continue
    if x.size == 0: continue
    e = np.abs(x - y).max() / max(np.abs(y).max(), 1e-300)
    grp = k.rsplit(".", 1)[0]
    worst[grp] = max(worst.get(grp, 0), e)
print(worst)
