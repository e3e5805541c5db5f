"""Summarise an MTKV_ATTN_TRACE dump (per-CTA event times of one attn_tc launch)."""
import sys
import numpy as np
C, K, T = 64, 6, 32
a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(C, K, T).astype(np.int64)
names = ["issue", "S", "PV", "s_ready", "P_done"]
for c in range(min(int(sys.argv[2]) if len(sys.argv) > 2 else 3, C)):
    t0 = a[c, 5, 0]
    if t0 == 0:
        continue
    print(f"CTA {c}: init {(a[c,5,1]-t0)/1e3:.2f}us end {(a[c,5,2]-t0)/1e3:.2f}us")
    n = int((a[c, 0] > 0).sum())
    for t in range(n):
        row = " ".join(f"{names[k]}={(a[c,k,t]-t0)/1e3:7.2f}" if a[c, k, t] else f"{names[k]}=   -   " for k in range(5))
        print(f"  tile {t:2d}: {row}")
# aggregate: per-CTA duration and data-latency (S issue - producer issue)
dur, lat, per_tile = [], [], []
for c in range(C):
    if a[c, 5, 0] == 0 or a[c, 5, 2] == 0:
        continue
    dur.append((a[c, 5, 2] - a[c, 5, 0]) / 1e3)
    n = int((a[c, 0] > 0).sum())
    for t in range(n):
        if a[c, 1, t] and a[c, 0, t]:
            lat.append((a[c, 1, t] - a[c, 0, t]) / 1e3)
    if n > 1:
        per_tile.append((a[c, 2, n - 1] - a[c, 0, 0]) / 1e3 / n)
print(f"CTAs {len(dur)}: duration mean {np.mean(dur):.2f}us; issue->S mean {np.mean(lat):.2f}us "
      f"p50 {np.median(lat):.2f}; per-tile {np.mean(per_tile):.2f}us")
