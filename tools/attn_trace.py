"""Summarise an MTKV_ATTN_TRACE dump (per-CTA event times of one attn_tc launch).

kinds: 0 K issue (producer), 1 S issued, 2 PV issued, 3 S ready (softmax woke),
4 P in TMEM (warp 0 of the pipeline), 5 CTA start/init/end, 6 S loaded,
7 exps done, 8 o_done passed, 9 MMA: S wait entered, 10 MMA: PV wait entered,
11 P in TMEM (warp 3 of the pipeline)."""
import sys
import numpy as np
C, K, T = 64, 12, 96
a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(C, K, T).astype(np.int64)
names = ["Kiss", "S", "PV", "s_rdy", "Pdone", "", "mx", "exp", "orsc", "Swt", "PVwt", "P3"]
order = [0, 9, 1, 3, 6, 7, 8, 4, 11, 10, 2]
for c in range(min(int(sys.argv[2]) if len(sys.argv) > 2 else 3, C)):
    t0 = a[c, 5, 0]
    if t0 == 0:
        continue
    print(f"CTA {c}: init {(a[c,5,1]-t0)/1e3:.2f}us end {(a[c,5,2]-t0)/1e3:.2f}us")
    n = int((a[c, 0] > 0).sum())
    for t in range(n):
        row = " ".join(f"{names[k]}={(a[c,k,t]-t0)/1e3:6.2f}" if a[c, k, t] else f"{names[k]}=   -  " for k in order)
        print(f"  {t:2d}: {row}")
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
# piece epilogues (pipeline 0, thread 128): kind 5, slots 3+2k (start) / 4+2k (end)
for c in range(min(int(sys.argv[2]) if len(sys.argv) > 2 else 3, C)):
    t0 = a[c, 5, 0]
    ep = [(k, (a[c, 5, 3 + 2 * k] - t0) / 1e3, (a[c, 5, 4 + 2 * k] - t0) / 1e3) for k in range(8) if a[c, 5, 3 + 2 * k]]
    n = int((a[c, 0] > 0).sum())
    print(f"CTA {c}: tiles traced {n}, last S {(a[c,1,n-1]-t0)/1e3:.2f}us, end {(a[c,5,2]-t0)/1e3:.2f}us, "
          f"epilogues " + ", ".join(f"#{k}: {s:.2f}-{e:.2f}" for k, s, e in ep))
# epilogue phases (kind 11, slots 4k..4k+3): o_done passed, l exchanged, store pass 1, store pass 2
for c in range(min(int(sys.argv[2]) if len(sys.argv) > 2 else 3, C)):
    t0 = a[c, 5, 0]
    for k in range(8):
        if not a[c, 5, 3 + 2 * k]:
            continue
        st = (a[c, 5, 3 + 2 * k] - t0) / 1e3
        ph = [(a[c, 11, 4 * k + i] - t0) / 1e3 if a[c, 11, 4 * k + i] else float("nan") for i in range(4)]
        print(f"CTA {c} epilogue #{k}: start {st:.2f} odone {ph[0]:.2f} l {ph[1]:.2f} pass1 {ph[2]:.2f} pass2 {ph[3]:.2f} "
              f"end {(a[c, 5, 4 + 2 * k] - t0) / 1e3:.2f}")
