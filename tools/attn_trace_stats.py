"""Timeline statistics of an MTKV_ATTN_TRACE dump (one attn_tc launch, first 64 CTAs).

  python tools/attn_trace_stats.py trace.bin
Per-CTA start / first K issue / first S / end (us from the earliest CTA start),
softmax per-tile phases, K issue -> S latency and the end-time spread."""
import sys

import numpy as np

C, K, T = 64, 12, 96
a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(C, K, T).astype(np.int64)
g0 = min(a[c, 5, 0] for c in range(C) if a[c, 5, 0])
us = lambda x: (x - g0) / 1e3
print("cta  start  init firstK firstS lastPV    end tiles  epilogues")
for c in range(0, C, 4):
    if not a[c, 5, 0]:
        continue
    n = int((a[c, 0] > 0).sum())
    ep = [(us(a[c, 5, 3 + 2 * k]), us(a[c, 5, 4 + 2 * k])) for k in range(8) if a[c, 5, 3 + 2 * k]]
    print(f"{c:3d} {us(a[c,5,0]):6.2f} {us(a[c,5,1]):6.2f} {us(a[c,0,0]):6.2f} {us(a[c,1,0]):6.2f} "
          f"{us(a[c,2,n-1]):6.2f} {us(a[c,5,2]):6.2f} {n:5d}  " + " ".join(f"{s:.1f}-{e:.1f}" for s, e in ep))
ends = np.array([us(a[c, 5, 2]) for c in range(C) if a[c, 5, 2]])
print(f"end min {ends.min():.2f} mean {ends.mean():.2f} max {ends.max():.2f}")


def dist(name, x):
    x = np.array(x)
    if len(x):
        print(f"{name:34s} p10 {np.percentile(x,10):.3f} p50 {np.median(x):.3f} mean {x.mean():.3f} "
              f"p90 {np.percentile(x,90):.3f}")


iv = []
for c in range(C):
    n = int((a[c, 3] > 0).sum())
    if n > 4:
        iv += list(np.diff(a[c, 3, 2:n]) / 1e3)
dist("softmax wake interval (us)", iv)
lat = [(a[c, 1, t] - a[c, 0, t]) / 1e3 for c in range(C) for t in range(T) if a[c, 1, t] and a[c, 0, t]]
dist("K issue -> S issued", lat)
for k1, k2, nm in ((3, 6, "S ld + max exchange"), (6, 7, "exp"), (7, 8, "P st + o_done wait + rescale"),
                   (8, 4, "st wait + arrive")):
    dist(nm, [(a[c, k2, t] - a[c, k1, t]) / 1e3 for c in range(C) for t in range(T) if a[c, k1, t] and a[c, k2, t]])
dist("softmax idle waiting for S", [(a[c, 3, t] - a[c, 4, t - 1]) / 1e3 for c in range(C) for t in range(1, T)
                                    if a[c, 4, t - 1] and a[c, 3, t]])
dist("MMA: p_full wait -> PV issued", [(a[c, 2, t] - a[c, 10, t]) / 1e3 for c in range(C) for t in range(T)
                                       if a[c, 2, t] and a[c, 10, t]])
dist("MMA: S wait entered -> S issued", [(a[c, 1, t] - a[c, 9, t]) / 1e3 for c in range(C) for t in range(T)
                                         if a[c, 1, t] and a[c, 9, t]])
