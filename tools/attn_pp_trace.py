"""Timeline statistics of an MTKV_ATTN_TRACE dump of the two-lane attention
kernel (attn_pp.cu; lane A of the first 64 CTAs).

  python tools/attn_pp_trace.py trace.bin"""
import sys

import numpy as np

C, K, T = 64, 12, 96
a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(C, K, T).astype(np.int64)
g0 = min(a[c, 5, 0] for c in range(C) if a[c, 5, 0])
us = lambda v: (v - g0) / 1e3


def dist(name, xs):
    xs = np.array([v for v in xs if np.isfinite(v)])
    if len(xs):
        print(f"{name:36s} p10 {np.percentile(xs, 10):7.3f} p50 {np.median(xs):7.3f} mean {xs.mean():7.3f} "
              f"p90 {np.percentile(xs, 90):7.3f}  (n={len(xs)})")


def pairs(k1, k2, shift=0):
    out = []
    for c in range(C):
        for t in range(T - shift):
            if a[c, k1, t] and a[c, k2, t + shift]:
                out.append((a[c, k2, t + shift] - a[c, k1, t]) / 1e3)
    return out


print("cta  start  setup firstK firstS  end  subtiles epilogues")
for c in range(0, C, 8):
    if not a[c, 5, 0]:
        continue
    n = int((a[c, 3] > 0).sum())
    ep = [(us(a[c, 5, 3 + 2 * k]), us(a[c, 5, 4 + 2 * k])) for k in range(8) if a[c, 5, 3 + 2 * k]]
    print(f"{c:3d} {us(a[c,5,0]):6.2f} {us(a[c,5,1]):6.2f} {us(a[c,0,0]):6.2f} {us(a[c,3,0]):6.2f} {us(a[c,5,2]):6.2f} "
          f"{n:5d}  " + " ".join(f"{s_:.1f}-{e_:.1f}" for s_, e_ in ep))
ends = np.array([us(a[c, 5, 2]) for c in range(C) if a[c, 5, 2]])
print(f"end min {ends.min():.2f} mean {ends.mean():.2f} max {ends.max():.2f}")
per = []
for c in range(C):
    n = int((a[c, 3] > 0).sum())
    if n > 4:
        per += list(np.diff(a[c, 3, 2:n]) / 1e3)
dist("softmax wake interval (per sub-tile)", per)
dist("K issued -> S issued", pairs(0, 1))
dist("V issued -> V ready at PV", pairs(9, 11))
dist("P ready -> V ready (>0: waits V)", pairs(10, 11))
dist("S issued -> S ready (softmax)", pairs(1, 3))
dist("softmax: S ld + max", pairs(3, 6))
dist("softmax: exps", pairs(6, 7))
dist("softmax: P st + rescale + arrive", pairs(7, 4))
dist("softmax idle (P arrive -> next S)", pairs(4, 3, 1))
dist("P arrive -> PV issued", pairs(4, 2))
