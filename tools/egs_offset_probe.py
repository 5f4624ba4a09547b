"""Retention of the count-only EGS candidate by member offset: how early its in-kernel
rejection could come if the column-offset CTAs ran in the order of their retained density
(|dj| = 2 first) and segments densest first.  C5, h = 5:  python tools/egs_offset_probe.py C5 5"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1407_3535_b200 import api, workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
h = int(sys.argv[2]) if len(sys.argv) > 2 else 5
wl = W.make(name)
ctx = api.Context(0)
img = ctx.image(wl.image)
m, n = wl.templates[0].pixels.shape
er, ec = wl.image.shape[0] - m + 1, wl.image.shape[1] - n + 1
amap = ctx.local_autocorrelation(img, m, n, h, h)
thr = 0.6
tr, tc = (er + h - 1) // h, (ec + h - 1) // h
G3 = ((er + 2) // 3) * ((ec + 2) // 3)
nr3 = int(ctx.autocorr_retained(img, m, n, 3, 3))
bound = 0.995 * (G3 + nr3) - tr * tc
hr = h // 2
# offsets of every location from its group's centre (regular groups)
rows = np.arange(er)
cols = np.arange(ec)
ti = np.minimum(rows // h, tr - 1)
tj = np.minimum(cols // h, tc - 1)
r0 = ti * h
r1 = np.minimum(r0 + h, er) - 1
cr = (r0 + r1) // 2
c0 = tj * h
c1 = np.minimum(c0 + h, ec) - 1
cc = (c0 + c1) // 2
di = rows - cr
dj = cols - cc
ret = amap < thr
tot = 0
print("n_r bound", bound)
per_dj = {}
for d in range(-hr, hr + 1):
    sel = ret[:, dj == d]
    # centres are not members
    cnt = int(sel.sum()) - int(((di[:, None] == 0) & sel).sum()) if d == 0 else int(sel.sum())
    per_dj[d] = cnt
    tot += cnt
    print(f"dj={d:+d} retained {cnt} ({cnt / max(1, (dj == d).sum() * er):.3f} of its locations)")
print("total", tot)
for d in range(-hr, hr + 1):
    sel = ret[di == d, :]
    cnt = int(sel.sum()) - (int(((dj[None, :] == 0) & sel).sum()) if d == 0 else 0)
    print(f"di={d:+d} retained {cnt} ({cnt / max(1, (di == d).sum() * ec):.3f} of its locations)")
for order in ([-2, -1, 0, 1, 2], [-2, 2, -1, 1, 0]):
    cum, work = 0, 0
    for d in order:
        if cum + per_dj[d] >= bound:
            frac = (bound - cum) / per_dj[d]
            work += frac
            break
        cum += per_dj[d]
        work += 1
    print("dj order", order, f"-> rejection after {work / len(order) * 100:.1f}% of the work (uniform density within a dj)")
