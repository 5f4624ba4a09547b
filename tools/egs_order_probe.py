"""How early the count-only EGS candidate could reject with its blocks ordered by retained
density (best case: the true density) versus launch order.  C5, h = 5."""
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
ret = amap < 0.6
tr, tc = (er + h - 1) // h, (ec + h - 1) // h
# centres are not members
for ti in range(tr):
    r0, r1 = ti * h, min(ti * h + h, er) - 1
    cr = (r0 + r1) // 2
    cols = np.array([(tj * h + min(tj * h + h, ec) - 1) // 2 for tj in range(tc)])
    ret[cr, cols] = False
G3 = ((er + 2) // 3) * ((ec + 2) // 3)
nr3 = int(ctx.autocorr_retained(img, m, n, 3, 3))
cost3 = G3 + nr3
bound = 0.995 * cost3 - tr * tc
print("n_r total", int(ret.sum()), "bound", bound)
# blocks: 109 group columns x 96 group rows (the launch geometry of k_acg<5,128> on C5)
bg, br = 109 * h, 96 * h
R, Cc = (er + br - 1) // br, (ec + bg - 1) // bg
pad = np.zeros((R * br, Cc * bg), bool)
pad[:er, :ec] = ret
per = pad.reshape(R, br, Cc, bg).sum(axis=(1, 3)).T.ravel()  # tile-major like blockIdx
for label, order in (("launch order", np.arange(per.size)), ("by density", np.argsort(-per))):
    cum = np.cumsum(per[order])
    k = int(np.searchsorted(cum, bound)) + 1
    print(f"{label}: reject after {k} of {per.size} blocks ({k / per.size * 100:.1f}%)")
