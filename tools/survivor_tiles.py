"""How the scan-2 survivors of a config spread over the dense pass's 16x2048 tiles."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1407_3535_b200 import api, workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
wl = W.make(name)
ctx = api.Context(0)
img = ctx.image(wl.image)
t = wl.templates[0].pixels
m, n = t.shape
prep = ctx.prepare(img, m, n, mode="egs")
r, vis = ctx.run(prep, t, policy="seeded", record_visits=True)
_, _, fl = ctx.window_stats(img, m, n)
surv = (vis == 2) & (fl == 0)
er, ec = surv.shape
print("survivors (non-flat retained):", int(surv.sum()), "of", er * ec)
for th, tw in ((16, 2048), (16, 512), (16, 128), (64, 64)):
    R, Cc = (er + th - 1) // th, (ec + tw - 1) // tw
    pad = np.zeros((R * th, Cc * tw), bool)
    pad[:er, :ec] = surv
    per = pad.reshape(R, th, Cc, tw).sum(axis=(1, 3))
    on = per > 0
    print(f"tiles {th}x{tw}: {int(on.sum())} of {on.size} flagged ({on.mean() * 100:.1f}%), "
          f"median survivors per flagged tile {np.median(per[on]):.0f}")
