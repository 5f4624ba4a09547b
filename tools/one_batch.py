"""One prepare + batch run of a config (short command for ncu)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1407_3535_b200 import api, workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
policy = sys.argv[2] if len(sys.argv) > 2 else "seeded"
wl = W.make(name)
ctx = api.Context(0)
img = ctx.image(wl.image)
m, n = wl.templates[0].pixels.shape
prep = ctx.prepare(img, m, n, mode=wl.mode)
rs = ctx.run(prep, np.stack([t.pixels for t in wl.templates]), policy=policy)
print(name, [(r.best_row, r.best_col) for r in rs][:4])
