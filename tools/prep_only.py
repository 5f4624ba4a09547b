"""Prepare (EGS/OptA) on one config, twice: a short command for ncu launch lists."""
import sys
sys.path.insert(0, ".")
from paper_1407_3535_b200 import api, workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
wl = W.make(cfg)
ctx = api.Context(0)
img = ctx.image(wl.image)
m, n = wl.templates[0].pixels.shape
for _ in range(2):
    img.reset_cache()
    prep = ctx.prepare(img, m, n, mode=wl.mode)
    print(prep.info, flush=True)
    prep.close()
