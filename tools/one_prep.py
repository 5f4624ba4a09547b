"""One preparation of a config (short command for ncu launch lists)."""
import sys

sys.path.insert(0, ".")
from paper_1407_3535_b200 import api, workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C6"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
wl = W.make(name)
ctx = api.Context(0)
img = ctx.image(wl.image)
m, n = wl.templates[0].pixels.shape
for _ in range(reps):
    img.reset_cache()
    prep = ctx.prepare(img, m, n, mode=wl.mode)
    print(name, prep.info["h"], prep.info["kappa"], prep.info["prep_ms"])
    prep.close()
