"""One (or a few) searches of a config -- a short command for ncu launch lists."""
import sys

sys.path.insert(0, ".")
from paper_1407_3535_b200 import api, workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
policy = sys.argv[2] if len(sys.argv) > 2 else "seeded"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
wl = W.make(name)
ctx = api.Context(0)
img = ctx.image(wl.image)
for _ in range(reps):
    img.reset_cache()
    r = ctx.search(img, wl.templates[0].pixels, mode="egs", policy=policy,
                   parallel=policy == "frozen", threads=2)
print(name, policy, r.best_row, r.best_col, r.best_rho, r.eliminated, r.retained)
