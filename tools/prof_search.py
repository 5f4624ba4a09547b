"""tm_search (prepare + run in one call, the bench step) on one config `reps` times:
a short command for ncu captures of the current search path.
    python tools/prof_search.py C2 [reps]"""
import sys
sys.path.insert(0, ".")
from paper_1407_3535_b200 import api, workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
wl = W.make(cfg)
ctx = api.Context(0)
img = ctx.image(wl.image)
t = wl.templates[0].pixels.astype("uint8")
for _ in range(reps):
    img.reset_cache()
    r = ctx.search(img, t, mode="egs", policy="seeded")
print(r)
