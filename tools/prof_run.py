"""Prepare once, then run the search of template 0 `reps` times (for ncu captures of the
search kernels).  python tools/prof_run.py C4 [policy] [reps]"""
import sys
sys.path.insert(0, ".")
from paper_1407_3535_b200 import api, workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
policy = sys.argv[2] if len(sys.argv) > 2 else "seeded"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
wl = W.make(cfg)
ctx = api.Context(0)
img = ctx.image(wl.image)
t = wl.templates[0].pixels
prep = ctx.prepare(img, *t.shape, mode=wl.mode)
for _ in range(reps):
    r = ctx.run(prep, t, policy=policy)
print(r)
