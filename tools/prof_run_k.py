"""Prepare once, run template k once (for ncu captures of one search of a config).
    python tools/prof_run_k.py C4 12"""
import sys
sys.path.insert(0, ".")
from paper_1407_3535_b200 import api, workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 0
wl = W.make(cfg)
ctx = api.Context(0)
img = ctx.image(wl.image)
t = wl.templates[k].pixels
prep = ctx.prepare(img, *t.shape, mode=wl.mode)
print(ctx.run(prep, t, policy="seeded"))
