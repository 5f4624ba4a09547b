"""Per-phase device times of one config's search under environment variants (A/B runs of
kernel geometry knobs).  Each variant runs in a fresh process (the knobs are read once)."""
import json
import os
import subprocess
import sys

CODE = r'''
import json, sys
sys.path.insert(0, ".")
from paper_1407_3535_b200 import api, workloads as W
wl = W.make(sys.argv[1])
ctx = api.Context(0)
img = ctx.image(wl.image)
t = wl.templates[0].pixels
for _ in range(2):
    img.reset_cache(); ctx.search(img, t, mode="egs", policy="seeded")
ctx.set_profiling(True)
base = ctx.phase_times()
for _ in range(3):
    img.reset_cache(); r = ctx.search(img, t, mode="egs", policy="seeded")
ph = ctx.phase_times()
print(json.dumps({k: round((v["ms"] - base.get(k, {"ms": 0})["ms"]) / 3, 4) for k, v in ph.items()}
                 | {"best": [r.best_row, r.best_col, r.best_rho]}))
'''

cfg = sys.argv[1]
for spec in sys.argv[2:]:
    env = dict(os.environ)
    for kv in spec.split(","):
        if "=" in kv:
            k, v = kv.split("=", 1)
            env[k] = v
    out = subprocess.run([sys.executable, "-c", CODE, cfg], env=env, capture_output=True,
                         text=True)
    print(spec, out.stdout.strip()[-600:] or out.stderr[-600:], flush=True)
