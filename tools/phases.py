"""Per-phase device time of one search per template (after a warm-up run), any config.

    python tools/phases.py C4 [policy] [template indices...]
Prints one JSON object per template: {phase: ms} from the context's event timers.
"""
import json
import sys
import time

sys.path.insert(0, ".")
from paper_1407_3535_b200 import api, workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
policy = sys.argv[2] if len(sys.argv) > 2 else "seeded"
idx = [int(a) for a in sys.argv[3:]]
wl = W.make(cfg)
ctx = api.Context(0)
img = ctx.image(wl.image)
m, n = wl.templates[0].pixels.shape
prep = ctx.prepare(img, m, n, mode=wl.mode)
ctx.set_profiling(True)
img.reset_cache()
base = ctx.phase_times()
prep2 = ctx.prepare(img, m, n, mode=wl.mode)
after = ctx.phase_times()
print(json.dumps({"config": cfg, "prepare": {k: round(v["ms"] - base.get(k, {"ms": 0})["ms"], 3)
                                              for k, v in after.items()}}), flush=True)
for k in [i for i in (idx or range(len(wl.templates))) if i < len(wl.templates)]:
    t = wl.templates[k].pixels
    ctx.run(prep, t, policy=policy)  # warm
    b = ctx.phase_times()
    t0 = time.perf_counter()
    r = ctx.run(prep, t, policy=policy)
    wall = (time.perf_counter() - t0) * 1e3
    a = ctx.phase_times()
    d = {k2: round(v["ms"] - b.get(k2, {"ms": 0})["ms"], 3) for k2, v in a.items()
         if v["ms"] - b.get(k2, {"ms": 0})["ms"] > 0}
    print(json.dumps({"k": k, "wall_ms": round(wall, 3), "retained": r.retained,
                      "elim_pct": round(r.elim_pct, 2), "phases": d}), flush=True)
