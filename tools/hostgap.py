"""Wall time of prepare() and run() (each bracketed by device syncs) vs device phase time."""
import sys
import time

sys.path.insert(0, ".")
from paper_1407_3535_b200 import api, workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
wl = W.make(cfg)
ctx = api.Context(0)
img = ctx.image(wl.image)
t = wl.templates[0].pixels
m, n = t.shape
for i in range(25):
    img.reset_cache()
    ctx.synchronize()
    t0 = time.perf_counter()
    prep = ctx.prepare(img, m, n, mode="egs")
    ctx.synchronize()
    t1 = time.perf_counter()
    r = ctx.run(prep, t, policy="seeded")
    t2 = time.perf_counter()
    prep.close()
    if i >= 5:
        print(f"prepare {1e3 * (t1 - t0):.3f} ms  run {1e3 * (t2 - t1):.3f} ms")
ctx.set_profiling(True)
img.reset_cache()
b = ctx.phase_times()
prep = ctx.prepare(img, m, n, mode="egs")
r = ctx.run(prep, t, policy="seeded")
a = ctx.phase_times()
print({k: round(v["ms"] - b.get(k, {"ms": 0})["ms"], 3) for k, v in a.items()})
