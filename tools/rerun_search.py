"""Repeated searches of one config's templates after one preparation (warm timings):
    python tools/rerun_search.py C5 [policy] [reps] [--visits]
Prints wall ms per call (device-synchronous API calls)."""
import sys
import time

sys.path.insert(0, ".")
from paper_1407_3535_b200 import api, workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
policy = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else "seeded"
reps = int(sys.argv[3]) if len(sys.argv) > 3 and not sys.argv[3].startswith("--") else 3
visits = "--visits" in sys.argv
wl = W.make(cfg)
ctx = api.Context(0)
img = ctx.image(wl.image)
m, n = wl.templates[0].pixels.shape
prep = ctx.prepare(img, m, n, mode=wl.mode)
for k, tp in enumerate(wl.templates[:4]):
    for i in range(reps):
        t0 = time.perf_counter()
        r = ctx.run(prep, tp.pixels, policy=policy, parallel=(policy == "frozen"), threads=2,
                    record_visits=visits)
        if visits:
            r = r[0]
        print(cfg, policy, "template", k, "rep", i, f"{(time.perf_counter() - t0) * 1e3:.2f} ms",
              r.refined_row, r.refined_col, r.retained, flush=True)
