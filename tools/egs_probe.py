"""EGS numbers of a config: full retained counts per candidate size (no early stop), the
accepted size's cost, and the rejection bound of the next candidate."""
import sys
import time

sys.path.insert(0, ".")
from paper_1407_3535_b200 import api, workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
wl = W.make(name)
ctx = api.Context(0)
img = ctx.image(wl.image)
m, n = wl.templates[0].pixels.shape
er, ec = wl.image.shape[0] - m + 1, wl.image.shape[1] - n + 1
prep = ctx.prepare(img, m, n, mode="egs")
print("h_e", prep.info["h"], "trace", prep.info.get("egs_trace"))
for h in (3, 5, 7):
    ctx.synchronize()
    t0 = time.perf_counter()
    nr = ctx.autocorr_retained(img, m, n, h, h)
    ctx.synchronize()
    G = ((er + h - 1) // h) * ((ec + h - 1) // h)
    print(f"h={h} n_r={nr} G={G} cost={G + nr} ({(time.perf_counter() - t0) * 1e3:.1f} ms)")
