import sys
sys.path.insert(0, ".")
from paper_1407_3535_b200 import api, workloads as W
for cfg in ["C2", "C4", "C5"]:
    wl = W.make(cfg)
    ctx = api.Context(0)
    img = ctx.image(wl.image)
    m, n = wl.templates[0].pixels.shape
    er, ec = wl.image.shape[0] - m + 1, wl.image.shape[1] - n + 1
    e = ctx.efficient_group_size(img, m, n)
    print(cfg, "h_e", e["h"], "trace", [(x["h"], x["retained"], x["total"]) for x in e["trace"]])
    for h in (3, 5, 7):
        nr = ctx.autocorr_retained(img, m, n, h, h)
        central = ((er + h - 1) // h) * ((ec + h - 1) // h)
        print("   h", h, "n_r", nr, "central", central, "total", central + nr)
