import os, sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
from oracle.binding import Oracle
from paper_1407_3535_b200 import api
port = Oracle("port")
rng = np.random.default_rng(3)
for (p, q, m) in ((96, 96, 16), (256, 256, 32), (512, 512, 32)):
    base = np.cumsum(np.cumsum(rng.normal(size=(p, q)), 0), 1)
    img = np.clip(np.rint((base - base.min()) / np.ptp(base) * 255), 0, 255)
    b = port.blur(img)
    t = np.clip(np.rint(b[5:5 + m, 7:7 + m]), 0, 255)
    amap = port.local_autocorrelation(b, m, m, 3, 3)
    with api.Context(0) as ctx:
        g = ctx.image(b)
        for _ in range(3):
            ctx.transitive_search(t, g, amap, 3, 3, parallel=True, threads=2)
            ctx.brute_force_match(t, g)
        t0 = time.perf_counter()
        for _ in range(20):
            ctx.transitive_search(t, g, amap, 3, 3, parallel=True, threads=2)
        t1 = time.perf_counter()
        for _ in range(20):
            ctx.brute_force_match(t, g)
        t2 = time.perf_counter()
        print(os.environ.get("TMATCH_TC_SPLIT", "1"), (p, q, m), "search ms", (t1 - t0) / 20 * 1e3, "brute ms", (t2 - t1) / 20 * 1e3)
