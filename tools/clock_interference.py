"""Does NVML clock sampling during the timed region slow the search?  Times C5 steps
(seeded / frozen) with and without bench.ClockSampler running."""
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1407_3535_b200 import api, workloads as W  # noqa: E402

wl = W.make(sys.argv[1] if len(sys.argv) > 1 else "C5")
ctx = api.Context(0)
img = ctx.image(wl.image)
t = wl.templates[0].pixels
stream = torch.cuda.ExternalStream(ctx.stream_ptr, device=torch.device("cuda:0"))


def steps(policy, k=5):
    out = []
    for _ in range(k):
        img.reset_cache()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t0 = time.perf_counter()
        ctx.search(img, t, mode="egs", policy=policy, parallel=policy == "frozen", threads=2)
        e1.record(stream)
        e1.synchronize()
        out.append((e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3))
    return [round(statistics.mean(x), 2) for x in zip(*out)]


for pol in ("seeded", "frozen", "seeded"):
    steps(pol, 3)
    a = steps(pol)
    cs = bench.ClockSampler(0)
    cs.start()
    b = steps(pol)
    c = cs.stop()
    print(pol, "no-sampler (dev ms, wall ms)", a, "sampler", b, c["samples"], flush=True)
