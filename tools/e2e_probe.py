"""Where the e2e time goes on a config: resident searches vs the image stream vs the PCIe
copies alone (wall clock, K images)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1407_3535_b200 import api, workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
wl = W.make(name)
t = wl.templates[0].pixels
ctx = api.Context(0)
img = ctx.image(wl.image)
host = [torch.empty(wl.image.shape, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
for h in host:
    h.numpy()[:] = wl.image
dev = torch.empty(wl.image.shape, dtype=torch.uint8, device="cuda")
for _ in range(3):
    img.reset_cache()
    ctx.search(img, t, mode="egs", policy="seeded")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(K):
    img.reset_cache()
    ctx.search(img, t, mode="egs", policy="seeded")
torch.cuda.synchronize()
a = (time.perf_counter() - t0) * 1e3 / K
seq = [host[i & 1].numpy() for i in range(K)]
ctx.search_stream(seq[:2], t, mode="egs", policy="seeded")
torch.cuda.synchronize()
t0 = time.perf_counter()
ctx.search_stream(seq, t, mode="egs", policy="seeded")
b = (time.perf_counter() - t0) * 1e3 / K
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(K):
    dev.copy_(host[i & 1], non_blocking=True)
torch.cuda.synchronize()
c = (time.perf_counter() - t0) * 1e3 / K
print(f"{name}: resident search {a:.2f} ms, stream {b:.2f} ms/image, H2D alone {c:.2f} ms "
      f"({wl.image.nbytes / c / 1e6:.1f} GB/s)")
