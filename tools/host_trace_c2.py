import sys; sys.path.insert(0,'.')
from paper_1407_3535_b200 import api, workloads as W
wl=W.make("C2"); ctx=api.Context(0); img=ctx.image(wl.image); t=wl.templates[0].pixels
for _ in range(8):
    img.reset_cache(); ctx.search(img, t, policy="seeded")
