"""GPU timeline of a few C2 searches (or tm_search_stream_u8 calls: arg 3 = stream) via torch.profiler (CUPTI sees every kernel in the
process): prints each kernel / memcpy with its start offset, duration and the idle gap
before it, for the last search.   python tools/timeline.py [C2] [steps]"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1407_3535_b200 import api, workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
upload = len(sys.argv) > 3 and sys.argv[3] == "upload"  # the e2e step: tm_search_upload_u8
stream = len(sys.argv) > 3 and sys.argv[3] == "stream"  # tm_search_stream_u8 over `steps` images
wl = W.make(cfg)
ctx = api.Context(0)
img = ctx.image(wl.image)
t = wl.templates[0].pixels
pinned = torch.empty(wl.image.shape, dtype=torch.uint8, pin_memory=True)
pinned.numpy()[:] = wl.image


def step():
    if stream:
        ctx.search_stream([pinned.numpy()] * 4, t.astype("uint8"), policy="seeded")
    elif upload:
        ctx.search_upload(img, pinned.numpy(), t.astype("uint8"), policy="seeded")
    else:
        img.reset_cache()
        ctx.search(img, t, policy="seeded")


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
evs.sort(key=lambda e: e.time_range.start)
# split into searches at the first window-statistics kernel
def big_copy(e):  # an image chunk (the template copies are a few microseconds)
    return "Memcpy HtoD" in e.name and (e.time_range.end - e.time_range.start) > 8.0


starts = [i for i, e in enumerate(evs) if (upload and big_copy(e) and
                                           (i == 0 or not big_copy(evs[i - 1])))
          or (not upload and "k_sum_sq_u8" in e.name)]
if stream:  # the search before the last (its next image's copy overlaps it)
    starts = [i for i, e in enumerate(evs) if "k_tc_pitch" in e.name]
    starts = starts[-2:-1] + [len(evs)] if len(starts) >= 2 else starts
    evs, starts = evs[:starts[-1]], starts[:1]
last = evs[starts[-1]:] if starts else evs
t0 = last[0].time_range.start
prev_end = t0
busy = 0.0
for e in last:
    s, d = e.time_range.start, e.time_range.end - e.time_range.start
    gap = s - prev_end
    busy += d
    print(f"{s - t0:9.1f} us  gap {gap:7.1f}  dur {d:7.1f}  {e.name[:70]}")
    prev_end = max(prev_end, e.time_range.end)
span = prev_end - t0
print(f"span {span:.1f} us, busy {busy:.1f} us, idle {span - busy:.1f} us")
