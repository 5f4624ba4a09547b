"""Brute-force search of a NON-INTEGER image: split tensor-core screening vs the FP64 replica.

    python tools/split_probe.py [size] [m]      (TMATCH_TC_SPLIT=0 -> FP64 replica only)

Prints one JSON line per run: ms per search (CUDA events on the context stream), the
screened / exactly re-evaluated location counts and the result.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1407_3535_b200 import api, workloads as W  # noqa: E402


def main():
    size = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    rng = np.random.default_rng(11)
    img = np.asarray(W.spectral_image(21, size, size, 2.0, 1.0), dtype=np.float64)
    r0, c0 = size // 3, size // 2
    t = np.clip(np.rint(img[r0:r0 + m, c0:c0 + m] * 0.95 + 5 + rng.normal(0, 6, (m, m))), 0, 255)
    with api.Context(0) as ctx:
        integer = os.environ.get("PROBE_INTEGER") == "1"  # the 8-bit kind::i8 pass for scale
        blurred = img if integer else ctx.blur(img)
        g = ctx.image(blurred)
        stream = torch.cuda.ExternalStream(ctx.stream_ptr)
        res = ctx.brute_force_match(t, g)  # warm-up: planes, geometry, window statistics
        s0 = ctx.split_stats()
        steps = 5
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(steps):
            res = ctx.brute_force_match(t, g)
        b.record(stream)
        b.synchronize()
        s1 = ctx.split_stats()
        ms = a.elapsed_time(b) / steps
        E = (size - m + 1) ** 2
        print(json.dumps({
            "image": f"{size}x{size} " + ("8-bit" if integer else "blurred (non-integer)"), "template": f"{m}x{m}",
            "split": os.environ.get("TMATCH_TC_SPLIT", "1") != "0", "ms_per_search": ms,
            "locations_per_s": E / ms * 1e3, "macs_per_s": E * m * m / ms * 1e3,
            "screened_per_search": (s1["screened"] - s0["screened"]) // steps,
            "exact_per_search": (s1["exact"] - s0["exact"]) // steps,
            "best": [res.best_row, res.best_col, res.best_rho]}))


if __name__ == "__main__":
    main()
