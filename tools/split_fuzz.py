"""Randomised differential check of the split-plane paths against the oracle.

    python tools/split_fuzz.py [cases] [seed]        (FUZZ_INTEGER=1: 8-bit images -> the
                                                      kind::i8 passes and their FP32 pre-test;
                                                      FUZZ_LARGE=1: wide images, half the
                                                      templates without a match)

Non-integer images of random shape / smoothness / contrast (near-flat patches, values at
both ends of [0, 256), exact duplicates of the best window), integer templates; brute force
and transitive search under all three policies; every field and the visit map must equal
the oracle's.  Prints one line per mismatch and a summary.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.binding import Oracle  # noqa: E402  (checker only)
from paper_1407_3535_b200 import api  # noqa: E402

os.environ.setdefault("TMATCH_TC_SPLIT", "2")  # force the split planes on small images too

KEYS = ("best_row", "best_col", "best_rho", "best_degenerate", "final_threshold", "centers",
        "eliminated", "retained", "ops")


def make_case(rng):
    p, q = int(rng.integers(24, 220)), int(rng.integers(24, 260))
    if os.environ.get("FUZZ_LARGE") == "1":  # several 2048-column tiles, dense survivor rows
        p, q = int(rng.integers(300, 700)), int(rng.integers(1800, 2700))
    m, n = int(rng.integers(2, min(p, 70))), int(rng.integers(2, min(q, 70)))
    kind = rng.integers(0, 4)
    if kind == 0:
        base = np.cumsum(np.cumsum(rng.normal(size=(p, q)), 0), 1)
    elif kind == 1:
        base = rng.normal(size=(p, q))
    elif kind == 2:
        base = np.cumsum(rng.normal(size=(p, q)), 1) + 5 * (rng.random((p, q)) < 0.02)
    else:
        base = np.add.outer(np.sin(np.arange(p) / 3.0), np.cos(np.arange(q) / 5.0))
    lo, hi = sorted(rng.uniform(0, 255.99, 2))
    if hi - lo < 1.0:
        hi = min(255.99, lo + 1.0 + rng.random() * 20)
    img = (base - base.min()) / (np.ptp(base) + 1e-12) * (hi - lo) + lo
    img = img + rng.random((p, q)) * 2.0 ** -int(rng.integers(1, 30))  # fractional bits
    img = np.clip(img, 0.0, 255.99609375)
    if os.environ.get("FUZZ_INTEGER") == "1":  # the 8-bit tensor-core passes instead
        img = np.rint(np.clip(img, 0, 255))
    if rng.random() < 0.3:  # a near-flat patch
        r0, c0 = int(rng.integers(0, p - 3)), int(rng.integers(0, q - 3))
        img[r0:r0 + p // 3, c0:c0 + q // 3] = img[r0, c0] + rng.random() * 1e-9
    if os.environ.get("FUZZ_INTEGER") == "1":
        img = np.rint(img)
    r0, c0 = int(rng.integers(0, p - m + 1)), int(rng.integers(0, q - n + 1))
    t = np.clip(np.rint(img[r0:r0 + m, c0:c0 + n] * rng.uniform(0.8, 1.2) +
                        rng.uniform(-10, 10) + rng.normal(0, rng.uniform(0, 6), (m, n))), 0, 255)
    if os.environ.get("FUZZ_LARGE") == "1" and rng.random() < 0.5:
        t = np.clip(np.rint(rng.normal(128, 50, (m, n))), 0, 255)  # no match: weak elimination
    if rng.random() < 0.25:  # plant an exact duplicate of the cut window
        r1, c1 = int(rng.integers(0, p - m + 1)), int(rng.integers(0, q - n + 1))
        img[r1:r1 + m, c1:c1 + n] = img[r0:r0 + m, c0:c0 + n]
    h = int(rng.choice([1, 3, 5, 7]))
    w = int(rng.choice([1, 3, 5]))
    return img, t, h, w


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2024)
    port = Oracle("port")
    bad = 0
    split_used = 0
    with api.Context(0) as ctx:
        for k in range(cases):
            img, t, h, w = make_case(rng)
            if np.ptp(t) == 0:
                continue
            g = ctx.image(img)
            s0 = ctx.split_stats()["screened"]
            a, b = ctx.brute_force_match(t, g), port.brute(t, img)
            da, db = a.as_dict(), b.as_dict()
            diffs = {f: (da[f], db[f]) for f in KEYS[:4] if da[f] != db[f]}
            amap = port.local_autocorrelation(img, t.shape[0], t.shape[1], h, w)
            for par in (True, False):
                x, vx = ctx.transitive_search(t, g, amap, h, w, parallel=par, threads=3,
                                              record_visits=True)
                y, vy = port.transitive_search(t, img, amap, h, w, parallel=par, threads=3,
                                               visits=True)
                dx, dy = x.as_dict(), y.as_dict()
                diffs.update({f"{f}/par={par}": (dx[f], dy[f]) for f in KEYS if dx[f] != dy[f]})
                if not np.array_equal(vx, vy):
                    diffs[f"visits/par={par}"] = int(np.sum(vx != vy))
            z = ctx.transitive_search(t, g, amap, h, w, policy="seeded")
            if (z.best_row, z.best_col, z.best_rho) != (b.best_row, b.best_col, b.best_rho):
                diffs["seeded"] = ((z.best_row, z.best_col, z.best_rho),
                                   (b.best_row, b.best_col, b.best_rho))
            split_used += ctx.split_stats()["screened"] > s0
            if diffs:
                bad += 1
                print(f"case {k}: image {img.shape} template {t.shape} h,w={h},{w}: {diffs}")
            g.close()
    print(f"{cases} cases, {split_used} through the split planes, {bad} mismatching")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
