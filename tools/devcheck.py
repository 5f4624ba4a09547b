"""Developer smoke check: GPU path vs the C oracle on small seeded inputs (prints a table)."""
import sys
import time
import traceback

import numpy as np

sys.path.insert(0, ".")
from oracle.binding import Oracle  # noqa: E402
from paper_1407_3535_b200 import api, workloads as W  # noqa: E402


def cmp(name, a, b):
    a, b = np.asarray(a), np.asarray(b)
    same = a.shape == b.shape and np.array_equal(a, b)
    diff = "" if same else f" maxdiff={np.max(np.abs(a.astype(float) - b.astype(float))) if a.shape == b.shape else 'shape'}" \
        f" n={int(np.sum(a != b)) if a.shape == b.shape else -1}"
    print(f"{'OK ' if same else 'BAD'} {name}{diff}", flush=True)
    return same


def res_cmp(name, g, o, keys=("best_row", "best_col", "best_rho", "best_degenerate",
                              "refined_row", "refined_col", "refined_rho", "eliminated",
                              "retained", "centers", "ops", "final_threshold", "below_threshold")):
    gd, od = g.as_dict(), o.as_dict()
    bad = {k: (gd[k], od[k]) for k in keys if gd[k] != od[k]}
    print(f"{'OK ' if not bad else 'BAD'} {name} {bad if bad else ''} "
          f"gpu_ms={gd['wall_ms']:.3f} elim={gd['elim_pct']:.2f}", flush=True)
    return not bad


def main():
    port = Oracle("port")
    ctx = api.Context(0)
    w = W.config1()
    img_u8 = w.image
    img = img_u8.astype(np.float64)
    t = w.templates[0].pixels.astype(np.float64)
    m, n = t.shape
    steps = []

    def step(fn):
        try:
            fn()
        except Exception:
            traceback.print_exc()

    gi = ctx.image(img)
    print("integer image:", gi.is_integer)
    step(lambda: cmp("window_stats", np.concatenate([x.ravel().astype(float) for x in ctx.window_stats(gi, m, n)]),
                     np.concatenate([x.ravel().astype(float) for x in port.window_stats(img, m, n)])))
    step(lambda: cmp("running_sum", ctx.running_sum(gi, m, n), port.running_sum(img, m, n)))

    def brute():
        g, gs = ctx.brute_force_match(t, gi, record_surface=True)
        o, os_ = port.brute(t, img, surface=True)
        res_cmp("brute", g, o)
        cmp("brute surface", gs, os_)
    step(brute)
    for h in (1, 3, 5, 7, 9):
        step(lambda h=h: cmp(f"autocorr h={h}", ctx.local_autocorrelation(gi, m, n, h, h),
                             port.local_autocorrelation(img, m, n, h, h)))

    def egs():
        g = ctx.efficient_group_size(gi, m, n)
        o = port.efficient_group_size(img, m, n)
        print("egs gpu", g["h"], [(x["h"], x["total"]) for x in g["trace"]])
        print("egs ora", o["h"], [(x["h"], x["total"]) for x in o["trace"]])
        cmp("egs map", g["map"], o["map"])
    step(egs)
    for mode in ("egs", "opta"):
        for pol, par in (("frozen", True), ("sequential", False)):
            def run(mode=mode, pol=pol, par=par):
                t0 = time.time()
                g, gv = ctx.match(t, img, mode=mode, policy=pol, parallel=par, threads=4,
                                  record_visits=True)
                t1 = time.time()
                o, ov = port.match(t, img, mode=mode, parallel=par, threads=4, visits=True)
                res_cmp(f"match {mode} {pol} ({t1 - t0:.2f}s)", g, o)
                cmp(f"visits {mode} {pol}", gv, ov)
            step(run)
        step(lambda mode=mode: print("seeded", mode, ctx.match(t, img, mode=mode, policy="seeded")))
    # blur pieces
    step(lambda: cmp("blur", ctx.blur(img), port.blur(img)))
    b = port.blur(img)
    step(lambda: cmp("fidelity", ctx.blur_fidelity_map(img, b, m, n), port.blur_fidelity_map(img, b, m, n)))
    # non-integer image path: search on blurred image
    def nonint():
        gb = ctx.image(b)
        print("blurred integer?", gb.is_integer)
        cmp("ws blurred", np.concatenate([x.ravel().astype(float) for x in ctx.window_stats(gb, m, n)]),
            np.concatenate([x.ravel().astype(float) for x in port.window_stats(b, m, n)]))
        cmp("autocorr blurred h=3", ctx.local_autocorrelation(gb, m, n, 3, 3),
            port.local_autocorrelation(b, m, n, 3, 3))
        g = ctx.brute_force_match(t, gb)
        o = port.brute(t, b)
        res_cmp("brute blurred", g, o)
    step(nonint)
    print("launches", ctx.launches)


if __name__ == "__main__":
    main()
