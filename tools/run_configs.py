"""Run the five BASELINE.json configs on one GPU and check size-independent properties.

For every template: the seeded, frozen (and, for small extents, sequential) searches must
return the brute-force argmax (location and rho bits; brute force = the exact sm_100a
dense kernel), and every eliminated member must satisfy rho <= final threshold on the
brute-force surface (soundness, acceptance.cpp:105-116); for EGS configs tm_search (the
fused single-call path) must equal prepare + run.  Timings are device-synchronous
wall clock around each API call.  Prints one JSON object per config.

    python tools/run_configs.py C1 C2 C3 C4 C5 [--no-sequential]
"""
import faulthandler
import json
import sys
import time

faulthandler.enable()

import numpy as np

sys.path.insert(0, ".")
from paper_1407_3535_b200 import api, workloads as W  # noqa: E402


def run(name, seq=True):
    t0 = time.perf_counter()
    wl = W.make(name)
    gen_s = time.perf_counter() - t0
    ctx = api.Context(0)
    img = ctx.image(wl.image)
    m, n = wl.templates[0].pixels.shape
    out = dict(config=name, shape=list(wl.image.shape), template=[m, n],
               templates=len(wl.templates), mode=wl.mode, extent=wl.extent, gen_s=gen_s,
               sha256=wl.sha256()[:16], results=[])
    print(f"{name} generated {gen_s:.1f}s; preparing", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    prep = ctx.prepare(img, m, n, mode=wl.mode)
    out["prep_wall_ms"] = (time.perf_counter() - t0) * 1e3
    out["prep_device_ms"] = prep.info["prep_ms"]
    out["h_e"] = prep.info["h"]
    out["kappa"] = prep.info["kappa"]
    search_img = ctx.image(prep.search_image()) if wl.mode == "opta" else img
    for k, tp in enumerate(wl.templates):
        print(f"{name} template {k}", file=sys.stderr, flush=True)
        t = tp.pixels
        rec = dict(k=k, truth=[tp.row, tp.col])
        t0 = time.perf_counter()
        b, surf = ctx.brute_force_match(t, img, record_surface=True)
        rec["brute_ms"] = (time.perf_counter() - t0) * 1e3
        rec["brute"] = [b.best_row, b.best_col, b.best_rho]
        if wl.mode == "opta":
            _, surf_s = ctx.brute_force_match(t, search_img, record_surface=True)
        else:
            surf_s = surf
        pols = ["seeded", "frozen"] + (["sequential"] if seq else [])
        ok = True
        for pol in pols:
            t0 = time.perf_counter()
            r, vis = ctx.run(prep, t, policy=pol, parallel=(pol == "frozen"), threads=2,
                             record_visits=True)
            ms = (time.perf_counter() - t0) * 1e3
            loc = (r.refined_row, r.refined_col, r.refined_rho)
            same = loc == (b.best_row, b.best_col, b.best_rho)
            sound = bool(np.all(surf_s[vis == 1] <= r.final_threshold + 1e-9))
            ok = ok and same and sound
            rec[pol] = dict(ms=ms, refined=list(loc), elim_pct=r.elim_pct, retained=r.retained,
                            eliminated=r.eliminated, ops=r.ops, argmax_equals_brute=same,
                            sound=sound, final_threshold=r.final_threshold)
        if wl.mode == "egs":
            # tm_search (prepare + run in one call; scan 2 fused into the R_co launch of the
            # predicted group size) must give exactly the prepare + run result
            for pol in ("seeded", "frozen"):
                t0 = time.perf_counter()
                r = ctx.search(img, t, mode="egs", policy=pol, parallel=(pol == "frozen"),
                               threads=2)
                ms = (time.perf_counter() - t0) * 1e3
                same = ([r.best_row, r.best_col, r.best_rho, r.eliminated, r.retained, r.ops,
                         r.final_threshold] ==
                        [rec[pol]["refined"][0], rec[pol]["refined"][1], rec[pol]["refined"][2],
                         rec[pol]["eliminated"], rec[pol]["retained"], rec[pol]["ops"],
                         rec[pol]["final_threshold"]])
                rec[f"search_{pol}"] = dict(ms=ms, equals_prepare_run=same)
                ok = ok and same
        rec["ok"] = ok
        out["results"].append(rec)
    out["all_ok"] = all(r["ok"] for r in out["results"])
    prep.close()
    ctx.close()
    return out


if __name__ == "__main__":
    names = [a for a in sys.argv[1:] if not a.startswith("--")] or ["C1", "C2", "C3"]
    for nm in names:
        print(json.dumps(run(nm, seq="--no-sequential" not in sys.argv)), flush=True)
