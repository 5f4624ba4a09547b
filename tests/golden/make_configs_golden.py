"""Pin BASELINE configs C1-C5 to the REFERENCE implementation (test infrastructure).

Runs here, where /root/reference exists: oracle/_ref/libtmatch_ref.so is the unmodified
reference compiled by oracle/Makefile.  For every config (paper_1407_3535_b200.workloads,
bit-deterministic generator) it records

  * SHA-256 of the image and of every template (the GPU tests regenerate the inputs and
    assert these, so "same seeded inputs" is checked, not assumed);
  * brute_force_match (stats.cpp:156-213, the reference's own thread pool) per template:
    argmax (row, col), rho bits, degenerate flag;
  * one prepare_egs / prepare_opta (matcher.cpp:205-233) + run_egs / run_opta per template
    (cmd_bench's preparation cache, cli.cpp:213-237) under the reference's frozen
    --parallel policy (threads = nproc >= 2, matcher.cpp:129-143): location, rho bits,
    refined cell, final threshold, centres / eliminated / retained / ops, h_e, kappa;
  * the sequential policy as well where it finishes in reasonable time (C1, C2);
  * the reference's wall times (context for DESIGN.md's CPU-baseline table).

Output: tests/golden/configs/<C>.json (small; committed; read by tests/test_configs*.py
on the GPU box, which never reads /root/reference).

    python tests/golden/make_configs_golden.py C2 C3 ...      (default: all five)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle.binding import Oracle  # noqa: E402
from paper_1407_3535_b200 import workloads as W  # noqa: E402

OUT = os.path.join(HERE, "configs")
SEQUENTIAL = {"C1", "C2", "C6"}  # the running-threshold policy is cheap enough only here


def res_dict(r):
    d = r.as_dict()
    out = {k: int(d[k]) for k in ("best_row", "best_col", "best_degenerate", "refined_row",
                                  "refined_col", "below_threshold", "centers", "eliminated",
                                  "retained", "ops", "extent_rows", "extent_cols")}
    for k in ("best_rho", "refined_rho", "final_threshold", "elim_pct"):
        out[k] = float(d[k]).hex()
    out["wall_ms"] = float(d["wall_ms"])
    return out


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def run(name, ref, threads):
    t0 = time.time()
    wl = W.make(name)
    img = wl.image.astype(np.float64)
    tm = [t.pixels.astype(np.float64) for t in wl.templates]
    out = {"config": name, "description": wl.description, "mode": wl.mode,
           "sha256": wl.sha256(), "image_sha256": sha(wl.image),
           "template_sha256": [sha(t.pixels) for t in wl.templates],
           "template_cut": [[t.row, t.col] for t in wl.templates],
           "image_shape": list(wl.image.shape), "template_shape": list(tm[0].shape),
           "threads": threads, "generated_s": time.time() - t0}
    print(name, "generated", f"{out['generated_s']:.1f}s", flush=True)

    t1 = time.time()
    out["brute"] = [res_dict(ref.brute_threads(t, img, threads)) for t in tm]
    out["brute_s"] = time.time() - t1
    print(name, "brute", f"{out['brute_s']:.1f}s", flush=True)

    pols = [("frozen", True)] + ([("sequential", False)] if name in SEQUENTIAL else [])
    modes = [wl.mode] + (["opta"] if name in SEQUENTIAL and wl.mode != "opta" else [])
    for mode in modes:
        for pol, par in pols:
            t1 = time.time()
            res, info, prep_ms, run_ms = ref.prepare_run_batch(tm, img, mode=mode,
                                                               parallel=par, threads=threads)
            out[f"{mode}_{pol}"] = {"prep": info | {"lam": float(info["lam"]).hex(),
                                                   "prep_ms": prep_ms},
                                    "results": [res_dict(r) for r in res],
                                    "run_ms": [float(x) for x in run_ms]}
            print(name, mode, pol, f"{time.time() - t1:.1f}s", info, flush=True)
    out["total_s"] = time.time() - t0
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, f"{name}.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(name, "done", f"{out['total_s']:.1f}s", flush=True)


def main():
    names = sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5", "C6"]
    ref = Oracle("ref")
    threads = max(2, os.cpu_count() or 2)
    for nm in names:
        run(nm, ref, threads)


if __name__ == "__main__":
    main()
