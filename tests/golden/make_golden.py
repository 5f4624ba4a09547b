"""Generate tests/golden/*.npz from the REFERENCE implementation itself.

Runs here (where /root/reference exists): oracle/_ref/libtmatch_ref.so is the unmodified
reference library compiled by oracle/Makefile from /root/reference/proj/src.  The fixtures
are small, committed, and travel to the GPU box; nothing at test time reads
/root/reference.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.binding import Oracle  # noqa: E402

RESULT_KEYS = ("best_row", "best_col", "best_rho", "best_degenerate", "refined_row",
               "refined_col", "refined_rho", "below_threshold", "final_threshold", "centers",
               "eliminated", "retained", "ops", "elim_pct")


def res_arr(r):
    d = r.as_dict()
    return np.array([float(d[k]) for k in RESULT_KEYS])


HEAVY = ("ws_mu", "ws_omega", "surface", "egs_map", "opta_image", "opta_map", "blur",
         "fidelity")


def case(ref, name, img, t, extra_modes=True, init_threshold=None, light=False):
    m, n = t.shape
    out = {"image": img, "template": t}
    mu, om, fl = ref.window_stats(img, m, n)
    out.update(ws_mu=mu, ws_omega=om, ws_flat=fl)
    b, surf = ref.brute(t, img, surface=True)
    out.update(brute=res_arr(b), surface=surf)
    e = ref.efficient_group_size(img, m, n)
    out.update(egs_h=np.array([e["h"], e["w"]]), egs_map=e["map"],
               egs_trace=np.array([[x["h"], x["w"], x["central"], x["retained"], x["total"]]
                                   for x in e["trace"]]))
    for mode in ("egs", "opta") if extra_modes else ("egs",):
        for pol, par in (("seq", False), ("frozen", True)):
            r, vis = ref.match(t, img, mode=mode, parallel=par, threads=4, visits=True,
                               init_threshold=init_threshold)
            out[f"{mode}_{pol}"] = res_arr(r)
            out[f"{mode}_{pol}_visits"] = vis
    if extra_modes:
        o = ref.optimize_autocorrelation(img, m, n)
        out.update(opta_image=o["image"], opta_kappa=np.array([o["kappa"]]),
                   opta_h=np.array([o["h"], o["w"]]), opta_map=o["map"],
                   opta_trace=np.array([[x["h"], x["w"], x["cost"], x["restored"]]
                                        for x in o["trace"]]))
        out["blur"] = ref.blur(img)
        out["fidelity"] = ref.blur_fidelity_map(img, out["blur"], m, n)
    if light:  # keep the fixture small: results, visit maps, traces and scalars only
        out = {k: v for k, v in out.items() if k not in HEAVY}
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, sorted(out))


def main():
    ref = Oracle("ref")
    # 1. the reference's own corpus generator (synth.cpp, mt19937_64), as acceptance uses it
    imgs, ents = ref.synth_corpus(96, 96, 1.5, 2, 15, 1, 20260810)
    for k in range(2):
        r, c = ents[k]
        img = imgs[k]
        t = img[r:r + 15, c:c + 15].copy()  # extract_template with gain 1, offset 0
        case(ref, f"synth96_{k}", img, t)
    # 2. the acceptance bundled corpus (256^2, m=31, seed 777, sigma 2.5), first image,
    #    at the experiment's user threshold 0.8 (acceptance.cpp:228-231)
    imgs, ents = ref.synth_corpus(256, 256, 2.5, 1, 31, 1, 777)
    r, c = ents[0]
    case(ref, "acceptance256", imgs[0], imgs[0][r:r + 31, c:c + 31].copy(), init_threshold=0.8,
         light=True)
    # 3. seeded u8 noise with a planted, photometrically perturbed non-square template
    rng = np.random.default_rng(47)
    img = rng.integers(0, 256, size=(64, 80)).astype(np.float64)
    t = np.clip(np.rint(0.9 * img[17:28, 23:36] + 12), 0, 255)
    case(ref, "u8noise_64x80", img, t)
    # 4. BASELINE config 1 workload (512^2 1/f^2 + blur, 32^2), scalar results only
    from paper_1407_3535_b200 import workloads as W
    w = W.config1()
    img = w.image.astype(np.float64)
    t = w.templates[0].pixels.astype(np.float64)
    out = {"image_sha": np.frombuffer(bytes.fromhex(w.sha256()), dtype=np.uint8)}
    for mode in ("brute", "egs", "opta"):
        for pol, par in (("seq", False), ("frozen", True)):
            out[f"{mode}_{pol}"] = res_arr(ref.match(t, img, mode=mode, parallel=par, threads=4))
    np.savez_compressed(os.path.join(HERE, "config1.npz"), **out)
    print("config1", list(out))


if __name__ == "__main__":
    main()
