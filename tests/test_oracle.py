"""CPU: pin the oracle (C restatement, oracle/tmatch_oracle.c) before trusting it.

1. Against golden fixtures produced by the reference itself (tests/golden/make_golden.py).
2. Against the reference library (oracle/_ref) on seeded random cases, when present.
3. Against the known-answer constants of the reference's own unit tests
   (proj/tests/test_*.cpp), re-asserted here.
"""
import numpy as np
import pytest

from conftest import RESULT_KEYS, golden, golden_names, res_vec


@pytest.mark.parametrize("name", golden_names())
def test_port_matches_reference_golden(port, name):
    g = golden(name)
    img, t = g["image"], g["template"]
    m, n = t.shape
    mu, om, fl = port.window_stats(img, m, n)
    np.testing.assert_array_equal(fl, g["ws_flat"])
    if "ws_mu" in g:
        np.testing.assert_array_equal(mu, g["ws_mu"])
        np.testing.assert_array_equal(om, g["ws_omega"])
    b, surf = port.brute(t, img, surface=True)
    np.testing.assert_array_equal(res_vec(b), g["brute"])
    if "surface" in g:
        np.testing.assert_array_equal(surf, g["surface"])
    e = port.efficient_group_size(img, m, n)
    assert [e["h"], e["w"]] == list(g["egs_h"])
    np.testing.assert_array_equal(
        np.array([[x["h"], x["w"], x["central"], x["retained"], x["total"]] for x in e["trace"]]),
        g["egs_trace"])
    if "egs_map" in g:
        np.testing.assert_array_equal(e["map"], g["egs_map"])
    init = 0.8 if name == "acceptance256" else None
    for mode in ("egs", "opta"):
        for pol, par in (("seq", False), ("frozen", True)):
            r, vis = port.match(t, img, mode=mode, parallel=par, threads=4, visits=True,
                                init_threshold=init)
            np.testing.assert_array_equal(res_vec(r), g[f"{mode}_{pol}"], err_msg=f"{mode} {pol}")
            np.testing.assert_array_equal(vis, g[f"{mode}_{pol}_visits"])
    o = port.optimize_autocorrelation(img, m, n)
    assert o["kappa"] == int(g["opta_kappa"][0])
    np.testing.assert_array_equal(
        np.array([[x["h"], x["w"], x["cost"], x["restored"]] for x in o["trace"]]),
        g["opta_trace"])
    if "opta_image" in g:
        np.testing.assert_array_equal(o["image"], g["opta_image"])
        np.testing.assert_array_equal(o["map"], g["opta_map"])
        np.testing.assert_array_equal(port.blur(img), g["blur"])
        np.testing.assert_array_equal(port.blur_fidelity_map(img, g["blur"], m, n),
                                      g["fidelity"])


def test_port_matches_reference_config1(port):
    from paper_1407_3535_b200 import workloads as W
    g = golden("config1")
    w = W.config1()
    assert bytes(g["image_sha"]).hex() == w.sha256(), "C1 generator drifted"
    img = w.image.astype(np.float64)
    t = w.templates[0].pixels.astype(np.float64)
    for mode in ("brute", "egs", "opta"):
        for pol, par in (("seq", False), ("frozen", True)):
            r = port.match(t, img, mode=mode, parallel=par, threads=4)
            np.testing.assert_array_equal(res_vec(r), g[f"{mode}_{pol}"], err_msg=f"{mode} {pol}")


def _random_cases():
    rng = np.random.default_rng(2026)
    cases = []
    for k in range(10):
        p, q = rng.integers(20, 70, size=2)
        m, n = rng.integers(3, 14, size=2)
        smooth = k % 2 == 0
        img = rng.integers(0, 256, size=(p, q)).astype(np.float64)
        if smooth:  # correlated content so elimination actually happens
            img = np.rint(np.cumsum(np.cumsum(rng.normal(size=(p, q)), 0), 1))
            img = np.clip(img - img.min(), 0, 255)
        r0, c0 = rng.integers(0, p - m + 1), rng.integers(0, q - n + 1)
        t = np.clip(np.rint(img[r0:r0 + m, c0:c0 + n] * 0.9 + 7 + rng.normal(0, 2, (m, n))),
                    0, 255)
        cases.append((img, t))
    return cases


@pytest.mark.parametrize("idx", range(10))
def test_port_vs_reference_library(port, ref, idx):
    img, t = _random_cases()[idx]
    for mode in ("brute", "egs", "opta"):
        for par in (False, True):
            a, va = port.match(t, img, mode=mode, parallel=par, threads=3, visits=True)
            b, vb = ref.match(t, img, mode=mode, parallel=par, threads=3, visits=True)
            np.testing.assert_array_equal(res_vec(a), res_vec(b), err_msg=f"{mode} {par}")
            if mode != "brute":
                np.testing.assert_array_equal(va, vb)


def test_port_vs_reference_nonuniform_blur_image(port, ref):
    # non-integer search image (the OptA search domain): FP64 op order must match
    img, t = _random_cases()[0]
    b = port.blur(img)
    np.testing.assert_array_equal(b, ref.blur(img))
    m, n = t.shape
    for a, r in zip(port.window_stats(b, m, n), ref.window_stats(b, m, n)):
        np.testing.assert_array_equal(a, r)
    np.testing.assert_array_equal(port.local_autocorrelation(b, m, n, 5, 5),
                                  ref.local_autocorrelation(b, m, n, 5, 5))
    np.testing.assert_array_equal(res_vec(port.brute(t, b)), res_vec(ref.brute(t, b)))


# ---- known answers from the reference unit tests ------------------------------------------

def test_window_stats_hand_example(port):
    # test_stats.cpp:54-64: {0,0,255,255} -> mu 127.5, omega 255
    img = np.array([[0.0, 0.0, 255.0, 255.0]])
    mu, om, fl = port.window_stats(img, 1, 4)
    assert mu[0, 0] == 127.5 and om[0, 0] == 255.0 and fl[0, 0] == 0


def test_bounds_hand_values(port):
    lo, hi = port.transitive_bounds(0.61, 0.81)  # test_bounds.cpp:22-30
    assert abs(lo - 0.0294) < 1e-4 and abs(hi - 0.9588) < 1e-4
    assert abs(port.transitive_gap(0.61, 0.81) - 0.9294) < 1e-4
    assert port.transitive_bounds(1.0, 0.3) == (0.3, 0.3)
    assert port.transitive_bounds(0.0, 0.0) == (-1.0, 1.0)
    assert abs(port.expected_elimination_threshold(0.8) - 0.6) < 1e-12  # test_bounds.cpp:81
    assert abs(port.quality_threshold(0.8, 0.95) - 0.947349939) < 1e-6  # test_blur.cpp:92
    assert abs(port.quality_threshold(0.8, 1.0) - 0.8) < 1e-12  # test_blur.cpp:91
    with pytest.raises(ValueError):
        port.transitive_bounds(1.5, 0.2)
    assert port.sec_holds(1.0, 0.5, 0.5) is True


def test_grid_counts(port):
    assert port.group_count(9, 9, 3, 3) == 9      # test_autocorr.cpp:12-22
    assert port.group_count(10, 10, 3, 3) == 16   # test_autocorr.cpp:24-34
    with pytest.raises(ValueError):
        port.group_count(10, 10, 2, 3)


def test_ramp_autocorrelation_is_one(port):
    # test_autocorr.cpp:71-78: I(r,c) = c makes every member perfectly correlated
    img = np.tile(np.arange(40, dtype=np.float64), (30, 1))
    amap = port.local_autocorrelation(img, 7, 7, 5, 5)
    np.testing.assert_allclose(amap, 1.0, atol=1e-12)


def test_brute_planted_and_constant(port):
    rng = np.random.default_rng(47)  # test_stats.cpp:132-154 (layout, our RNG)
    img = rng.integers(0, 256, size=(64, 80)).astype(np.float64)
    t = img[17:28, 23:36].copy()
    r = port.brute(t, img)
    assert (r.best_row, r.best_col) == (17, 23) and abs(r.best_rho - 1.0) < 1e-12
    assert r.ops == 54 * 68
    flat = np.full((20, 20), 7.0)
    r = port.brute(t[:5, :5], flat)
    assert (r.best_row, r.best_col, r.best_rho, r.best_degenerate) == (0, 0, 0.0, 1)


def test_total_cost_examples(port):
    # egs.cpp:27-37 via the egs trace on uniform maps is indirect; check the closed form
    # test_egs.cpp:72-89: (100^2, 5) -> 400, (10^2, 3) -> 16 groups, clipped ceil tiling
    assert port.group_count(100, 100, 5, 5) == 400
    assert port.group_count(10, 10, 3, 3) == 16
    assert port.group_count(9, 9, 3, 3) + 10 == 19


def test_result_layout_matches_c_header():
    import ctypes as C

    from oracle.binding import TmoResult
    from paper_1407_3535_b200.native import MatchResult
    assert C.sizeof(TmoResult) == C.sizeof(MatchResult)
    assert [f for f, _ in TmoResult._fields_] == [f for f, _ in MatchResult._fields_]
    assert set(RESULT_KEYS) <= {f for f, _ in MatchResult._fields_}
