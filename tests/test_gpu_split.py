"""Split tensor-core screening of NON-INTEGER search images (k_tc.cu "split planes").

The reference evaluates window_dot (detail.hpp:32-41) on FP64 pixels in sequence; the
B200 path brackets every rho on three byte planes with tcgen05 kind::i8 and re-evaluates
only the locations that can still win with the FP64 replica.  The bar is the same as
everywhere else: results bit-identical to the oracle (which is pinned to the reference).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import RESULT_KEYS, assert_same_result

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ctx():
    """A context with the split planes forced (TMATCH_TC_SPLIT=2): by default passes below a
    work threshold stay on the FP64 replica, and these tests use small images."""
    from paper_1407_3535_b200 import api
    old = os.environ.get("TMATCH_TC_SPLIT")
    os.environ["TMATCH_TC_SPLIT"] = "2"
    try:
        c = api.Context(0)
    finally:
        if old is None:
            os.environ.pop("TMATCH_TC_SPLIT", None)
        else:
            os.environ["TMATCH_TC_SPLIT"] = old
    yield c
    c.close()


def _image(rng, p, q, smooth=True):
    base = np.cumsum(np.cumsum(rng.normal(size=(p, q)), 0), 1) if smooth else rng.normal(size=(p, q))
    return np.clip(np.rint((base - base.min()) / (np.ptp(base) + 1e-9) * 255), 0, 255)


def _template(rng, img, m, n, noise=3.0):
    p, q = img.shape
    r0, c0 = int(rng.integers(0, p - m + 1)), int(rng.integers(0, q - n + 1))
    return np.clip(np.rint(img[r0:r0 + m, c0:c0 + n] * 1.1 - 5 + rng.normal(0, noise, (m, n))),
                   0, 255)


SHAPES = [(96, 96, 16, 16), (70, 131, 33, 31), (128, 96, 17, 64), (40, 2100, 8, 8),
          (300, 260, 64, 64), (61, 61, 5, 3)]


@pytest.mark.parametrize("idx", range(len(SHAPES)))
def test_brute_on_blurred_image_equals_oracle(ctx, port, idx):
    p, q, m, n = SHAPES[idx]
    rng = np.random.default_rng(100 + idx)
    img = _image(rng, p, q, smooth=idx % 2 == 0)
    if idx == 2:
        img[10:60, 5:50] = 77.0  # flat windows (degenerate locations never win)
    t = _template(rng, img, m, n)
    blurred = port.blur(img)
    assert np.any(blurred != np.rint(blurred))
    g = ctx.image(blurred)
    assert not g.is_integer
    s0 = ctx.split_stats()
    a = ctx.brute_force_match(t, g)
    s1 = ctx.split_stats()
    b = port.brute(t, blurred)
    assert_same_result(a, b, keys=RESULT_KEYS[:-1])
    E = (p - m + 1) * (q - n + 1)
    assert s1["screened"] - s0["screened"] == E, "the split tensor-core pass did not run"
    assert 1 <= s1["exact"] - s0["exact"] <= max(16, E // 50)


def test_brute_ties_and_near_ties(ctx, port):
    """Exact duplicates of the best window: better_candidate's (row, col) order decides, so
    every tied location must survive the screening."""
    rng = np.random.default_rng(5)
    img = _image(rng, 90, 120)
    blurred = port.blur(img)
    patch = blurred[20:36, 30:46].copy()
    for (r, c) in ((50, 70), (3, 100), (70, 2)):
        blurred[r:r + 16, c:c + 16] = patch
    t = np.clip(np.rint(patch), 0, 255)
    a = ctx.brute_force_match(t, ctx.image(blurred))
    b = port.brute(t, blurred)
    assert_same_result(a, b, keys=RESULT_KEYS[:-1])
    # a copy that differs by less than the screening radius
    blurred[50, 70] += 2.0 ** -20
    a = ctx.brute_force_match(t, ctx.image(blurred))
    b = port.brute(t, blurred)
    assert_same_result(a, b, keys=RESULT_KEYS[:-1])


def test_out_of_range_and_flat_fall_back(ctx, port):
    rng = np.random.default_rng(9)
    img = _image(rng, 64, 64)
    t = _template(rng, img, 9, 9)
    for f in (lambda x: x * 1.5 + 0.25, lambda x: x - 40.5):  # pixels >= 256 / negative
        im2 = f(port.blur(img))
        s0 = ctx.split_stats()
        a = ctx.brute_force_match(t, ctx.image(im2))
        assert ctx.split_stats() == s0  # FP64 replica
        assert_same_result(a, port.brute(t, im2), keys=RESULT_KEYS[:-1])
    flat = np.full((40, 40), 12.25)
    a = ctx.brute_force_match(t, ctx.image(flat))
    assert_same_result(a, port.brute(t, flat), keys=RESULT_KEYS[:-1])


def test_split_switch_off_is_the_fp64_replica():
    code = (
        "import numpy as np\n"
        "from oracle.binding import Oracle\n"
        "from paper_1407_3535_b200 import api\n"
        "rng = np.random.default_rng(3)\n"
        "img = np.clip(np.rint(rng.normal(128, 40, (80, 80))), 0, 255)\n"
        "port = Oracle('port')\n"
        "b = port.blur(img)\n"
        "t = np.clip(np.rint(b[10:26, 20:36]), 0, 255)\n"
        "with api.Context(0) as ctx:\n"
        "    a = ctx.brute_force_match(t, ctx.image(b))\n"
        "    assert ctx.split_stats() == {'screened': 0, 'exact': 0}\n"
        "    o = port.brute(t, b)\n"
        "    assert (a.best_row, a.best_col, a.best_rho) == (o.best_row, o.best_col, o.best_rho)\n"
        "print('ok')\n")
    env = dict(os.environ, TMATCH_TC_SPLIT="0", PYTHONPATH=ROOT)
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=ROOT, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


# ---- scan 1 on the split planes (transitive search of a non-integer image) ---------------
SEARCH_SHAPES = [(96, 96, 16, 16, 3, 3), (70, 131, 33, 31, 5, 5), (128, 96, 17, 64, 3, 5),
                 (40, 2100, 8, 8, 3, 3), (300, 260, 64, 64, 5, 5), (61, 61, 5, 3, 7, 3),
                 (200, 180, 24, 24, 1, 1)]


@pytest.mark.parametrize("idx", range(len(SEARCH_SHAPES)))
def test_search_on_blurred_image_equals_oracle(ctx, port, idx):
    """Both reference policies (--parallel frozen scan, default sequential scan): counts,
    visit codes, threshold and result bit-identical to the oracle, with scan 1 bracketed on
    the tensor cores."""
    p, q, m, n, h, w = SEARCH_SHAPES[idx]
    rng = np.random.default_rng(200 + idx)
    img = _image(rng, p, q, smooth=idx % 2 == 0)
    if idx == 2:
        img[10:60, 5:50] = 77.0  # flat windows: degenerate centres and flat members
    t = _template(rng, img, m, n, noise=1.0 + idx)
    blurred = port.blur(img)
    amap = port.local_autocorrelation(blurred, m, n, h, w)
    g = ctx.image(blurred)
    er, ec = p - m + 1, q - n + 1
    G = -(-er // h) * -(-ec // w)
    # parallel=True: frozen threshold; parallel=False: the reference's default sequential scan
    # (running threshold), replayed exactly -- both with scan 1 on the split planes
    for par in (True, False):
        for init in (None, 0.5):
            s0 = ctx.split_stats()
            a, va = ctx.transitive_search(t, g, amap, h, w, parallel=par, threads=3,
                                          record_visits=True, init_threshold=init)
            b, vb = port.transitive_search(t, blurred, amap, h, w, parallel=par, threads=3,
                                           visits=True, init_threshold=init)
            np.testing.assert_array_equal(va, vb, err_msg=f"par={par} init={init}")
            assert_same_result(a, b, keys=RESULT_KEYS[:-1], msg=f"par={par} init={init}")
            # G centres (+ E when a large survivor set took the masked split pass)
            assert ctx.split_stats()["screened"] - s0["screened"] in (G, G + er * ec), \
                "split centre scan did not run"


@pytest.mark.parametrize("idx", [0, 1, 4])
def test_seeded_search_on_blurred_image(ctx, port, idx):
    """Seeded policy: same argmax / rho as brute force, sound eliminations, consistent counts."""
    p, q, m, n, h, w = SEARCH_SHAPES[idx]
    rng = np.random.default_rng(300 + idx)
    img = _image(rng, p, q)
    t = _template(rng, img, m, n)
    blurred = port.blur(img)
    amap = port.local_autocorrelation(blurred, m, n, h, w)
    b, surface = port.brute(t, blurred, surface=True)
    a, vis = ctx.transitive_search(t, ctx.image(blurred), amap, h, w, policy="seeded",
                                   record_visits=True)
    assert (a.best_row, a.best_col, a.best_rho) == (b.best_row, b.best_col, b.best_rho)
    assert np.all(surface[vis == 1] <= a.final_threshold + 1e-9)
    assert a.eliminated + a.retained + a.centers == b.ops


def test_opta_match_with_blur_uses_split_planes(ctx, port):
    """match(mode=opta) whose optimised image is blurred (kappa > 0): prepare + frozen run
    equal to the oracle, scan 1 on the split planes."""
    rng = np.random.default_rng(17)
    img = _image(rng, 160, 160, smooth=False)
    t = _template(rng, img, 16, 16, noise=2.0)
    s0 = ctx.split_stats()
    a, va = ctx.match(t, img, mode="opta", parallel=True, threads=3, record_visits=True)
    b, vb = port.match(t, img, mode="opta", parallel=True, threads=3, visits=True)
    np.testing.assert_array_equal(va, vb)
    assert_same_result(a, b)


def test_many_survivors_are_bracketed_then_replayed(ctx, port):
    """Weak elimination (a template without a true match) under the frozen policy: the
    survivors' rho only matter for the argmax, so they are bracketed by one masked split pass
    and the near-maximal ones replayed -- same result, counts and visit codes."""
    rng = np.random.default_rng(77)
    img = _image(rng, 400, 380)
    blurred = port.blur(img)
    t = np.clip(np.rint(rng.normal(128, 50, (16, 16))), 0, 255)
    h = w = 3
    amap = port.local_autocorrelation(blurred, 16, 16, h, w)
    g = ctx.image(blurred)
    E = (400 - 15) * (380 - 15)
    G = -(-(400 - 15) // h) * -(-(380 - 15) // w)
    for policy in ("frozen", "seeded"):
        s0 = ctx.split_stats()
        a, va = ctx.transitive_search(t, g, amap, h, w, policy=policy, record_visits=True)
        if policy == "frozen":
            b, vb = port.transitive_search(t, blurred, amap, h, w, parallel=True, threads=3,
                                           visits=True)
            np.testing.assert_array_equal(va, vb)
            assert_same_result(a, b, keys=RESULT_KEYS[:-1])
            assert a.retained > max(9472, E // 64), "workload does not reach the split pass"
            assert ctx.split_stats()["screened"] - s0["screened"] == G + E
        else:
            bb = port.brute(t, blurred)
            assert (a.best_row, a.best_col, a.best_rho) == (bb.best_row, bb.best_col, bb.best_rho)


def test_candidate_list_overflow_falls_back_to_the_replica(ctx, port):
    """A periodic non-integer image whose template matches exactly at every second row and
    column: more than 2^20 tied candidates survive the screening, the list overflows and the
    dense FP64 replica decides (first tie in (row, col) order, as better_candidate says)."""
    cell = np.array([[10.25, 200.5], [77.75, 31.125]])
    img = np.tile(cell, (1050, 1050))
    t = np.tile(np.array([[10.0, 200.0], [78.0, 31.0]]), (8, 8))
    g = ctx.image(img)
    assert not g.is_integer
    s0 = ctx.split_stats()
    a = ctx.brute_force_match(t, g)
    assert ctx.split_stats()["exact"] == s0["exact"], "expected the overflow fallback"
    b = port.brute(t, img)
    assert_same_result(a, b, keys=RESULT_KEYS[:-1])
    assert (a.best_row, a.best_col) == (0, 0)


def test_randomised_differential_sample():
    """A short run of tools/split_fuzz.py (random non-integer images, every policy, visit maps
    and all result fields against the oracle)."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "split_fuzz.py"), "60", "5"],
                         cwd=ROOT, env=dict(os.environ, PYTHONPATH=ROOT), capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0 and "0 mismatching" in out.stdout, out.stdout[-3000:] + out.stderr[-2000:]


def test_default_threshold_keeps_tiny_passes_on_the_replica(port):
    """Default mode (TMATCH_TC_SPLIT unset): a 96x96 search stays on the FP64 replica (faster
    there), a 600x600 one takes the split planes; both equal the oracle."""
    from paper_1407_3535_b200 import api
    rng = np.random.default_rng(4)
    with api.Context(0) as c:
        for size, m, expect_split in ((96, 16, False), (600, 32, True)):
            img = _image(rng, size, size)
            blurred = port.blur(img)
            t = _template(rng, img, m, m)
            s0 = c.split_stats()
            a = c.brute_force_match(t, c.image(blurred))
            assert_same_result(a, port.brute(t, blurred), keys=RESULT_KEYS[:-1])
            assert (c.split_stats()["screened"] > s0["screened"]) == expect_split
