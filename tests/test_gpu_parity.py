"""GPU parity: the sm_100a path through the C ABI vs the oracle, bit for bit.

Integer (8-bit) inputs take the exact-integer kernels; non-integer inputs (OptA's blurred
image) take the FP64 replica kernels.  Both must reproduce the reference's results exactly:
locations, rho bits, skip counts, visit maps, EGS traces, OptA kappa/traces.  (The
north-star tolerance is rho within 1e-5; we assert equality.)
"""
import numpy as np
import pytest

from conftest import RESULT_KEYS, assert_same_result, golden, golden_names, res_vec

pytestmark = pytest.mark.gpu


def _ws_equal(a, b):
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("name", golden_names())
def test_golden_fixtures(ctx, name):
    g = golden(name)
    img, t = g["image"], g["template"]
    m, n = t.shape
    gi = ctx.image(img)
    mu, om, fl = ctx.window_stats(gi, m, n)
    np.testing.assert_array_equal(fl, g["ws_flat"])
    if "ws_mu" in g:
        np.testing.assert_array_equal(mu, g["ws_mu"])
        np.testing.assert_array_equal(om, g["ws_omega"])
    b, surf = ctx.brute_force_match(t, gi, record_surface=True)
    np.testing.assert_array_equal(res_vec(b)[:-1], g["brute"][:-1])
    if "surface" in g:
        np.testing.assert_array_equal(surf, g["surface"])
    e = ctx.efficient_group_size(gi, m, n)
    assert [e["h"], e["w"]] == list(g["egs_h"])
    np.testing.assert_array_equal(
        np.array([[x["h"], x["w"], x["central"], x["retained"], x["total"]] for x in e["trace"]]),
        g["egs_trace"])
    if "egs_map" in g:
        np.testing.assert_array_equal(e["map"], g["egs_map"])
    init = 0.8 if name == "acceptance256" else None
    for mode in ("egs", "opta"):
        for pol, par in (("seq", False), ("frozen", True)):
            r, vis = ctx.match(t, img, mode=mode, parallel=par, threads=4, record_visits=True,
                               init_threshold=init)
            np.testing.assert_array_equal(res_vec(r), g[f"{mode}_{pol}"], err_msg=f"{mode} {pol}")
            np.testing.assert_array_equal(vis, g[f"{mode}_{pol}_visits"])
    prep = ctx.prepare(gi, m, n, mode="opta")
    assert prep.info["kappa"] == int(g["opta_kappa"][0])
    np.testing.assert_array_equal(
        np.array([[x["h"], x["w"], x["cost"], x["restored"]] for x in prep.info["opta_trace"]]),
        g["opta_trace"])
    if "opta_image" in g:
        np.testing.assert_array_equal(prep.search_image(), g["opta_image"])
        np.testing.assert_array_equal(prep.map(), g["opta_map"])
        np.testing.assert_array_equal(ctx.blur(gi), g["blur"])
        np.testing.assert_array_equal(ctx.blur_fidelity_map(gi, g["blur"], m, n), g["fidelity"])


def test_config1_all_modes(ctx, port):
    from paper_1407_3535_b200 import workloads as W
    g = golden("config1")
    w = W.config1()
    t = w.templates[0].pixels.astype(np.float64)
    for mode in ("brute", "egs", "opta"):
        for pol, par in (("seq", False), ("frozen", True)):
            r = ctx.match(t, w.image.astype(np.float64), mode=mode, parallel=par, threads=4)
            np.testing.assert_array_equal(res_vec(r), g[f"{mode}_{pol}"], err_msg=f"{mode} {pol}")


def _cases():
    rng = np.random.default_rng(7)
    out = []
    shapes = [(40, 40, 5, 5), (37, 53, 7, 4), (64, 48, 16, 16), (30, 90, 3, 11), (70, 70, 33, 31),
              (25, 25, 25, 25), (20, 64, 1, 1), (128, 96, 17, 64)]
    for k, (p, q, m, n) in enumerate(shapes):
        base = np.cumsum(np.cumsum(rng.normal(size=(p, q)), 0), 1)
        img = np.clip(np.rint((base - base.min()) / (np.ptp(base) + 1e-9) * 255), 0, 255)
        if k % 3 == 1:
            img = rng.integers(0, 256, size=(p, q)).astype(np.float64)
        if k == 2:
            img[10:40, 5:30] = 77.0  # flat region: flat windows, degenerate centres
        r0, c0 = rng.integers(0, p - m + 1), rng.integers(0, q - n + 1)
        t = np.clip(np.rint(img[r0:r0 + m, c0:c0 + n] * 1.1 - 5 + rng.normal(0, 3, (m, n))),
                    0, 255)
        out.append((img, t))
    return out


@pytest.mark.parametrize("idx", range(8))
def test_match_vs_oracle_edge_shapes(ctx, port, idx):
    img, t = _cases()[idx]
    for mode in ("brute", "egs", "opta"):
        for par in (False, True):
            if np.ptp(t) == 0 and mode != "brute":
                continue
            a, va = ctx.match(t, img, mode=mode, parallel=par, threads=3, record_visits=True)
            b, vb = port.match(t, img, mode=mode, parallel=par, threads=3, visits=True)
            np.testing.assert_array_equal(res_vec(a), res_vec(b), err_msg=f"{mode} par={par}")
            if mode != "brute":
                np.testing.assert_array_equal(va, vb)


@pytest.mark.parametrize("h", [1, 3, 5, 7, 9, 11])
def test_autocorrelation_and_retained(ctx, port, h):
    img, t = _cases()[0]
    m, n = t.shape
    np.testing.assert_array_equal(ctx.local_autocorrelation(img, m, n, h, h),
                                  port.local_autocorrelation(img, m, n, h, h))
    amap = port.local_autocorrelation(img, m, n, h, h)
    assert ctx.autocorr_retained(img, m, n, h, h, 0.8) == port.retained_count(amap, h, h, 0.8)


def test_nonsquare_groups_and_transitive_search(ctx, port):
    img, t = _cases()[3]
    m, n = t.shape
    for h, w in ((3, 5), (5, 1), (7, 3)):
        amap = port.local_autocorrelation(img, m, n, h, w)
        np.testing.assert_array_equal(ctx.local_autocorrelation(img, m, n, h, w), amap)
        for par in (False, True):
            a, va = ctx.transitive_search(t, img, amap, h, w, parallel=par, threads=2,
                                          record_visits=True)
            b, vb = port.transitive_search(t, img, amap, h, w, parallel=par, threads=2,
                                           visits=True)
            np.testing.assert_array_equal(res_vec(a)[:-1], res_vec(b)[:-1])
            np.testing.assert_array_equal(va, vb)


def test_center_scan_and_refine(ctx, port):
    img, t = _cases()[4]
    m, n = t.shape
    cs = ctx.center_scan(t, img, 5, 5)
    b, surface = port.brute(t, img, surface=True)  # zncc_at at every location
    _, _, fl = port.window_stats(img, m, n)
    er, ec = img.shape[0] - m + 1, img.shape[1] - n + 1
    want_rho, want_deg, best = [], [], None
    for ti in range((er + 4) // 5):
        r0, r1 = ti * 5, min(ti * 5 + 5, er) - 1
        for tj in range((ec + 4) // 5):
            c0, c1 = tj * 5, min(tj * 5 + 5, ec) - 1
            cr, cc = (r0 + r1) // 2, (c0 + c1) // 2  # autocorr.cpp:26-30
            want_rho.append(surface[cr, cc])
            want_deg.append(fl[cr, cc])
            key = (not fl[cr, cc], surface[cr, cc], -cr, -cc)  # better_candidate order
            if best is None or key > best[0]:
                best = (key, (cr, cc, surface[cr, cc], bool(fl[cr, cc])))
    np.testing.assert_array_equal(cs["rho"], np.array(want_rho))
    np.testing.assert_array_equal(cs["degenerate"], np.array(want_deg, np.uint8))
    assert cs["best"] == best[1]
    r, c, rho, deg = ctx.refine_localization(t, img, b.best_row, b.best_col, 3)
    assert (r, c, rho) == (b.best_row, b.best_col, b.best_rho)
    assert port.refine(t, img, 5, 7, 4) == ctx.refine_localization(t, img, 5, 7, 4)


def test_nonintegral_image_replica_path(ctx, port):
    img, t = _cases()[0]
    m, n = t.shape
    blurred = port.blur(img)
    gb = ctx.image(blurred)
    assert not gb.is_integer
    _ws_equal(ctx.window_stats(gb, m, n), port.window_stats(blurred, m, n))
    np.testing.assert_array_equal(ctx.running_sum(gb, m, n), port.running_sum(blurred, m, n))
    for h in (3, 5):
        np.testing.assert_array_equal(ctx.local_autocorrelation(gb, m, n, h, h),
                                      port.local_autocorrelation(blurred, m, n, h, h))
    a, sa = ctx.brute_force_match(t, gb, record_surface=True)
    b, sb = port.brute(t, blurred, surface=True)
    np.testing.assert_array_equal(sa, sb)
    assert_same_result(a, b, keys=RESULT_KEYS[:-1])
    # non-integer template on an integer image also takes the FP64 path
    tf = t * 0.5 + 0.25
    a = ctx.brute_force_match(tf, img)
    b = port.brute(tf, img)
    assert_same_result(a, b, keys=RESULT_KEYS[:-1])


def test_seeded_policy_same_argmax_and_sound(ctx, port):
    img, t = _cases()[0]
    b, surface = port.brute(t, img, surface=True)
    for mode in ("egs", "opta"):
        r, vis = ctx.match(t, img, mode=mode, policy="seeded", record_visits=True)
        if mode == "egs":
            assert (r.best_row, r.best_col, r.best_rho) == (b.best_row, b.best_col, b.best_rho)
            # soundness: every eliminated member is <= the final threshold (acceptance c4)
            assert np.all(surface[vis == 1] <= r.final_threshold + 1e-9)
        else:
            assert (r.refined_row, r.refined_col, r.refined_rho) == \
                (b.best_row, b.best_col, b.best_rho)
        assert r.eliminated + r.retained + r.centers == b.ops


def test_batch_run_matches_individual(ctx, port):
    from paper_1407_3535_b200 import workloads as W
    w = W.config1()
    rng = np.random.default_rng(3)
    ts = [W.cut_template(rng, w.image, 32, 32, 1.0, 0.0, 4.0).pixels for _ in range(4)]
    gi = ctx.image(w.image)
    for mode in ("egs", "opta"):
        prep = ctx.prepare(gi, 32, 32, mode=mode)
        batch = ctx.run(prep, np.stack(ts), parallel=True, threads=4)
        for t, r in zip(ts, batch):
            o = port.match(t.astype(float), w.image.astype(float), mode=mode, parallel=True,
                           threads=4)
            np.testing.assert_array_equal(res_vec(r)[:-1], res_vec(o)[:-1])


def test_errors_match_reference_messages(ctx):
    from paper_1407_3535_b200.api import InvalidArgument
    img = np.random.default_rng(1).integers(0, 256, (32, 32)).astype(np.float64)
    with pytest.raises(InvalidArgument, match="constant template"):
        ctx.match(np.full((5, 5), 3.0), img, mode="egs")
    with pytest.raises(InvalidArgument, match="template larger than search image"):
        ctx.match(np.ones((40, 5)), img, mode="egs")
    with pytest.raises(InvalidArgument, match="odd"):
        ctx.local_autocorrelation(img, 5, 5, 4, 3)
    with pytest.raises(InvalidArgument, match="init threshold"):
        ctx.match(img[:5, :5], img, mode="egs", init_threshold=1.5)
    with pytest.raises(InvalidArgument, match="rho_tb"):
        ctx.efficient_group_size(img, 5, 5, rho_tb=1.0)
    r = ctx.match(np.full((5, 5), 3.0), img, mode="brute")  # brute accepts flat templates
    assert r.best_degenerate and r.best_rho == 0.0


def test_below_threshold_flag(ctx, port):
    img, t = _cases()[0]
    for mode in ("egs", "opta"):
        a = ctx.match(t, img, mode=mode, init_threshold=0.9999)
        b = port.match(t, img, mode=mode, init_threshold=0.9999)
        np.testing.assert_array_equal(res_vec(a), res_vec(b))
        assert a.below_threshold


@pytest.mark.gpu
def test_context_closed_before_its_images(port):
    """Closing a context first defers its release to the last image/preparation."""
    from paper_1407_3535_b200 import api
    rng = np.random.default_rng(5)
    img = rng.integers(0, 256, (48, 52)).astype(np.uint8)
    t = img[10:19, 12:21].copy()
    c = api.Context(0)
    im = c.image(img)
    prep = c.prepare(im, 9, 9)
    c.close()
    r = c.__class__(0).match(t, img)  # an independent context still works
    prep2 = prep
    prep2.close()
    im.close()
    b = port.brute(t.astype(np.float64), img.astype(np.float64))
    assert (r.best_row, r.best_col) == (b.best_row, b.best_col)


@pytest.mark.gpu
@pytest.mark.parametrize("m,n", [(9, 7), (16, 16), (33, 20)])
def test_fused_autocorr_equals_colwalk(port, m, n):
    """The fused sliding-window R_co kernel and the column-walk pair agree bit for bit
    (clipped last group row/column included) and match the oracle."""
    import os
    from paper_1407_3535_b200 import api
    rng = np.random.default_rng(m * 100 + n)
    base = np.cumsum(np.cumsum(rng.normal(size=(101, 87)), 0), 1)
    img = np.clip(np.rint((base - base.min()) / np.ptp(base) * 255), 0, 255).astype(np.uint8)
    maps = {}
    for path in ("fused", "colwalk"):
        os.environ["TMATCH_AUTOCORR"] = path
        try:
            c = api.Context(0)
        finally:
            os.environ.pop("TMATCH_AUTOCORR", None)
        im = c.image(img)
        for h in (1, 3, 5, 7, 9, 11):
            maps[(path, h)] = c.local_autocorrelation(im, m, n, h, h)
        im.close()
        c.close()
    for h in (1, 3, 5, 7, 9, 11):
        want = port.local_autocorrelation(img.astype(np.float64), m, n, h, h)
        assert np.array_equal(maps[("fused", h)], maps[("colwalk", h)]), h
        assert np.array_equal(maps[("fused", h)], want), h


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,cols", [(64, 64, 2000), (20, 63, 1997), (17, 65, 1531),
                                      (9, 7, 2100), (40, 10, 801)])
def test_fused_autocorr_wide(ctx, port, m, n, cols):
    """The group-column R_co kernel (h = 3, 5) over several column tiles: every remainder
    n mod h (head columns), clipped and unclipped last group columns (tail columns), clipped
    last group rows, flat patches — equal to the oracle bit for bit."""
    rng = np.random.default_rng(m * 7 + n + cols)
    base = np.cumsum(np.cumsum(rng.normal(size=(m + 40, cols)), 0), 1)
    img = np.clip(np.rint((base - base.min()) / np.ptp(base) * 255), 0, 255).astype(np.uint8)
    img[5:30, 100:180] = 91  # flat windows (degenerate statistics)
    gi = ctx.image(img)
    for h in (3, 5):
        got = ctx.local_autocorrelation(gi, m, n, h, h)
        want = port.local_autocorrelation(img.astype(np.float64), m, n, h, h)
        assert np.array_equal(got, want), (h, np.argwhere(got != want)[:5])
        assert ctx.autocorr_retained(gi, m, n, h, h) == port.retained_count(want, h, h), h


@pytest.mark.gpu
@pytest.mark.parametrize("m,n", [(1, 1), (5, 7), (33, 64), (64, 200), (130, 3)])
def test_window_stats_fused_tiles(ctx, port, m, n):
    """Fused window statistics over several column tiles and row segments, with flat
    patches (variance exactly zero and near the noise floor), equal to the oracle."""
    rng = np.random.default_rng(m * 1000 + n)
    img = rng.integers(0, 256, (300, 700)).astype(np.uint8)
    img[40:200, 100:400] = 77  # flat region
    img[210:260, 500:690] = rng.integers(100, 102, (50, 190))  # tiny variance
    gi = ctx.image(img)
    _ws_equal(ctx.window_stats(gi, m, n), port.window_stats(img.astype(np.float64), m, n))


def _ctx_with(env, value):
    import os
    from paper_1407_3535_b200 import api
    old = os.environ.get(env)
    os.environ[env] = value
    try:
        return api.Context(0)
    finally:
        if old is None:
            os.environ.pop(env, None)
        else:
            os.environ[env] = old


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,h", [(16, 16, 3), (40, 64, 5), (33, 70, 7), (96, 96, 3),
                                   (130, 120, 3), (20, 24, 11)])
def test_tc_centre_scan_equals_cuda_core(m, n, h):
    """The tcgen05 kind::i8 centre scan (2 column tiles, several bands, B chunking for the
    130x120 template, clipped last group row/column) equals the CUDA-core FP32-exact scan
    bit for bit: centre rho, degenerate flags and the best centre."""
    rng = np.random.default_rng(m * 7 + n * 3 + h)
    base = np.cumsum(np.cumsum(rng.normal(size=(m + 61, n + 2200)), 0), 1)
    img = np.clip(np.rint((base - base.min()) / np.ptp(base) * 255), 0, 255).astype(np.uint8)
    img[5:25, 100:300] = 40  # flat windows
    t = np.clip(np.rint(img[11:11 + m, 1500:1500 + n] * 0.9 + 7 + rng.normal(0, 3, (m, n))),
                0, 255)
    tc, cc = _ctx_with("TMATCH_TC", "1"), _ctx_with("TMATCH_TC", "0")
    a = tc.center_scan(t, img, h, h)
    b = cc.center_scan(t, img, h, h)
    np.testing.assert_array_equal(a["rho"], b["rho"])
    np.testing.assert_array_equal(a["degenerate"], b["degenerate"])
    assert a["best"] == b["best"]
    tc.close()
    cc.close()


@pytest.mark.gpu
@pytest.mark.parametrize("m,n", [(16, 16), (40, 64), (96, 96), (130, 120)])
def test_tc_brute_surface_equals_cuda_core(m, n):
    """Tensor-core brute force (dense mode 0): the whole rho surface and the argmax equal
    the CUDA-core FP32-exact kernel bit for bit (2 column tiles, B chunking)."""
    rng = np.random.default_rng(m + 5 * n)
    base = np.cumsum(np.cumsum(rng.normal(size=(m + 40, n + 2100)), 0), 1)
    img = np.clip(np.rint((base - base.min()) / np.ptp(base) * 255), 0, 255).astype(np.uint8)
    img[3:30, 50:400] = 9
    t = np.clip(np.rint(img[17:17 + m, 1900:1900 + n] * 1.1 - 4 + rng.normal(0, 2, (m, n))),
                0, 255)
    tc, cc = _ctx_with("TMATCH_TC", "1"), _ctx_with("TMATCH_TC", "0")
    a, sa = tc.brute_force_match(t, img, record_surface=True)
    b, sb = cc.brute_force_match(t, img, record_surface=True)
    np.testing.assert_array_equal(sa, sb)
    assert (a.best_row, a.best_col, a.best_rho) == (b.best_row, b.best_col, b.best_rho)
    tc.close()
    cc.close()


@pytest.mark.gpu
def test_tc_dense_survivors_weak_template(port):
    """A noise template (no elimination) takes the dense survivor path: tensor-core and
    CUDA-core runs give identical results, equal to the brute-force argmax."""
    rng = np.random.default_rng(77)
    base = np.cumsum(np.cumsum(rng.normal(size=(300, 2200)), 0), 1)
    img = np.clip(np.rint((base - base.min()) / np.ptp(base) * 255), 0, 255).astype(np.uint8)
    t = rng.integers(0, 256, (24, 24)).astype(np.float64)
    res = []
    for flag in ("1", "0"):
        c = _ctx_with("TMATCH_TC", flag)
        prep = c.prepare(c.image(img), 24, 24)
        for pol in ("seeded", "frozen", "sequential"):
            r = c.run(prep, t, policy=pol, parallel=(pol == "frozen"), threads=2)
            res.append((pol, r.best_row, r.best_col, r.best_rho, r.eliminated, r.retained))
        prep.close()
        c.close()
    assert res[:3] == res[3:]
    b = port.brute(t, img.astype(np.float64))
    assert (res[0][1], res[0][2], res[0][3]) == (b.best_row, b.best_col, b.best_rho)


@pytest.mark.gpu
@pytest.mark.parametrize("policy", ["seeded", "frozen", "sequential", "reference"])
@pytest.mark.parametrize("mode", ["egs", "opta"])
def test_search_equals_prepare_run(ctx, policy, mode):
    """tm_search / tm_search_u8 (prepare + run in one call, template uploaded while the
    preparation runs) give exactly the prepare + run results."""
    rng = np.random.default_rng(3)
    base = np.cumsum(np.cumsum(rng.normal(size=(140, 170)), 0), 1)
    img = np.clip(np.rint((base - base.min()) / np.ptp(base) * 255), 0, 255).astype(np.uint8)
    t = np.clip(np.rint(img[50:70, 90:112] * 0.9 + 8 + rng.normal(0, 3, (20, 22))), 0, 255)
    gi = ctx.image(img)
    prep = ctx.prepare(gi, 20, 22, mode=mode)
    want = ctx.run(prep, t, policy=policy, parallel=True, threads=4)
    prep.close()
    for tt in (t, t.astype(np.uint8)):
        got = ctx.search(gi, tt, mode=mode, policy=policy, parallel=True, threads=4)
        for k in ("best_row", "best_col", "best_rho", "refined_row", "refined_col",
                  "refined_rho", "eliminated", "retained", "centers", "ops",
                  "final_threshold"):
            assert getattr(got, k) == getattr(want, k), k


def test_search_speculation_hit_and_miss(ctx):
    """tm_search enqueues the centre scan for the predicted group size (the last h_e seen for
    this shape) behind the EGS batch, gated on the device decision.  Alternating images of
    one shape whose h_e differ exercises hits and misses; every result must equal the
    prepare + run result, and the EGS sizes must differ (so misses really happen)."""
    rng = np.random.default_rng(11)
    rough = rng.integers(0, 256, (160, 190)).astype(np.uint8)  # white noise: small h_e
    base = np.cumsum(np.cumsum(rng.normal(size=(160, 190)), 0), 1)  # smooth: larger h_e
    smooth = np.clip(np.rint((base - base.min()) / np.ptp(base) * 255), 0, 255).astype(np.uint8)
    keys = ("best_row", "best_col", "best_rho", "eliminated", "retained", "centers", "ops",
            "final_threshold")
    seen = set()
    for img in (rough, smooth, smooth, rough, rough, smooth):
        t = np.clip(np.rint(img[60:84, 70:96] * 1.05 - 4 + rng.normal(0, 3, (24, 26))), 0, 255)
        gi = ctx.image(img)
        prep = ctx.prepare(gi, 24, 26, mode="egs")
        seen.add(prep.info["h"])
        want = ctx.run(prep, t, policy="seeded")
        prep.close()
        got = ctx.search(gi, t.astype(np.uint8), mode="egs", policy="seeded")
        for k in keys:
            assert getattr(got, k) == getattr(want, k), k
        gi.close()
    assert len(seen) >= 2, seen


@pytest.mark.parametrize("policy", ["seeded", "frozen"])
@pytest.mark.parametrize("case", ["cut", "noise"])
def test_search_fused_scan2_equals_prepare_run(ctx, policy, case):
    """tm_search runs scan 2 inside the R_co launch of the predicted group size (no map):
    on smooth (h_e = 5, packed walk), rough (h_e = 3) and wide multi-tile images, with a cut
    template (few survivors, list path) and a pure-noise template (weak elimination, dense
    tensor-core survivor pass driven by the visit codes), repeated (the second call
    predicts from the first), every result equals prepare + run bit for bit."""
    rng = np.random.default_rng(23)
    keys = ("best_row", "best_col", "best_rho", "best_degenerate", "eliminated", "retained",
            "centers", "ops", "final_threshold", "elim_pct")
    seen = set()
    for rows, cols, m, n, smooth in [(300, 420, 32, 32, True), (260, 333, 24, 40, False),
                                     (200, 1500, 48, 64, True), (257, 260, 31, 17, True)]:
        if smooth:
            base = np.cumsum(np.cumsum(rng.normal(size=(rows, cols)), 0), 1)
            img = np.clip(np.rint((base - base.min()) / np.ptp(base) * 255), 0,
                          255).astype(np.uint8)
            img[20:60, 30:90] = 77  # flat windows
        else:
            img = rng.integers(0, 256, (rows, cols)).astype(np.uint8)
        if case == "cut":
            t = np.clip(np.rint(img[rows // 3:rows // 3 + m, cols // 2:cols // 2 + n] * 0.95 + 6
                                + rng.normal(0, 4, (m, n))), 0, 255).astype(np.uint8)
        else:
            t = rng.integers(0, 256, (m, n)).astype(np.uint8)
        gi = ctx.image(img)
        prep = ctx.prepare(gi, m, n, mode="egs")
        seen.add(prep.info["h"])
        want = ctx.run(prep, t, policy=policy, parallel=(policy == "frozen"), threads=2)
        prep.close()
        for _ in range(2):
            gi.reset_cache()
            got = ctx.search(gi, t, mode="egs", policy=policy, parallel=(policy == "frozen"),
                             threads=2)
            for k in keys:
                assert getattr(got, k) == getattr(want, k), (rows, cols, k)
        gi.close()
    assert {3, 5} <= seen, seen


@pytest.mark.parametrize("shape", [(300, 420, 40, 37), (700, 260, 64, 64), (130, 90, 20, 30)])
def test_search_upload_streamed_equals_resident(ctx, port, shape):
    """tm_search_upload_u8 (upload + search in one call) == tm_image_upload_u8 +
    tm_search_u8, bit for bit, repeated on the same image; the image holds near-constant
    windows, and the window statistics equal the oracle's."""
    rows, cols, m, n = shape
    rng = np.random.default_rng(rows + cols)
    base = np.cumsum(np.cumsum(rng.normal(size=(rows, cols)), 0), 1)
    img = np.clip(np.rint((base - base.min()) / np.ptp(base) * 255), 0, 255).astype(np.uint8)
    img[5:5 + 2 * m, 3:3 + 2 * n] = 200
    img[5 + m, 3 + n] = 201  # variance 1 pixel away from flat: decided by the noise floor
    t = np.clip(np.rint(img[rows // 3:rows // 3 + m, cols // 4:cols // 4 + n] * 1.05 + 3
                        + rng.normal(0, 3, (m, n))), 0, 255).astype(np.uint8)
    keys = ("best_row", "best_col", "best_rho", "eliminated", "retained", "centers", "ops",
            "final_threshold")
    a = ctx.image(np.zeros_like(img))
    a.upload_u8(img)
    want = ctx.search(a, t, policy="seeded")
    b = ctx.image(np.zeros_like(img))
    for _ in range(2):
        got = ctx.search_upload(b, img, t, policy="seeded")
        for k in keys:
            assert getattr(got, k) == getattr(want, k), k
    _ws_equal(ctx.window_stats(b, m, n), port.window_stats(img.astype(np.float64), m, n))


def test_search_stream_equals_single_calls(ctx):
    """tm_search_stream_u8 over a stream of different images (two device slots, the next
    copy overlapped with the current search) == tm_search_upload_u8 per image, bit for bit;
    then a stream with a different shape (slots re-created) and an empty stream."""
    keys = ("best_row", "best_col", "best_rho", "eliminated", "retained", "centers", "ops",
            "final_threshold")
    rng = np.random.default_rng(11)
    for rows, cols, m, n in [(300, 420, 40, 37), (257, 190, 21, 16)]:
        imgs = []
        for k in range(5):
            base = np.cumsum(np.cumsum(rng.normal(size=(rows, cols)), 0), 1)
            imgs.append(np.clip(np.rint((base - base.min()) / np.ptp(base) * 255), 0,
                                255).astype(np.uint8))
        src = imgs[2]
        t = np.clip(np.rint(src[rows // 3:rows // 3 + m, cols // 4:cols // 4 + n] * 1.05 + 3
                            + rng.normal(0, 3, (m, n))), 0, 255).astype(np.uint8)
        for policy in ("seeded", "frozen", "sequential"):
            got = ctx.search_stream(imgs, t, policy=policy)
            assert len(got) == len(imgs)
            b = ctx.image(np.zeros((rows, cols), np.uint8))
            for g, a in zip(got, imgs):
                want = ctx.search_upload(b, a, t, policy=policy)
                for k in keys:
                    assert getattr(g, k) == getattr(want, k), (policy, k)
            b.close()
    assert ctx.search_stream([], t) == []


@pytest.mark.parametrize("policy", ["seeded", "frozen"])
def test_search_stream_mixed_group_sizes(ctx, policy):
    """A stream whose images alternate between white noise (small h_e) and smooth fields
    (larger h_e): the next image's scan 1 + seeding, enqueued behind the current search on
    the predicted grid, is mispredicted every other image and must fall back to the
    standard path -- every result equals the single-call result."""
    rng = np.random.default_rng(29)
    rows, cols, m, n = 170, 230, 24, 26
    rough = [rng.integers(0, 256, (rows, cols)).astype(np.uint8) for _ in range(3)]
    smooth = []
    for _ in range(3):
        base = np.cumsum(np.cumsum(rng.normal(size=(rows, cols)), 0), 1)
        smooth.append(np.clip(np.rint((base - base.min()) / np.ptp(base) * 255), 0,
                              255).astype(np.uint8))
    imgs = [rough[0], smooth[0], smooth[1], rough[1], smooth[2], rough[2]]
    t = np.clip(np.rint(smooth[1][60:84, 70:96] * 1.05 - 4 + rng.normal(0, 3, (m, n))), 0,
                255).astype(np.uint8)
    keys = ("best_row", "best_col", "best_rho", "eliminated", "retained", "centers", "ops",
            "final_threshold")
    got = ctx.search_stream(imgs, t, policy=policy, parallel=(policy == "frozen"), threads=2)
    b = ctx.image(np.zeros((rows, cols), np.uint8))
    hs = set()
    for g, a in zip(got, imgs):
        want = ctx.search_upload(b, a, t, policy=policy, parallel=(policy == "frozen"),
                                 threads=2)
        for k in keys:
            assert getattr(g, k) == getattr(want, k), (policy, k)
        gi = ctx.image(a)
        prep = ctx.prepare(gi, m, n, mode="egs")
        hs.add(prep.info["h"])
        prep.close()
        gi.close()
    b.close()
    assert len(hs) >= 2, hs  # the group size really changes along the stream


@pytest.mark.parametrize("dense", [False, True])
def test_search_upload_undecided_windows(ctx, port, dense):
    """A 3400 x 3300 image whose noise floor ((rows + cols) * eps * sum of squares, about
    0.36 here) sits just below the variance sum of windows with exactly one bumped pixel in
    a constant region ((mn-1)/mn): window statistics equal the oracle's (flat decisions
    included) and the one-call search equals upload + search."""
    rng = np.random.default_rng(17 + dense)
    rows, cols, m, n = 3400, 3300, 16, 16
    img = rng.integers(0, 256, (rows, cols)).astype(np.uint8)
    img[200:1400, 300:1500] = 90
    step = 17 if dense else 97
    img[200:1400:step, 300:1500:step] = 91
    t = img[2000:2016, 2500:2516].copy()
    b = ctx.image(np.zeros_like(img))
    got = ctx.search_upload(b, img, t, policy="seeded")
    _ws_equal(ctx.window_stats(b, m, n), port.window_stats(img.astype(np.float64), m, n))
    a = ctx.image(np.zeros_like(img))
    a.upload_u8(img)
    want = ctx.search(a, t, policy="seeded")
    for k in ("best_row", "best_col", "best_rho", "eliminated", "retained", "final_threshold"):
        assert getattr(got, k) == getattr(want, k), k


@pytest.mark.parametrize("m,n", [(1, 1), (2, 2), (3, 4), (4, 3), (5, 5), (2, 9), (7, 15), (1, 30)])
def test_group_column_autocorr_small_windows(ctx, port, m, n):
    """The group-column R_co kernel at window widths below, at and just above the group
    width (n < h: head columns only, no whole blocks; n % h == 0: no head), one-row extents
    and every clipped last group column, h = 3 and 5, equal to the oracle with counts."""
    rng = np.random.default_rng(m * 31 + n)
    for rows, cols in ((m + 2, 263), (m, 131), (m + 11, 517)):
        img = rng.integers(0, 256, (rows, cols)).astype(np.uint8)
        img[:, 40:70] = 128  # flat columns: degenerate members
        gi = ctx.image(img)
        for h in (3, 5):
            want = port.local_autocorrelation(img.astype(np.float64), m, n, h, h)
            got = ctx.local_autocorrelation(gi, m, n, h, h)
            assert np.array_equal(got, want), (rows, cols, h, np.argwhere(got != want)[:3])
            assert ctx.autocorr_retained(gi, m, n, h, h) == port.retained_count(want, h, h)
        gi.close()


@pytest.mark.gpu
@pytest.mark.parametrize("replay", ["0", "1"])
def test_nonintegral_noise_floor_replay(ctx, port, replay, monkeypatch):
    """Non-integer images (OptA's blurred image): the image-global q_total (stats.cpp:79) is
    the reference's SEQUENTIAL sum only where it matters -- windows whose variance falls in
    the error bracket of the parallel sum trigger the sequential replay on the device and a
    redo pass.  replay=1 widens the bracket so every window takes that path.  Either way the
    flat map, mu and omega equal the oracle's bit for bit, on an image whose blurred
    constant regions put window variances at the noise floor."""
    monkeypatch.setenv("TMATCH_PN_REPLAY", replay)
    rng = np.random.default_rng(91)
    img = rng.integers(0, 256, size=(120, 140)).astype(np.float64)
    img[10:70, 20:90] = 137.0   # constant patches: blurred, their windows sit at the floor
    img[80:115, 60:130] = 3.0
    img = port.blur(port.blur(img))  # non-integer, the reference blur twice
    for m, n in ((9, 11), (17, 17)):
        gi = ctx.image(img)
        assert not gi.is_integer
        mu, om, fl = ctx.window_stats(gi, m, n)
        pm, po, pf = port.window_stats(img, m, n)
        assert fl.sum() > 0  # flat windows present
        np.testing.assert_array_equal(fl, pf)
        np.testing.assert_array_equal(mu, pm)
        np.testing.assert_array_equal(om, po)
        gi.close()


@pytest.mark.gpu
def test_large_template_bright_image_u32_guard(ctx, port):
    """Templates with m*n*255^2 >= 2^32 (here 258x260 = 67,080 pixels) on a near-saturated
    image: the 8-bit R_co kernels' u32 cross sums would wrap, so these shapes must take the
    64-bit path -- R_co, EGS and the search equal the oracle."""
    rng = np.random.default_rng(5)
    img = rng.integers(235, 256, size=(280, 290)).astype(np.float64)
    t = np.clip(np.rint(img[10:268, 20:280] * 0.98 + rng.normal(0, 1, (258, 260))), 0, 255)
    m, n = t.shape
    for h in (1, 3):
        np.testing.assert_array_equal(ctx.local_autocorrelation(img, m, n, h, h),
                                      port.local_autocorrelation(img, m, n, h, h))
    got = ctx.match(t, img, mode="egs")
    want = port.match(t, img, mode="egs")
    assert_same_result(got, want, keys=RESULT_KEYS[:-1])


@pytest.mark.gpu
def test_transitive_search_with_prepared_statistics(ctx, port):
    """run_egs on a preparation of EARLIER pixels (the reference correlates the current
    pixels with the prepared map and window statistics, matcher.cpp:235-246):
    tm_transitive_search_ws equals the oracle's transitive_search with the same explicit
    statistics, bit for bit."""
    img, t = _cases()[0]
    m, n = t.shape
    ws_old = port.window_stats(img, m, n)
    e = port.efficient_group_size(img, m, n, ws=ws_old)
    edited = img.copy()
    edited[5:5 + m, 7:7 + n] = t  # the pixels change after the preparation
    for par in (False, True):
        want = port.transitive_search(t, edited, e["map"], e["h"], e["w"], ws=ws_old,
                                      parallel=par, threads=2)
        got = ctx.transitive_search(t, edited, e["map"], e["h"], e["w"], ws=ws_old,
                                    parallel=par, threads=2)
        assert_same_result(got, want, keys=RESULT_KEYS[:-1])
