"""The A/B kernel variants behind the environment switches give
the oracle's bits too.  The switches are read once per process, so every variant runs in
a subprocess: window statistics, R_co maps and retained counts for h = 3, 5, 7 on four
image shapes (multi-tile; clipped and unclipped group columns; n % h = 0 and != 0, i.e.
every packed-walk part layout), compared with the oracle; and one full frozen-policy
search per shape (the fused R_co + scan-2 path of tm_search) against the oracle's
`--parallel` match: location, rho bits, eliminated / retained / ops."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
from paper_1407_3535_b200 import api
from oracle.binding import Oracle
port = Oracle("port")
ctx = api.Context(0)
rng = np.random.default_rng(5)
for (rows, cols, m, n) in ((150, 1300, 40, 64), (120, 700, 33, 10), (140, 1063, 36, 64),
                          (90, 619, 20, 20)):
    base = np.cumsum(np.cumsum(rng.normal(size=(rows, cols)), 0), 1)
    img = np.clip(np.rint((base - base.min()) / np.ptp(base) * 255), 0, 255).astype(np.uint8)
    img[10:40, 50:120] = 60
    gi = ctx.image(img)
    for a, b in zip(ctx.window_stats(gi, m, n), port.window_stats(img.astype(np.float64), m, n)):
        assert np.array_equal(a, b), "window_stats"
    for h in (3, 5, 7):
        want = port.local_autocorrelation(img.astype(np.float64), m, n, h, h)
        got = ctx.local_autocorrelation(gi, m, n, h, h)
        assert np.array_equal(got, want), ("map", h)
        assert ctx.autocorr_retained(gi, m, n, h, h) == port.retained_count(want, h, h), ("n_r", h)
    r0, c0 = rows // 3, cols // 2
    t = img[r0:r0 + m, c0:c0 + n].astype(np.float64)
    t = np.clip(np.rint(t * 0.9 + 7 + rng.normal(0, 3, t.shape)), 0, 255)
    got = ctx.search(gi, t, mode="egs", policy="frozen", parallel=True, threads=2)
    want = port.match(t, img.astype(np.float64), mode="egs", parallel=True)
    for f in ("best_row", "best_col", "best_rho", "eliminated", "retained", "ops"):
        assert getattr(got, f) == getattr(want, f), ("search", f, getattr(got, f), getattr(want, f))
    gi.close()
ctx.close()
print("ok")
"""


@pytest.mark.parametrize("env", [
    {},
    {"TMATCH_ACF": "column"},
    {"TMATCH_ACG_THREADS": "128"},
    {"TMATCH_ACG_THREADS": "256"},
    {"TMATCH_ACG_PACK": "0"},
    {"TMATCH_ACG_PACK": "1"},
    {"TMATCH_ACG_PACK": "1", "TMATCH_ACG_THREADS": "256"},
    {"TMATCH_ACG_PACK": "1", "TMATCH_ACG_THREADS": "128"},
    {"TMATCH_AUTOCORR": "colwalk"},
    {"TMATCH_WSTATS": "column"},
    {"TMATCH_WSTATS4": "256x4"},
    {"TMATCH_WSTATS4": "128x4"},
    {"TMATCH_WSTATS4": "128x2"},
    {"TMATCH_RCO3": "0"},
    {"TMATCH_RCO3": "0", "TMATCH_ACG_PACK": "1"},
    {"TMATCH_RCO3_FUSED": "1"},
    {"TMATCH_RCO3_FUSED": "1", "TMATCH_RCO3_NT": "256"},
    {"TMATCH_RCO3_NT": "128"},
    {"TMATCH_EPI_V": "2"},
    {"TMATCH_EPI_V": "4"},
    {"TMATCH_EPI_V": "9"},
    {"TMATCH_EPI_MINB": "2"},
    {"TMATCH_EGS_ORDER": "0"},
    {"TMATCH_RCO5_MIN": "0"},
    {"TMATCH_RCO5": "0"},
], ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()) or "default")
def test_kernel_variant_parity(env):
    full = dict(os.environ)
    full.update(env)
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], env=full, cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
