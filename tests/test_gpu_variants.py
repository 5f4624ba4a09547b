"""The A/B kernel variants behind the environment switches give
the oracle's bits too.  The switches are read once per process, so every variant runs in
a subprocess: window statistics, R_co maps and retained counts for h = 3, 5, 7 on four
image shapes (multi-tile; clipped and unclipped group columns; n % h = 0 and != 0, i.e.
every packed-walk part layout), compared with the oracle."""
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
], ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()) or "default")
def test_kernel_variant_parity(env):
    full = dict(os.environ)
    full.update(env)
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], env=full, cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
