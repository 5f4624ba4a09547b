"""TMACMAP1 map-cache interoperability with the reference (CPU, host functions only).

The B200 library's content_hash / autocorr_cache_key / save_autocorr / load_autocorr
(libtmatch.so, tests/cpp/cache_interop.cpp) against the reference's own image.cpp:215-228
and autocorr.cpp:102-153 (oracle/_ref, compiled from the reference sources): equal keys on
integer and non-integer images, and a map saved by either library loads in the other.
"""
import os
import subprocess

import numpy as np
import pytest

from paper_1407_3535_b200 import native as N

TOOL = os.path.join(os.path.dirname(N.API_LIB_PATH), "cache_interop")


def run(*args):
    r = subprocess.run([TOOL, *map(str, args)], capture_output=True, text=True, check=True)
    return r.stdout.split()


def keys(tmp_path, img, m, n, h, w):
    f = tmp_path / "img.f64"
    np.ascontiguousarray(img, np.float64).tofile(f)
    ch, key = run("key", f, img.shape[0], img.shape[1], m, n, h, w)
    return int(ch), int(key)


@pytest.mark.parametrize("kind", ["u8", "fractional"])
def test_content_hash_and_cache_key_equal_reference(tmp_path, ref, kind):
    rng = np.random.default_rng(11)
    img = rng.integers(0, 256, size=(37, 53)).astype(np.float64)
    if kind == "fractional":
        img = img + rng.random(img.shape) * 0.5  # OptA-blurred images are non-integer
    ch, key = keys(tmp_path, img, 7, 9, 3, 5)
    assert ch == ref.content_hash(img)
    assert key == ref.autocorr_cache_key(img, 7, 9, 3, 5)


def test_hash_separates_images_that_round_to_the_same_bytes(tmp_path, ref):
    rng = np.random.default_rng(12)
    a = rng.integers(0, 256, size=(20, 30)).astype(np.float64)
    b = a.copy()
    b[3, 4] += 0.25  # rounds to the same u8 pixel
    assert keys(tmp_path, a, 5, 5, 3, 3)[0] != keys(tmp_path, b, 5, 5, 3, 3)[0]
    # same dims, transposed layout: dims are part of the key
    assert keys(tmp_path, a.reshape(30, 20), 5, 5, 3, 3)[0] != keys(tmp_path, a, 5, 5, 3, 3)[0]


def test_map_files_round_trip_between_libraries(tmp_path, ref):
    rng = np.random.default_rng(13)
    img = rng.integers(0, 256, size=(40, 44)).astype(np.float64)
    er, ec, h, w = 40 - 8 + 1, 44 - 8 + 1, 5, 5
    amap = rng.uniform(-1, 1, size=(er, ec))
    key = ref.autocorr_cache_key(img, 8, 8, h, w)
    # reference writes, B200 library reads
    ref.save_autocorr(amap, h, w, key, str(tmp_path / "ref.tmac"))
    out = tmp_path / "ours.f64"
    assert run("load", tmp_path / "ref.tmac", key, er, ec, h, w, out) == ["hit"]
    assert np.array_equal(np.fromfile(out), amap.ravel())
    assert run("load", tmp_path / "ref.tmac", key + 1, er, ec, h, w, out) == ["miss"]
    # B200 library writes, reference reads
    mf = tmp_path / "map.f64"
    amap.tofile(mf)
    run("save", mf, er, ec, h, w, key, tmp_path / "ours.tmac")
    back = ref.load_autocorr(str(tmp_path / "ours.tmac"), key, er, ec, h, w)
    assert back is not None and np.array_equal(back, amap)
    assert ref.load_autocorr(str(tmp_path / "ours.tmac"), key ^ 1, er, ec, h, w) is None
    # byte-identical files
    assert (tmp_path / "ours.tmac").read_bytes() == (tmp_path / "ref.tmac").read_bytes()
