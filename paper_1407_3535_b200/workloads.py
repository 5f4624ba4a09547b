"""Seeded synthetic workloads for the five BASELINE.json configurations.

The reference ships no generator for these configs (its synth.cpp:19-40 makes smoothed
white noise) and the paper's SI/AI datasets are not available, so these seeded inputs
stand in for them.  The generator is:

1. Gaussian white field (numpy PCG64, explicit seed), FP64.
2. FFT; multiply by |f|^(-beta/2) with DC = 0; optional Gaussian blur applied as the
   transfer function exp(-2 pi^2 sigma^2 |f|^2) in the same spectrum (periodic border).
3. Inverse FFT, real part; min-max rescale to [0, 255], round, clamp -> uint8.

The bytes are host-independent: FP64 pocketfft (compile-time vectorised, thread-count
invariant) and elementwise math restricted to correctly rounded operations (det_exp /
det_log below).  Each config's SHA-256 is pinned in tests/golden/configs.json.

Templates are cut at seeded locations and perturbed photometrically:
round(clip(gain * t + offset + N(0, sigma^2), 0, 255)).  Everything is integer-valued
uint8, the reference's input domain (image.hpp: loaded 8-bit data).

This module is input plumbing for tests and bench.py; it is not on the timed path.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

try:  # multithreaded pocketfft (each 1-D transform is independent: thread-count invariant)
    import scipy.fft as _fft

    def _rfft2(x):
        return _fft.rfft2(x, workers=-1)

    def _irfft2(x, s):
        return _fft.irfft2(x, s=s, workers=-1)
except Exception:  # pragma: no cover
    def _rfft2(x):
        return np.fft.rfft2(x)

    def _irfft2(x, s):
        return np.fft.irfft2(x, s=s)


# ---- bit-deterministic elementwise transcendental functions ---------------------------
# numpy dispatches exp/log/power to CPU-specific SIMD kernels (AVX512_SKX SVML vs AVX2 vs
# scalar libm) whose last-ulp results differ, and a single ulp can move a pixel across a
# rounding boundary of the u8 quantisation: measured here, C1-C3 hashed differently with
# NPY_DISABLE_CPU_FEATURES=AVX512*.  These use only +, -, *, /, frexp, ldexp and rint,
# which IEEE 754 rounds exactly on every CPU, so the inputs are the same bytes on any host.
_LN2 = 0.6931471805599453


def det_log(x: np.ndarray) -> np.ndarray:
    """Natural log of x > 0 (float64): frexp range reduction + atanh series."""
    m, e = np.frexp(np.asarray(x, dtype=np.float64))
    low = m < 0.7071067811865476
    m = np.where(low, m * 2.0, m)
    e = e - low.astype(e.dtype)
    s = (m - 1.0) / (m + 1.0)          # |s| <= 0.1716
    s2 = s * s
    acc = np.full_like(s, 1.0 / 25.0)
    for k in range(23, 0, -2):          # 2 * (s + s^3/3 + ... + s^25/25)
        acc = acc * s2 + 1.0 / k
    return 2.0 * s * acc + e.astype(np.float64) * _LN2


def det_exp(y: np.ndarray) -> np.ndarray:
    """exp(y) (float64): k = rint(y / ln2), Taylor series of the remainder, ldexp."""
    y = np.asarray(y, dtype=np.float64)
    k = np.rint(y / _LN2)
    r = y - k * _LN2                    # |r| <= 0.35
    acc = np.full_like(r, 1.0)
    for j in range(18, 0, -1):          # Horner form of sum r^j / j!
        acc = acc * (r / j) + 1.0
    return np.ldexp(acc, k.astype(np.int32))


def det_pow(x: np.ndarray, a: float) -> np.ndarray:
    return det_exp(a * det_log(x))


@dataclass
class Template:
    pixels: np.ndarray  # uint8 m x n
    row: int            # ground-truth cut location (-1 for pure-noise templates)
    col: int
    gain: float = 1.0
    offset: float = 0.0
    noise_sigma: float = 0.0


@dataclass
class Workload:
    name: str
    image: np.ndarray                     # uint8 p x q
    templates: list = field(default_factory=list)
    mode: str = "egs"                     # egs | opta
    gpus: tuple = (1,)
    description: str = ""

    @property
    def extent(self) -> int:
        m, n = self.templates[0].pixels.shape
        p, q = self.image.shape
        return (p - m + 1) * (q - n + 1)

    def sha256(self) -> str:
        h = hashlib.sha256(self.image.tobytes())
        for t in self.templates:
            h.update(t.pixels.tobytes())
        return h.hexdigest()


def _spectral_field(rng, rows, cols, beta, blur_sigmas=(0.0,)):
    """Return one float field per blur sigma, all sharing the same white noise.

    FP64 throughout; the spectral weights use det_pow/det_exp (bit-deterministic)."""
    white = rng.standard_normal((rows, cols))
    spec = _rfft2(white)
    fy = np.fft.fftfreq(rows)[:, None]          # k / rows: exact divisions
    fx = np.fft.rfftfreq(cols)[None, :]
    f2 = fy * fy + fx * fx
    f2[0, 0] = 1.0
    amp = det_pow(f2, -beta / 4.0)              # |f|^(-beta/2)
    amp[0, 0] = 0.0
    spec *= amp
    out = []
    for s in blur_sigmas:
        if s > 0:
            g = det_exp((-2.0 * np.pi ** 2 * s * s) * f2)
            out.append(_irfft2(spec * g, (rows, cols)))
        else:
            out.append(_irfft2(spec, (rows, cols)))
    return out


def _to_u8(x: np.ndarray) -> np.ndarray:
    lo, hi = float(x.min()), float(x.max())
    scale = 255.0 / (hi - lo) if hi > lo else 0.0
    y = np.rint((x - lo) * scale)
    return np.clip(y, 0, 255).astype(np.uint8)


def spectral_image(seed, rows, cols, beta=2.0, blur_sigma=0.0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    (f,) = _spectral_field(rng, rows, cols, beta, (blur_sigma,))
    return _to_u8(f)


def cut_template(rng, image, m, n, gain, offset, sigma, row=None, col=None) -> Template:
    p, q = image.shape
    if row is None:
        row = int(rng.integers(0, p - m + 1))
        col = int(rng.integers(0, q - n + 1))
    patch = image[row:row + m, col:col + n].astype(np.float64)
    noisy = gain * patch + offset + rng.normal(0.0, sigma, size=patch.shape)
    px = np.clip(np.rint(noisy), 0, 255).astype(np.uint8)
    return Template(px, row, col, gain, offset, sigma)


def noise_template(rng, m, n) -> Template:
    return Template(rng.integers(0, 256, size=(m, n), dtype=np.uint8), -1, -1)


# ---- the five BASELINE.json configs -------------------------------------------------

def config1(seed=101) -> Workload:
    """512^2 1/f^2 + blur sigma 1.0; one 32^2 template (gain .9, +10, noise 5)."""
    img = spectral_image(seed, 512, 512, beta=2.0, blur_sigma=1.0)
    rng = np.random.default_rng(seed + 1)
    t = cut_template(rng, img, 32, 32, 0.9, 10.0, 5.0)
    return Workload("C1", img, [t], "egs", (1,), "512x512 1/f^2+blur1, 32x32 template")


def config2(seed=202) -> Workload:
    """2048^2 1/f^1.8, half the 256^2 tiles from a sigma-2 blurred copy; one 64^2."""
    rng = np.random.default_rng(seed)
    base, smooth = _spectral_field(rng, 2048, 2048, 1.8, (0.0, 2.0))
    tiles = rng.random((8, 8)) < 0.5
    mask = np.kron(tiles, np.ones((256, 256), dtype=bool))
    img = _to_u8(np.where(mask, smooth, base))
    t = cut_template(np.random.default_rng(seed + 1), img, 64, 64, 1.1, -15.0, 8.0)
    return Workload("C2", img, [t], "egs", (1,),
                    "2048x2048 1/f^1.8 half tiles blurred sigma 2, 64x64 template")


def config3(seed=303, n_templates=8) -> Workload:
    """4096^2 1/f^2; 8 templates 128^2 with gain U[.8,1.2], offset U[-20,20], noise U[2,10]."""
    img = spectral_image(seed, 4096, 4096, beta=2.0)
    rng = np.random.default_rng(seed + 1)
    ts = [cut_template(rng, img, 128, 128, rng.uniform(0.8, 1.2), rng.uniform(-20, 20),
                       rng.uniform(2, 10)) for _ in range(n_templates)]
    return Workload("C3", img, ts, "opta", (1, 2), "4096x4096 1/f^2, 8x128^2 templates, OptA")


def config4(seed=404, n_present=12, n_noise=4) -> Workload:
    """8192^2 1/f^2; 16 templates 64^2: 12 cut + 4 pure uniform noise (no true match)."""
    img = spectral_image(seed, 8192, 8192, beta=2.0)
    rng = np.random.default_rng(seed + 1)
    ts = [cut_template(rng, img, 64, 64, rng.uniform(0.8, 1.2), rng.uniform(-20, 20),
                       rng.uniform(2, 10)) for _ in range(n_present)]
    ts += [noise_template(rng, 64, 64) for _ in range(n_noise)]
    return Workload("C4", img, ts, "egs", (4, 8), "8192x8192 1/f^2, 12+4 templates 64^2")


def config5(seed=505, size=16384) -> Workload:
    """16384^2 1/f^2 mixed with constant rectangles and high-frequency texture; one 96^2."""
    img = spectral_image(seed, size, size, beta=2.0)
    rng = np.random.default_rng(seed + 1)
    n_rect = max(4, size // 256)
    for _ in range(n_rect):  # piecewise-constant field-like regions (flat windows)
        h, w = rng.integers(size // 64, size // 12, size=2)
        r, c = rng.integers(0, size - h), rng.integers(0, size - w)
        img[r:r + h, c:c + w] = np.uint8(rng.integers(0, 256))
    for _ in range(n_rect):  # high-frequency texture patches
        h, w = rng.integers(size // 128, size // 24, size=2)
        r, c = rng.integers(0, size - h), rng.integers(0, size - w)
        tex = rng.integers(-40, 41, size=(h, w))
        img[r:r + h, c:c + w] = np.clip(img[r:r + h, c:c + w].astype(np.int32) + tex, 0,
                                        255).astype(np.uint8)
    t = cut_template(rng, img, 96, 96, 0.95, 5.0, 6.0)
    return Workload("C5", img, [t], "egs", (1, 2, 4, 8),
                    "16384x16384 1/f^2 + rectangles + texture, 96x96 template")


def config6(seed=707, n_templates=8) -> Workload:
    """Not a BASELINE config: OptA at scale with kappa > 0 (the reference accepts two blur
    iterations here), so the search runs on the non-integer blurred image -- 2048^2 1/f^2 +
    blur sigma 1.0 (C1's content at 16x the area), 8 templates 32^2 with C1's perturbation."""
    img = spectral_image(seed, 2048, 2048, beta=2.0, blur_sigma=1.0)
    rng = np.random.default_rng(seed + 1)
    ts = [cut_template(rng, img, 32, 32, 0.9, 10.0, 5.0) for _ in range(n_templates)]
    return Workload("C6", img, ts, "opta", (1,),
                    "2048x2048 1/f^2+blur1, 8x32^2 templates, OptA (kappa = 2)")


CONFIGS = {"C1": config1, "C2": config2, "C3": config3, "C4": config4, "C5": config5,
           "C6": config6}


def make(name: str, **kw) -> Workload:
    return CONFIGS[name](**kw)
