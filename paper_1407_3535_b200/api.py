"""Python mirror of the reference matcher API (proj/include/tmatch/*.hpp) over the C ABI.

Names, argument meaning and error behaviour follow the reference so the parity tests read
like its own tests: InvalidArgument carries the reference's std::invalid_argument text.
Images are numpy arrays (uint8 -> exact 8-bit path; float64 -> the reference's Image,
classified on the device).  Every call runs the sm_100a kernels; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import native as N
from .native import InvalidArgument, MatchResult, NoDeviceError, TmatchError  # noqa: F401

DEFAULT_PROFILE = (0.05, 0.20, 0.50, 0.20, 0.05)  # BlurKernel::default_profile (blur.cpp:20)


def _dptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _u8ptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


_PARAMS_CACHE: dict = {}


def cached_params(**kw):
    """make_params memoised on its (hashable) arguments: the per-call cost of building the
    struct is most of a small search's Python overhead.  The returned struct is shared and
    must not be modified."""
    try:
        key = tuple(sorted(kw.items()))
        hash(key)
    except TypeError:  # e.g. a numpy kernel profile
        return make_params(**kw)
    p = _PARAMS_CACHE.get(key)
    if p is None:
        if len(_PARAMS_CACHE) > 256:
            _PARAMS_CACHE.clear()
        p = _PARAMS_CACHE[key] = make_params(**kw)
    return p


def make_params(mode="egs", policy="reference", init_threshold=None, parallel=False, threads=2,
                h0=3, w0=3, rho_th=0.8, rho_max=0.95, xi_fraction=0.005, opta_margin=0.005,
                kernel=DEFAULT_PROFILE, record_visits=False, max_group=127, seed_margin=0.02):
    """MatchParams (matcher.hpp:45-58) + the B200 scan-2 policy."""
    p = N.MatchParams()
    N.lib().tm_default_params(C.byref(p))
    p.mode = N.MODE[mode] if isinstance(mode, str) else int(mode)
    p.policy = N.POLICY[policy] if isinstance(policy, str) else int(policy)
    p.has_init_threshold = init_threshold is not None
    p.init_threshold = float(init_threshold or 0.0)
    p.parallel = int(bool(parallel))
    p.threads = int(threads)
    p.h0, p.w0 = int(h0), int(w0)
    p.rho_th, p.rho_max = float(rho_th), float(rho_max)
    p.xi_fraction, p.opta_margin = float(xi_fraction), float(opta_margin)
    prof = np.ascontiguousarray(kernel, dtype=np.float64)
    p._profile = prof  # keep alive
    p.kernel_profile = _dptr(prof)
    p.kernel_len = len(prof)
    p.record_visits = int(bool(record_visits))
    p.max_group = int(max_group)
    p.seed_margin = float(seed_margin)
    return p


class Image:
    """Device-resident search image (reference Image, image.hpp:14-55)."""

    def __init__(self, ctx: "Context", pixels):
        self.ctx = ctx
        a = np.asarray(pixels)
        if a.ndim != 2:
            raise InvalidArgument("image dimensions must be at least 1x1")
        self.rows, self.cols = a.shape
        h = C.c_void_p()
        if a.dtype == np.uint8:
            a = np.ascontiguousarray(a)
            N.check(N.lib().tm_image_create_u8(ctx.h, _u8ptr(a), a.shape[0], a.shape[1],
                                               C.byref(h)))
        else:
            a = np.ascontiguousarray(a, dtype=np.float64)
            N.check(N.lib().tm_image_create(ctx.h, _dptr(a), a.shape[0], a.shape[1],
                                            C.byref(h)))
        self.h = h

    @classmethod
    def strip(cls, ctx: "Context", pixels, shape, row0: int):
        """A rows x cols 8-bit image holding only rows [row0, row0 + len(pixels)) -- one
        rank's strip + halo of a row-strip search (tm_image_create_strip_u8)."""
        a = np.ascontiguousarray(pixels, dtype=np.uint8)
        self = cls.__new__(cls)
        self.ctx = ctx
        self.rows, self.cols = int(shape[0]), int(shape[1])
        if a.ndim != 2 or a.shape[1] != self.cols:
            raise InvalidArgument("strip pixels must be nrows x cols")
        h = C.c_void_p()
        N.check(N.lib().tm_image_create_strip_u8(ctx.h, self.rows, self.cols, int(row0),
                                                 a.shape[0], _u8ptr(a), C.byref(h)))
        self.h = h
        self.row0, self.nrows = int(row0), a.shape[0]
        return self

    def upload_strip(self, pixels):
        a = np.ascontiguousarray(pixels, dtype=np.uint8)
        N.check(N.lib().tm_image_upload_strip_u8(self.ctx.h, self.h, _u8ptr(a)))

    def sum_sq_rows(self, row0: int, nrows: int) -> int:
        v = C.c_uint64()
        N.check(N.lib().tm_image_sum_sq_rows(self.ctx.h, self.h, int(row0), int(nrows),
                                             C.byref(v)))
        return v.value

    def set_noise_floor(self, q_total: int):
        N.check(N.lib().tm_image_set_noise_floor(self.ctx.h, self.h, C.c_uint64(int(q_total))))

    @property
    def is_integer(self) -> bool:
        return bool(N.lib().tm_image_is_integer(self.h))

    def reset_cache(self):
        N.check(N.lib().tm_image_reset_cache(self.h))

    def upload_u8(self, pixels):
        a = np.ascontiguousarray(pixels, dtype=np.uint8)
        N.check(N.lib().tm_image_upload_u8(self.ctx.h, self.h, _u8ptr(a)))

    def numpy(self) -> np.ndarray:
        out = np.empty((self.rows, self.cols))
        N.check(N.lib().tm_image_download(self.ctx.h, self.h, _dptr(out)))
        return out

    def close(self):
        if self.h:
            N.lib().tm_image_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class Prepared:
    """PreparedEgs / PreparedOptA (matcher.hpp:61-69), device resident."""
    ctx: "Context"
    h: C.c_void_p
    image: Image
    info: dict = field(default_factory=dict)

    def map(self) -> np.ndarray:
        out = np.empty((self.info["extent_rows"], self.info["extent_cols"]))
        N.check(N.lib().tm_prep_download(self.ctx.h, self.h, _dptr(out), None))
        return out

    def search_image(self) -> np.ndarray:
        out = np.empty((self.image.rows, self.image.cols))
        N.check(N.lib().tm_prep_download(self.ctx.h, self.h, None, _dptr(out)))
        return out

    def close(self):
        if self.h:
            N.lib().tm_prep_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _prep_info(h) -> dict:
    info = N.PrepInfo()
    N.check(N.lib().tm_prep_get_info(h, C.byref(info)))
    return dict(mode=info.mode, m=info.m, n=info.n, h=info.h, w=info.w,
                extent_rows=info.extent_rows, extent_cols=info.extent_cols, kappa=info.kappa,
                lam=info.lambda_, cost=info.cost.as_dict(),
                egs_trace=[info.egs_trace[k].as_dict() for k in range(info.egs_trace_len)],
                opta_trace=[info.opta_trace[k].as_dict() for k in range(info.opta_trace_len)],
                prep_ms=info.prep_ms)


class Context:
    """One device + stream (tm_ctx).  Raises NoDeviceError without an sm_100a GPU."""

    def __init__(self, device: int = 0):
        self.h = C.c_void_p()
        N.check(N.lib().tm_ctx_create(device, C.byref(self.h)))

    def close(self):
        if self.h:
            N.lib().tm_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def launches(self) -> int:
        return int(N.lib().tm_ctx_launch_count(self.h))

    @property
    def stream_ptr(self) -> int:
        return int(N.lib().tm_ctx_stream(self.h) or 0)

    def search_stats(self) -> dict:
        """tm_search h_e prediction outcomes: fused scan-2 path hit / missed."""
        h, m = C.c_int64(), C.c_int64()
        N.check(N.lib().tm_ctx_search_stats(self.h, C.byref(h), C.byref(m)))
        return {"fused_hits": h.value, "fused_misses": m.value}

    def split_stats(self) -> dict:
        """Split tensor-core screening of non-integer images: locations bracketed on the
        tensor cores / re-evaluated exactly by the FP64 replica."""
        a, b = C.c_int64(), C.c_int64()
        N.check(N.lib().tm_ctx_split_stats(self.h, C.byref(a), C.byref(b)))
        return {"screened": a.value, "exact": b.value}

    def set_profiling(self, enable=True):
        N.check(N.lib().tm_ctx_set_profiling(self.h, int(bool(enable))))

    def phase_times(self) -> dict:
        import json
        buf = C.create_string_buffer(1 << 16)
        N.check(N.lib().tm_ctx_phase_times(self.h, buf, len(buf)))
        return {k: {"count": v[0], "ms": v[1]} for k, v in json.loads(buf.value.decode()).items()}

    def synchronize(self):
        N.check(N.lib().tm_ctx_synchronize(self.h))

    def image(self, pixels) -> Image:
        return pixels if isinstance(pixels, Image) else Image(self, pixels)

    # ---- stats.hpp ----------------------------------------------------------------
    def running_sum(self, img, m, n):
        img = self.image(img)
        out = np.empty((img.rows - m + 1, img.cols - n + 1)) if m <= img.rows and n <= img.cols \
            else np.empty(1)
        N.check(N.lib().tm_running_sum(self.h, img.h, m, n, _dptr(out)))
        return out

    def window_stats(self, img, m, n):
        img = self.image(img)
        er, ec = max(img.rows - m + 1, 1), max(img.cols - n + 1, 1)
        mu, om = np.empty((er, ec)), np.empty((er, ec))
        fl = np.empty((er, ec), np.uint8)
        N.check(N.lib().tm_window_stats(self.h, img.h, m, n, _dptr(mu), _dptr(om), _u8ptr(fl)))
        return mu, om, fl

    def brute_force_match(self, t, img, record_surface=False):
        img = self.image(img)
        t = np.ascontiguousarray(t, dtype=np.float64)
        m, n = t.shape
        res = MatchResult()
        surf = np.empty((img.rows - m + 1, img.cols - n + 1)) if record_surface else None
        N.check(N.lib().tm_brute_force_match(self.h, _dptr(t), m, n, img.h, C.byref(res),
                                             _dptr(surf) if record_surface else None))
        return (res, surf) if record_surface else res

    # ---- autocorr.hpp / egs.hpp ---------------------------------------------------
    def local_autocorrelation(self, img, m, n, h, w):
        img = self.image(img)
        out = np.empty((max(img.rows - m + 1, 1), max(img.cols - n + 1, 1)))
        N.check(N.lib().tm_local_autocorrelation(self.h, img.h, m, n, h, w, _dptr(out)))
        return out

    def autocorr_retained(self, img, m, n, h, w, rho_tb=0.8):
        img = self.image(img)
        v = C.c_int64()
        N.check(N.lib().tm_autocorr_retained(self.h, img.h, m, n, h, w, rho_tb, C.byref(v)))
        return v.value

    def efficient_group_size(self, img, m, n, h0=3, w0=3, rho_tb=0.8, xi_fraction=0.005,
                             max_group=127, want_map=True):
        img = self.image(img)
        h, w, tl = C.c_int(), C.c_int(), C.c_int()
        tr = (N.EgsIter * N.TM_MAX_TRACE)()
        amap = np.empty((max(img.rows - m + 1, 1), max(img.cols - n + 1, 1))) if want_map \
            else None
        N.check(N.lib().tm_efficient_group_size(
            self.h, img.h, m, n, h0, w0, rho_tb, xi_fraction, max_group, C.byref(h),
            C.byref(w), tr, C.byref(tl), _dptr(amap) if want_map else None))
        return dict(h=h.value, w=w.value, map=amap,
                    trace=[tr[k].as_dict() for k in range(min(tl.value, N.TM_MAX_TRACE))])

    # ---- blur.hpp -------------------------------------------------------------------
    def blur(self, img, profile=DEFAULT_PROFILE):
        img = self.image(img)
        prof = np.ascontiguousarray(profile, dtype=np.float64)
        out = np.empty((img.rows, img.cols))
        N.check(N.lib().tm_blur(self.h, img.h, _dptr(prof), len(prof), _dptr(out)))
        return out

    def blur_fidelity_map(self, img, blurred, m, n):
        img, blurred = self.image(img), self.image(blurred)
        out = np.empty((max(img.rows - m + 1, 1), max(img.cols - n + 1, 1)))
        N.check(N.lib().tm_blur_fidelity_map(self.h, img.h, blurred.h, m, n, _dptr(out)))
        return out

    # ---- matcher.hpp ----------------------------------------------------------------
    def prepare(self, img, m, n, mode="egs", **kw) -> Prepared:
        img = self.image(img)
        p = make_params(mode=mode, **kw)
        h = C.c_void_p()
        N.check(N.lib().tm_prepare(self.h, img.h, m, n, C.byref(p), C.byref(h)))
        return Prepared(self, h, img, _prep_info(h))

    def prepare_egs(self, img, m, n, **kw):
        return self.prepare(img, m, n, mode="egs", **kw)

    def prepare_opta(self, img, m, n, **kw):
        return self.prepare(img, m, n, mode="opta", **kw)

    def run(self, prep: Prepared, templates, record_visits=False, **kw):
        """run_egs / run_opta for one template (2-D) or a batch (3-D)."""
        t = np.asarray(templates)
        single = t.ndim == 2
        if single:
            t = t[None]
        k = t.shape[0]
        res = (MatchResult * k)()
        p = make_params(mode=N.MODE["opta"] if prep.info["mode"] == 2 else N.MODE["egs"],
                        record_visits=record_visits, **kw)
        E = prep.info["extent_rows"] * prep.info["extent_cols"]
        vis = np.zeros((k, prep.info["extent_rows"], prep.info["extent_cols"]), np.uint8) \
            if record_visits else None
        if t.dtype == np.uint8:
            t = np.ascontiguousarray(t)
            N.check(N.lib().tm_run_u8(self.h, prep.h, prep.image.h, _u8ptr(t), k, C.byref(p),
                                      res, _u8ptr(vis) if record_visits else None))
        else:
            t = np.ascontiguousarray(t, dtype=np.float64)
            N.check(N.lib().tm_run(self.h, prep.h, prep.image.h, _dptr(t), k, C.byref(p), res,
                                   _u8ptr(vis) if record_visits else None))
        del E
        out = list(res)
        if record_visits:
            return (out[0], vis[0]) if single else (out, vis)
        return out[0] if single else out

    run_egs = run
    run_opta = run

    def transitive_search(self, t, img, amap, h, w, record_visits=False, ws=None, **kw):
        """transitive_search (matcher.hpp:37-38); `ws` = (mu, omega, flat) of a preparation
        (possibly of earlier pixels) in place of the image's own statistics."""
        img = self.image(img)
        t = np.ascontiguousarray(t, dtype=np.float64)
        amap = np.ascontiguousarray(amap, dtype=np.float64)
        m, n = t.shape
        p = make_params(record_visits=record_visits, **kw)
        res = MatchResult()
        vis = np.zeros(amap.shape, np.uint8) if record_visits else None
        if ws is None:
            N.check(N.lib().tm_transitive_search(self.h, _dptr(t), m, n, img.h, _dptr(amap), h,
                                                 w, C.byref(p), C.byref(res),
                                                 _u8ptr(vis) if record_visits else None))
        else:
            mu, om, fl = (np.ascontiguousarray(ws[0], np.float64),
                          np.ascontiguousarray(ws[1], np.float64),
                          np.ascontiguousarray(ws[2], np.uint8))
            N.check(N.lib().tm_transitive_search_ws(self.h, _dptr(t), m, n, img.h, _dptr(amap),
                                                    h, w, _dptr(mu), _dptr(om), _u8ptr(fl),
                                                    C.byref(p), C.byref(res),
                                                    _u8ptr(vis) if record_visits else None))
        return (res, vis) if record_visits else res

    def center_scan(self, t, img, h, w):
        img = self.image(img)
        t = np.ascontiguousarray(t, dtype=np.float64)
        m, n = t.shape
        er, ec = img.rows - m + 1, img.cols - n + 1
        G = ((er + h - 1) // h) * ((ec + w - 1) // w) if er > 0 and ec > 0 else 1
        rho, deg = np.empty(G), np.empty(G, np.uint8)
        br, bc, bd = C.c_int(), C.c_int(), C.c_int()
        brho = C.c_double()
        N.check(N.lib().tm_center_scan(self.h, _dptr(t), m, n, img.h, h, w, _dptr(rho),
                                       _u8ptr(deg), C.byref(br), C.byref(bc), C.byref(brho),
                                       C.byref(bd)))
        return dict(rho=rho, degenerate=deg, best=(br.value, bc.value, brho.value,
                                                   bool(bd.value)))

    def refine_localization(self, t, original, row, col, d):
        img = self.image(original)
        t = np.ascontiguousarray(t, dtype=np.float64)
        r, c, deg = C.c_int(), C.c_int(), C.c_int()
        rho = C.c_double()
        N.check(N.lib().tm_refine_localization(self.h, _dptr(t), t.shape[0], t.shape[1], img.h,
                                               row, col, d, C.byref(r), C.byref(c),
                                               C.byref(rho), C.byref(deg)))
        return r.value, c.value, rho.value, bool(deg.value)

    def search(self, img, t, mode="egs", **kw):
        """One full search on a device-resident image (tm_search / tm_search_u8): prepare +
        run in one call, the template upload overlapped with the preparation."""
        img = self.image(img)
        t = np.asarray(t)
        m, n = t.shape
        p = cached_params(mode=mode, **kw)
        res = MatchResult()
        if t.dtype == np.uint8:
            t = np.ascontiguousarray(t)
            N.check(N.lib().tm_search_u8(self.h, img.h, _u8ptr(t), m, n, C.byref(p), C.byref(res)))
        else:
            t = np.ascontiguousarray(t, dtype=np.float64)
            N.check(N.lib().tm_search(self.h, img.h, _dptr(t), m, n, C.byref(p), C.byref(res)))
        return res

    def search_upload(self, img, pixels, t, mode="egs", **kw):
        """match from host memory into a device image in one call (tm_search_upload_u8):
        upload the 8-bit pixels (img's shape), then the search."""
        if not isinstance(img, Image) or not img.is_integer:
            raise ValueError("search_upload: needs an 8-bit device image")
        px = np.ascontiguousarray(pixels, dtype=np.uint8)
        if px.shape != (img.rows, img.cols):
            raise ValueError("search_upload: pixel array shape differs from the image")
        t = np.ascontiguousarray(t, dtype=np.uint8)
        m, n = t.shape
        p = cached_params(mode=mode, **kw)
        res = MatchResult()
        N.check(N.lib().tm_search_upload_u8(self.h, img.h, _u8ptr(px), _u8ptr(t), m, n,
                                            C.byref(p), C.byref(res)))
        return res

    def search_stream(self, images, t, mode="egs", **kw):
        """match over a stream of 8-bit host images with one template
        (tm_search_stream_u8): image i+1 crosses PCIe while image i is searched.  `images`
        is a sequence of equally shaped uint8 arrays (pinned memory for an overlapped copy);
        returns one MatchResult per image."""
        imgs = [np.ascontiguousarray(a, dtype=np.uint8) for a in images]
        if not imgs:
            return []
        shape = imgs[0].shape
        if len(shape) != 2 or any(a.shape != shape for a in imgs):
            raise ValueError("search_stream: images must be equally shaped 2-D arrays")
        t = np.ascontiguousarray(t, dtype=np.uint8)
        m, n = t.shape
        p = cached_params(mode=mode, **kw)
        ptrs = (C.c_void_p * len(imgs))(*[a.ctypes.data for a in imgs])
        res = (MatchResult * len(imgs))()
        N.check(N.lib().tm_search_stream_u8(self.h, ptrs, len(imgs), shape[0], shape[1],
                                            _u8ptr(t), m, n, C.byref(p), res))
        return list(res)

    def match(self, t, image, mode="egs", record_visits=False, **kw):
        """match (matcher.hpp:80): host buffers in, host result out (end to end)."""
        t = np.ascontiguousarray(t, dtype=np.float64)
        a = np.ascontiguousarray(image, dtype=np.float64)
        m, n = t.shape
        p = make_params(mode=mode, record_visits=record_visits, **kw)
        res = MatchResult()
        vis = np.zeros((max(a.shape[0] - m + 1, 1), max(a.shape[1] - n + 1, 1)), np.uint8) \
            if record_visits else None
        N.check(N.lib().tm_match(self.h, _dptr(t), m, n, _dptr(a), a.shape[0], a.shape[1],
                                 C.byref(p), C.byref(res),
                                 _u8ptr(vis) if record_visits else None))
        return (res, vis) if record_visits else res
