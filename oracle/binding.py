"""ctypes binding for the CPU oracle libraries -- TEST INFRASTRUCTURE.

Two libraries export the same tmo_* C interface (oracle/tmatch_oracle.h):
  * "port": oracle/lib/libtmatch_oracle.so -- our C restatement of the reference;
  * "ref":  oracle/_ref/libtmatch_ref.so   -- the unmodified reference sources compiled
            by oracle/Makefile (only buildable where /root/reference exists; the built
            .so travels to the GPU box).
Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "lib", "libtmatch_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtmatch_ref.so")
DEFAULT_PROFILE = (0.05, 0.20, 0.50, 0.20, 0.05)


class TmoResult(C.Structure):
    _fields_ = [("mode", C.c_int32), ("best_row", C.c_int32), ("best_col", C.c_int32),
                ("best_degenerate", C.c_int32), ("best_rho", C.c_double),
                ("refined_row", C.c_int32), ("refined_col", C.c_int32),
                ("refined_rho", C.c_double), ("below_threshold", C.c_int32),
                ("extent_rows", C.c_int32), ("extent_cols", C.c_int32), ("_pad0", C.c_int32),
                ("final_threshold", C.c_double), ("centers", C.c_int64),
                ("eliminated", C.c_int64), ("retained", C.c_int64), ("ops", C.c_int64),
                ("elim_pct", C.c_double), ("wall_ms", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if not k.startswith("_")}


class TmoParams(C.Structure):
    _fields_ = [("mode", C.c_int32), ("h0", C.c_int32), ("w0", C.c_int32),
                ("has_init_threshold", C.c_int32), ("init_threshold", C.c_double),
                ("rho_th", C.c_double), ("rho_max", C.c_double), ("xi_fraction", C.c_double),
                ("opta_margin", C.c_double), ("kernel_profile", C.POINTER(C.c_double)),
                ("kernel_len", C.c_int32), ("parallel", C.c_int32), ("threads", C.c_int32),
                ("record_visits", C.c_int32)]


class TmoEgsIter(C.Structure):
    _fields_ = [("h", C.c_int32), ("w", C.c_int32), ("central", C.c_double),
                ("retained_cost", C.c_double), ("amortized", C.c_double),
                ("total", C.c_double), ("retained", C.c_int64)]


MODES = {"brute": 0, "egs": 1, "opta": 2}


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a, t=C.c_double):
    return a.ctypes.data_as(C.POINTER(t))


def build(kind="port"):
    target = "port" if kind == "port" else "ref"
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)


class Oracle:
    """One oracle library (port or reference) with numpy-friendly wrappers."""

    def __init__(self, kind="port", autobuild=True):
        self.kind = kind
        path = PORT_SO if kind == "port" else REF_SO
        if not os.path.exists(path) and autobuild:
            build(kind)
        self.lib = C.CDLL(path)
        L = self.lib
        L.tmo_last_error.restype = C.c_char_p
        L.tmo_zncc_at.restype = C.c_double
        L.tmo_group_count.restype = C.c_int64
        L.tmo_retained_count.restype = C.c_int64
        self._profile_keep = []

    def _check(self, rc):
        if rc != 0:
            raise ValueError(self.lib.tmo_last_error().decode())

    def params(self, mode="egs", init_threshold=None, parallel=False, threads=2, h0=3, w0=3,
               rho_th=0.8, rho_max=0.95, xi_fraction=0.005, opta_margin=0.005,
               kernel=DEFAULT_PROFILE):
        prof = np.ascontiguousarray(kernel, dtype=np.float64)
        self._profile_keep.append(prof)
        p = TmoParams()
        p.mode = MODES[mode] if isinstance(mode, str) else int(mode)
        p.h0, p.w0 = h0, w0
        p.has_init_threshold = init_threshold is not None
        p.init_threshold = 0.0 if init_threshold is None else float(init_threshold)
        p.rho_th, p.rho_max = rho_th, rho_max
        p.xi_fraction, p.opta_margin = xi_fraction, opta_margin
        p.kernel_profile = _ptr(prof)
        p.kernel_len = len(prof)
        p.parallel = int(bool(parallel))
        p.threads = int(threads)
        return p

    # -- stats ------------------------------------------------------------------------
    def running_sum(self, src, m, n):
        src = _d(src)
        p, q = src.shape
        out = np.empty((p - m + 1, q - n + 1))
        self._check(self.lib.tmo_running_sum(_ptr(src), p, q, m, n, _ptr(out)))
        return out

    def window_stats(self, img, m, n):
        img = _d(img)
        p, q = img.shape
        er, ec = p - m + 1, q - n + 1
        mu, om = np.empty((er, ec)), np.empty((er, ec))
        fl = np.empty((er, ec), dtype=np.uint8)
        self._check(self.lib.tmo_window_stats(_ptr(img), p, q, m, n, _ptr(mu), _ptr(om),
                                              _ptr(fl, C.c_uint8)))
        return mu, om, fl

    def window_stats_floor(self, img, m, n, floor):
        """Port only: window_stats with the flat-noise floor of a larger image."""
        img = _d(img)
        p, q = img.shape
        er, ec = p - m + 1, q - n + 1
        mu, om = np.empty((er, ec)), np.empty((er, ec))
        fl = np.empty((er, ec), dtype=np.uint8)
        self._check(self.lib.tmo_window_stats_floor(_ptr(img), p, q, m, n, C.c_double(floor),
                                                    _ptr(mu), _ptr(om), _ptr(fl, C.c_uint8)))
        return mu, om, fl

    def template_stats(self, t):
        t = _d(t)
        mu, om, fl = C.c_double(), C.c_double(), C.c_int()
        self.lib.tmo_template_stats(_ptr(t), t.shape[0], t.shape[1], C.byref(mu), C.byref(om),
                                    C.byref(fl))
        return mu.value, om.value, bool(fl.value)

    def brute(self, t, img, surface=False):
        t, img = _d(t), _d(img)
        m, n = t.shape
        p, q = img.shape
        res = TmoResult()
        surf = np.empty((p - m + 1, q - n + 1)) if surface else None
        self._check(self.lib.tmo_brute(_ptr(t), m, n, _ptr(img), p, q, C.byref(res),
                                       _ptr(surf) if surface else None))
        return (res, surf) if surface else res

    # -- bounds -----------------------------------------------------------------------
    def transitive_bounds(self, a, b):
        lo, hi = C.c_double(), C.c_double()
        self._check(self.lib.tmo_transitive_bounds(C.c_double(a), C.c_double(b), C.byref(lo),
                                                   C.byref(hi)))
        return lo.value, hi.value

    def transitive_gap(self, a, b):
        g = C.c_double()
        self._check(self.lib.tmo_transitive_gap(C.c_double(a), C.c_double(b), C.byref(g)))
        return g.value

    def sec_holds(self, tb, a, b):
        h = C.c_int()
        self._check(self.lib.tmo_sec_holds(C.c_double(tb), C.c_double(a), C.c_double(b),
                                           C.byref(h)))
        return bool(h.value)

    def elimination_autocorr_threshold(self, tb, tc):
        o = C.c_double()
        self._check(self.lib.tmo_elimination_autocorr_threshold(C.c_double(tb), C.c_double(tc),
                                                                C.byref(o)))
        return o.value

    def expected_elimination_threshold(self, tb):
        o = C.c_double()
        self._check(self.lib.tmo_expected_elimination_threshold(C.c_double(tb), C.byref(o)))
        return o.value

    def quality_threshold(self, a, b):
        o = C.c_double()
        self._check(self.lib.tmo_quality_threshold(C.c_double(a), C.c_double(b), C.byref(o)))
        return o.value

    # -- autocorrelation / EGS ------------------------------------------------------------
    def group_count(self, er, ec, h, w):
        g = self.lib.tmo_group_count(er, ec, h, w)
        if g < 0:
            raise ValueError(self.lib.tmo_last_error().decode())
        return g

    def local_autocorrelation(self, img, m, n, h, w, ws=None):
        img = _d(img)
        p, q = img.shape
        mu, om, fl = ws if ws is not None else self.window_stats(img, m, n)
        out = np.empty_like(mu)
        self._check(self.lib.tmo_local_autocorrelation(
            _ptr(img), p, q, m, n, h, w, _ptr(_d(mu)), _ptr(_d(om)),
            _ptr(np.ascontiguousarray(fl, np.uint8), C.c_uint8), _ptr(out)))
        return out

    def retained_count(self, amap, h, w, rho_tb=0.8):
        amap = _d(amap)
        r = self.lib.tmo_retained_count(_ptr(amap), amap.shape[0], amap.shape[1], h, w,
                                        C.c_double(rho_tb))
        if r < 0:
            raise ValueError(self.lib.tmo_last_error().decode())
        return r

    def efficient_group_size(self, img, m, n, h0=3, w0=3, rho_tb=0.8, xi=0.005, max_group=127,
                             ws=None, want_map=True):
        img = _d(img)
        p, q = img.shape
        mu, om, fl = ws if ws is not None else self.window_stats(img, m, n)
        h, w, tl = C.c_int(), C.c_int(), C.c_int()
        tr = (TmoEgsIter * 64)()
        amap = np.empty_like(mu) if want_map else None
        self._check(self.lib.tmo_efficient_group_size(
            _ptr(img), p, q, m, n, h0, w0, C.c_double(rho_tb), C.c_double(xi), max_group,
            _ptr(_d(mu)), _ptr(_d(om)), _ptr(np.ascontiguousarray(fl, np.uint8), C.c_uint8),
            C.byref(h), C.byref(w), tr, 64, C.byref(tl), _ptr(amap) if want_map else None))
        trace = [dict(h=tr[k].h, w=tr[k].w, central=tr[k].central, retained=tr[k].retained,
                      total=tr[k].total) for k in range(min(tl.value, 64))]
        return dict(h=h.value, w=w.value, trace=trace, map=amap)

    # -- blur / OptA ----------------------------------------------------------------------
    def blur(self, img, profile=DEFAULT_PROFILE):
        img = _d(img)
        prof = np.ascontiguousarray(profile, np.float64)
        out = np.empty_like(img)
        self._check(self.lib.tmo_blur(_ptr(img), img.shape[0], img.shape[1], _ptr(prof),
                                      len(prof), _ptr(out)))
        return out

    def blur_fidelity_map(self, img, blurred, m, n):
        img, blurred = _d(img), _d(blurred)
        p, q = img.shape
        out = np.empty((p - m + 1, q - n + 1))
        self._check(self.lib.tmo_blur_fidelity_map(_ptr(img), _ptr(blurred), p, q, m, n,
                                                   _ptr(out)))
        return out

    def optimize_autocorrelation(self, img, m, n, **kw):
        img = _d(img)
        p, q = img.shape
        prm = self.params(**kw)
        out = np.empty_like(img)
        amap = np.empty((p - m + 1, q - n + 1))
        kappa, h, w, tl = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        lam, cost = C.c_double(), C.c_double()
        tr = np.zeros(4 * 65)
        self._check(self.lib.tmo_optimize_autocorrelation(
            _ptr(img), p, q, m, n, C.byref(prm), _ptr(out), C.byref(kappa), C.byref(lam),
            C.byref(h), C.byref(w), C.byref(cost), _ptr(tr), 65, C.byref(tl), _ptr(amap)))
        trace = [dict(h=int(tr[4 * k]), w=int(tr[4 * k + 1]), cost=tr[4 * k + 2],
                      restored=int(tr[4 * k + 3])) for k in range(tl.value)]
        return dict(image=out, kappa=kappa.value, lam=lam.value, h=h.value, w=w.value,
                    cost=cost.value, trace=trace, map=amap)

    # -- search -----------------------------------------------------------------------
    def transitive_search(self, t, img, amap, h, w, ws=None, init_threshold=None,
                          parallel=False, threads=2, visits=False):
        t, img, amap = _d(t), _d(img), _d(amap)
        m, n = t.shape
        p, q = img.shape
        mu, om, fl = ws if ws is not None else self.window_stats(img, m, n)
        res = TmoResult()
        vis = np.zeros(amap.shape, np.uint8) if visits else None
        self._check(self.lib.tmo_transitive_search(
            _ptr(t), m, n, _ptr(img), p, q, _ptr(amap), h, w, _ptr(_d(mu)), _ptr(_d(om)),
            _ptr(np.ascontiguousarray(fl, np.uint8), C.c_uint8),
            int(init_threshold is not None), C.c_double(init_threshold or 0.0),
            int(parallel), threads, C.byref(res), _ptr(vis, C.c_uint8) if visits else None))
        return (res, vis) if visits else res

    def refine(self, t, img, row, col, d):
        t, img = _d(t), _d(img)
        r, c, rho, deg = C.c_int(), C.c_int(), C.c_double(), C.c_int()
        self._check(self.lib.tmo_refine(_ptr(t), t.shape[0], t.shape[1], _ptr(img),
                                        img.shape[0], img.shape[1], row, col, d, C.byref(r),
                                        C.byref(c), C.byref(rho), C.byref(deg)))
        return r.value, c.value, rho.value, bool(deg.value)

    def match(self, t, img, visits=False, **kw):
        t, img = _d(t), _d(img)
        m, n = t.shape
        p, q = img.shape
        prm = self.params(**kw)
        res = TmoResult()
        vis = np.zeros((p - m + 1, q - n + 1), np.uint8) if visits else None
        self._check(self.lib.tmo_match(_ptr(t), m, n, _ptr(img), p, q, C.byref(prm),
                                       C.byref(res), _ptr(vis, C.c_uint8) if visits else None))
        return (res, vis) if visits else res

    # -- reference-only extras ----------------------------------------------------------
    def synth_corpus(self, rows, cols, sigma, count, m, per_size, seed):
        assert self.kind == "ref", "synth_corpus needs the reference build"
        imgs = np.empty((count, rows, cols))
        ents = np.empty((count * per_size, 2), dtype=np.int32)
        self._check(self.lib.ref_synth_corpus(rows, cols, C.c_double(sigma), count, m,
                                              per_size, C.c_uint64(seed), _ptr(imgs),
                                              _ptr(ents, C.c_int)))
        return imgs, ents

    def prepare_run_egs(self, t, img, parallel=True, threads=None):
        assert self.kind == "ref"
        t, img = _d(t), _d(img)
        threads = threads or os.cpu_count()
        res = TmoResult()
        pm, rm = C.c_double(), C.c_double()
        self._check(self.lib.ref_prepare_run_egs(_ptr(t), t.shape[0], t.shape[1], _ptr(img),
                                                 img.shape[0], img.shape[1], int(parallel),
                                                 threads, C.byref(res), C.byref(pm),
                                                 C.byref(rm)))
        return res, pm.value, rm.value

    def brute_threads(self, t, img, threads=None):
        """brute_force_match with the reference's own thread pool (stats.cpp:186-195)."""
        assert self.kind == "ref"
        t, img = _d(t), _d(img)
        res = TmoResult()
        self._check(self.lib.ref_brute_threads(_ptr(t), t.shape[0], t.shape[1], _ptr(img),
                                               img.shape[0], img.shape[1],
                                               threads or os.cpu_count(), C.byref(res)))
        return res

    def prepare_run_batch(self, tmpls, img, mode="egs", parallel=True, threads=None):
        """One prepare_egs/prepare_opta + run_* per template (cmd_bench's cache,
        cli.cpp:213-237).  Returns (results, info{h,w,kappa,lambda}, prep_ms, run_ms[])."""
        assert self.kind == "ref"
        tm = np.ascontiguousarray(np.stack([_d(t) for t in tmpls]))
        img = _d(img)
        k, m, n = tm.shape
        res = (TmoResult * k)()
        info = np.zeros(4)
        run_ms = np.zeros(k)
        pm = C.c_double()
        self._check(self.lib.ref_prepare_run_batch(
            _ptr(tm), k, m, n, _ptr(img), img.shape[0], img.shape[1], MODES[mode],
            int(parallel), threads or os.cpu_count(), res, _ptr(info), C.byref(pm),
            _ptr(run_ms)))
        return list(res), dict(h=int(info[0]), w=int(info[1]), kappa=int(info[2]),
                               lam=float(info[3])), pm.value, run_ms

    def content_hash(self, img):
        assert self.kind == "ref"
        img = _d(img)
        self.lib.ref_content_hash.restype = C.c_uint64
        return self.lib.ref_content_hash(_ptr(img), img.shape[0], img.shape[1])

    def autocorr_cache_key(self, img, m, n, h, w):
        assert self.kind == "ref"
        img = _d(img)
        self.lib.ref_autocorr_cache_key.restype = C.c_uint64
        return self.lib.ref_autocorr_cache_key(_ptr(img), img.shape[0], img.shape[1], m, n,
                                               h, w)

    def save_autocorr(self, amap, h, w, key, path):
        assert self.kind == "ref"
        amap = _d(amap)
        self._check(self.lib.ref_save_autocorr(_ptr(amap), amap.shape[0], amap.shape[1], h, w,
                                               C.c_uint64(key), path.encode()))

    def load_autocorr(self, path, key, rows, cols, h, w):
        assert self.kind == "ref"
        out = np.empty((rows, cols))
        ok = self.lib.ref_load_autocorr(path.encode(), C.c_uint64(key), rows, cols, h, w,
                                        _ptr(out))
        return out if ok else None

    def load_image(self, path):
        assert self.kind == "ref"
        r, c = C.c_int(), C.c_int()
        self._check(self.lib.ref_load_image(path.encode(), C.byref(r), C.byref(c), None, 0))
        out = np.empty((r.value, c.value))
        self._check(self.lib.ref_load_image(path.encode(), C.byref(r), C.byref(c), _ptr(out),
                                            out.size))
        return out

    def save_image(self, img, path):
        assert self.kind == "ref"
        img = _d(img)
        self._check(self.lib.ref_save_image(_ptr(img), img.shape[0], img.shape[1],
                                            path.encode()))



def available(kind):
    return os.path.exists(PORT_SO if kind == "port" else REF_SO)
