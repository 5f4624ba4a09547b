"""Row-strip sharding of one search across GPUs.

One process per GPU (torch.distributed; NCCL between GPUs, gloo for the CPU tests).  Every
rank holds the whole search image (8-bit: 268 MB at 16384^2, small against 180 GB of HBM);
the group grid's rows are split evenly, rank r owning group rows
[floor(r*tr/W), floor((r+1)*tr/W)) -- whole groups, so no group straddles a strip and each
strip's windows read the template_height-1 rows below it from the replicated image (the
"halo").  The exchanges are the few scalars the reference's control flow needs:

* EGS (egs.cpp:39-91): per candidate group size, each rank builds the R_co map of its
  strip and counts its retained members; an allreduce SUM gives the global n_r, and every
  rank takes the same accept/stop decision (the cost model is integer arithmetic).
* Scan 1 -> threshold (matcher.cpp:121-125): allreduce MAX of the strip maxima.  This is
  exactly the reference's frozen threshold, so strip results equal the reference's
  `--parallel` results for any W.
* Seeded policy: allreduce MAX of the seeded thresholds.
* Merge (matcher.cpp:150-153): allgather of each strip's best cell, merged in
  better_candidate order (a strict total order, so the result is W-independent), and sums
  of the counts.

The orchestration is backend-agnostic: `DeviceBackend` drives the sm_100a kernels through
the C ABI (tm_strip_*); tests/test_distributed.py also runs it with a NumPy backend over
gloo on CPU to check the protocol without a GPU.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import native as N


StripPart = N.StripPart


def strip_rows(tr: int, rank: int, world: int) -> tuple:
    """Group rows [lo, hi) of rank `rank` (tm_strip_*: an even split of the grid rows)."""
    return (tr * rank) // world, (tr * (rank + 1)) // world


def noise_rows(p: int, rank: int, world: int) -> tuple:
    """Image rows whose squares rank `rank` sums for the image-global q_total (stats.cpp:79):
    a disjoint partition, allreduced by SUM."""
    return (p * rank) // world, (p * (rank + 1)) // world


HOLD_GROUP = 15  # group sizes a strip image covers up front (EGS rarely passes h = 7)


def strip_image_rows(p: int, q: int, m: int, n: int, rank: int, world: int, h0: int = 3,
                     max_group: int = HOLD_GROUP, pad: int = 16) -> tuple:
    """Image rows [lo, hi) a rank must hold for a strip-local EGS search: for every group
    size up to `max_group` (h0, h0+2, ...), the extent rows of the rank's group rows plus
    the template_height-1 halo below them (windows reach m-1 rows down), plus the rank's
    noise rows; `pad` rows of slack below (row walks read a few rows ahead).  A larger
    candidate makes the backend extend its rows (DeviceBackend.autocorr)."""
    er = p - m + 1
    cap = max_group if max_group > 0 else 2 ** 31 - 1
    if cap % 2 == 0:
        cap += 1
    lo, hi = noise_rows(p, rank, world)
    h = h0
    while True:
        tr = (er + h - 1) // h
        a, b = strip_rows(tr, rank, world)
        if b > a:
            lo = min(lo, a * h)
            hi = max(hi, min(b * h, er) + m - 1)
        if h >= er or h >= cap:
            break
        h = min(h + 2, cap)
    return max(0, lo), min(p, hi + pad)


# ---- cell order (stats.cpp:147-154) --------------------------------------------------------
def better(a: dict, b: dict) -> bool:
    """better_candidate: valid, non-degenerate > degenerate, larger rho, smaller (row, col)."""
    if not a["valid"]:
        return False
    if not b["valid"]:
        return True
    if a["degenerate"] != b["degenerate"]:
        return not a["degenerate"]
    if a["rho"] != b["rho"]:
        return a["rho"] > b["rho"]
    if a["row"] != b["row"]:
        return a["row"] < b["row"]
    return a["col"] < b["col"]


def cell_from_part(part: dict) -> dict:
    return dict(rho=part["best_rho"], row=part["best_row"], col=part["best_col"],
                valid=bool(part["best_flags"] & 1), degenerate=bool(part["best_flags"] & 2))


# ---- communication -----------------------------------------------------------------------
class Comm:
    """Scalar collectives over a torch.distributed process group."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.dist, self.torch, self.group = dist, torch, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        backend = dist.get_backend(group)
        self.device = device or (torch.device("cuda", torch.cuda.current_device())
                                 if backend == "nccl" else torch.device("cpu"))

    def allreduce_sum_i64(self, vals):
        t = self.torch.tensor(list(vals), dtype=self.torch.int64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return [int(v) for v in t.cpu().tolist()]

    def allreduce_max_f64(self, v: float) -> float:
        t = self.torch.tensor([v], dtype=self.torch.float64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def allgather_f64(self, vals):
        t = self.torch.tensor(list(vals), dtype=self.torch.float64, device=self.device)
        out = [self.torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return [o.cpu().tolist() for o in out]


# ---- EGS over strips (egs.cpp:39-91) ------------------------------------------------------
def total_cost(er, ec, h, w, n_r, amortized=0.0):
    central = float((er + h - 1) // h) * float((ec + w - 1) // w)
    return dict(h=h, w=w, central=central, retained=int(n_r), retained_cost=float(n_r),
                amortized=amortized, total=central + float(n_r) + amortized)


def egs_strips(backend, comm, p, q, m, n, h0=3, w0=3, rho_tb=0.8, xi=0.005, max_group=127):
    """Group-size search with the retained count summed over strips; returns the accepted
    (h, w, trace, slot) -- identical on every rank."""
    if h0 < 1 or w0 < 1 or h0 % 2 == 0 or w0 % 2 == 0:
        raise N.InvalidArgument("efficient_group_size: initial group size must be odd")
    if not (0.0 < rho_tb < 1.0):
        raise N.InvalidArgument("efficient_group_size: rho_tb must be in (0,1)")
    er, ec = p - m + 1, q - n + 1
    if er < 1 or ec < 1:
        raise N.InvalidArgument("efficient_group_size: template does not fit")
    cap = max_group if max_group > 0 else 2 ** 31 - 1
    if cap % 2 == 0:
        cap += 1
    prev, h, w = math.inf, h0, w0
    best, trace, slot, best_slot = None, [], 0, None
    while True:
        n_r_local = backend.autocorr(m, n, h, w, comm.rank, comm.world, rho_tb, slot)
        (n_r,) = comm.allreduce_sum_i64([n_r_local])
        cost = total_cost(er, ec, h, w, n_r)
        if math.isfinite(prev) and not (prev - cost["total"] > xi * prev):
            break
        best, best_slot = (h, w), slot
        trace.append(cost)
        prev = cost["total"]
        slot = 1 - slot  # the accepted map stays in best_slot
        if (h >= er and w >= ec) or (h >= cap and w >= cap):
            break
        h, w = min(h + 2, cap), min(w + 2, cap)
    return best[0], best[1], trace, best_slot


# ---- search over strips (matcher.cpp:95-177) ----------------------------------------------
@dataclass
class StripResult:
    best_row: int
    best_col: int
    best_rho: float
    best_degenerate: bool
    refined_row: int
    refined_col: int
    refined_rho: float
    below_threshold: bool
    final_threshold: float
    centers: int
    eliminated: int
    retained: int
    ops: int
    elim_pct: float
    extent_rows: int
    extent_cols: int

    def as_dict(self):
        return dict(self.__dict__)


def search_strips(backend, comm, prep, t, er, ec, policy="frozen", init_threshold=None,
                  seed_margin=0.02):
    """Scan 1 / threshold / [seed] / scan 2 on this rank's strip, merged over all ranks."""
    T0 = backend.search_begin(prep, t, comm.rank, comm.world, policy, init_threshold,
                              seed_margin)
    T = comm.allreduce_max_f64(T0)
    if policy == "seeded":
        T = comm.allreduce_max_f64(backend.search_seed(T))
    part = backend.search_finish(T)
    return _merge_parts(comm, part, T, policy, init_threshold, er, ec)


def _merge_parts(comm, part, T, policy, init_threshold, er, ec):
    """allgather of the strips' parts, merged in better_candidate order (matcher.cpp:150-153)."""
    vec = [part["best_rho"], part["best_row"], part["best_col"], part["best_flags"],
           part["centers"], part["eliminated"], part["retained"], part["final_threshold"]]
    parts = comm.allgather_f64(vec)
    best = dict(valid=False, degenerate=True, rho=0.0, row=-1, col=-1)
    centers = elim = kept = 0
    fin = -math.inf
    for v in parts:
        c = dict(rho=v[0], row=int(v[1]), col=int(v[2]), valid=bool(int(v[3]) & 1),
                 degenerate=bool(int(v[3]) & 2))
        if better(c, best):
            best = c
        centers += int(v[4])
        elim += int(v[5])
        kept += int(v[6])
        fin = max(fin, v[7])
    final = T if policy != "seeded" else fin
    below = init_threshold is not None and (best["degenerate"] or best["rho"] < init_threshold)
    return StripResult(best["row"], best["col"], best["rho"], best["degenerate"], best["row"],
                       best["col"], best["rho"], below, final if math.isfinite(final) else 0.0,
                       centers, elim, kept, centers + kept, 100.0 * elim / (float(er) * float(ec)),
                       er, ec)


def _egs_accepts(er, ec, cands, counts, xi, cap=127):
    """egs.cpp:61-88 on the allreduced counts of one candidate batch: (accepted h, complete)
    -- complete = False when every candidate was accepted and larger sizes could follow."""
    if cap % 2 == 0:
        cap += 1
    prev, acc = math.inf, None
    for h, n_r in zip(cands, counts):
        cost = total_cost(er, ec, h, h, n_r)["total"]
        if math.isfinite(prev) and not (prev - cost > xi * prev):
            return acc, True
        acc, prev = h, cost
        if (h >= er and h >= ec) or h >= cap:
            return acc, True
    return acc, False


def search_strips_fused(backend, comm, t, er, ec, policy, init_threshold, h0, xi, seed_margin):
    """The fused strip protocol (tm_strip_fused_*): 4 host round trips, scan 2 inside the
    predicted size's R_co.  Returns None when it does not apply or the prediction missed
    (the caller runs the classic protocol)."""
    pred = getattr(backend, "predicted", None) or h0
    ok, T0 = backend.fused_begin(t, comm.rank, comm.world, policy, init_threshold, pred,
                                 seed_margin)
    (ok_all,) = comm.allreduce_sum_i64([int(ok)])
    if ok_all != comm.world:
        return None
    T = comm.allreduce_max_f64(T0)
    if policy == "seeded":
        T = comm.allreduce_max_f64(backend.fused_seed(T))
    cands, local = backend.fused_egs(T)
    counts = comm.allreduce_sum_i64(local)
    acc, complete = _egs_accepts(er, ec, cands, counts, xi)
    backend.predicted = acc if acc else pred
    if not complete or acc != pred:
        return None  # misprediction: the classic protocol on the accepted grid
    part = backend.fused_finish()
    return _merge_parts(comm, part, T, policy, init_threshold, er, ec)


def match_strips(backend, comm, t, image_shape, mode="egs", policy="frozen", init_threshold=None,
                 h0=3, w0=3, rho_th=0.8, xi_fraction=0.005, seed_margin=0.02):
    """match() (matcher.cpp:278-307) with the grid rows split over the process group."""
    m, n = t.shape
    p, q = image_shape
    er, ec = p - m + 1, q - n + 1
    if mode == "egs" and getattr(backend, "strip_local", False) and not backend.noise_set:
        # strip-local window statistics need the image-global flat-noise floor
        # (stats.cpp:78-81): each rank sums the squares of a disjoint row range
        r0, r1 = noise_rows(p, comm.rank, comm.world)
        (q_total,) = comm.allreduce_sum_i64([backend.sum_sq(r0, r1)])
        backend.set_noise(q_total)
    if (mode == "egs" and h0 == w0 and policy in ("frozen", "seeded") and rho_th == 0.8 and
            hasattr(backend, "fused_begin")):
        res = search_strips_fused(backend, comm, t, er, ec, policy, init_threshold, h0,
                                  xi_fraction, seed_margin)
        if res is not None:
            return res
    if mode == "egs":
        h, w, trace, slot = egs_strips(backend, comm, p, q, m, n, h0, w0, rho_th, xi_fraction)
        prep = backend.commit(m, n, slot, h, w, trace)
        res = search_strips(backend, comm, prep, t, er, ec, policy, init_threshold, seed_margin)
        return res
    if mode == "opta":
        # the OptA preparation (blur / repair fixed point / EGS on the blurred image) runs
        # replicated on every rank; the search is strip-sharded, the refinement replicated
        prep, kappa, radius = backend.prepare_opta(m, n)
        res = search_strips(backend, comm, prep, t, er, ec, policy, init_threshold, seed_margin)
        r, c, rho, deg = backend.refine(t, res.best_row, res.best_col, kappa * radius)
        res.refined_row, res.refined_col, res.refined_rho = r, c, rho
        res.ops += (min(er - 1, res.best_row + kappa * radius) -
                    max(0, res.best_row - kappa * radius) + 1) * \
                   (min(ec - 1, res.best_col + kappa * radius) -
                    max(0, res.best_col - kappa * radius) + 1)
        if init_threshold is not None:
            res.below_threshold = deg or rho < init_threshold
        return res
    raise N.InvalidArgument("match_strips: mode must be egs or opta")


# ---- the GPU backend (C ABI) -----------------------------------------------------------------
class DeviceBackend:
    """tm_strip_* primitives on one GPU (one context and one resident image per rank).

    `DeviceBackend(ctx, image)` holds the whole image (OptA: the blur / repair passes need
    every row); `DeviceBackend.strip(...)` holds only the rank's rows (EGS): window
    statistics and R_co are computed for its strip only, with the global noise floor."""

    strip_local = False
    noise_set = False

    def __init__(self, ctx, image):
        from .api import Image
        self.ctx = ctx
        self.img = image if isinstance(image, Image) else ctx.image(image)
        self._preps = []

    @classmethod
    def strip(cls, ctx, image, m, n, rank, world, h0=3, hold=HOLD_GROUP):
        """Upload only rows strip_image_rows(...) of `image` (a full host array, kept by
        reference for a later extension)."""
        from .api import Image
        p, q = image.shape
        lo, hi = strip_image_rows(p, q, m, n, rank, world, h0, hold)
        self = cls(ctx, Image.strip(ctx, image[lo:hi], image.shape, lo))
        self.strip_local = True
        self.rows = (lo, hi)
        self.host, self.mn, self.h0, self.hold = image, (m, n), h0, hold
        return self

    def _extend(self, h):
        """EGS reached a group size beyond the held rows: re-upload a wider strip (the
        noise floor is image-global, so it carries over)."""
        from .api import Image
        m, n = self.mn
        p, q = self.host.shape
        lo, hi = strip_image_rows(p, q, m, n, self.rank, self.world, self.h0, h)
        q_total = self.q_total
        self.close()
        self.img.close()
        self.img = Image.strip(self.ctx, self.host[lo:hi], self.host.shape, lo)
        self.rows, self.hold = (lo, hi), h
        self.img.set_noise_floor(q_total)

    def sum_sq(self, r0, r1):
        return self.img.sum_sq_rows(r0, r1 - r0)

    def set_noise(self, q_total):
        self.img.set_noise_floor(q_total)
        self.q_total = q_total
        self.noise_set = True

    def upload_rows(self, rows):
        """New pixels for the same strip, given as this rank's rows only (the rows
        strip_image_rows chose; e.g. a pinned host buffer of just those rows)."""
        self.img.upload_strip(rows)
        self.noise_set = False
        self.reset()

    def upload(self, image):
        """New pixels for the same strip (e2e); the noise floor must be set again."""
        lo, hi = self.rows if self.strip_local else (0, image.shape[0])
        if self.strip_local:
            self.img.upload_strip(image[lo:hi])
        else:
            self.img.upload_u8(image)
        self.noise_set = False
        self.reset()

    def reset(self):
        """Drop per-search state (cached window statistics, preparations)."""
        self.img.reset_cache()
        self.close()

    def autocorr(self, m, n, h, w, rank, world, rho_tb, slot):
        if self.strip_local and max(h, w) > self.hold:
            self.rank, self.world = rank, world
            self._extend(max(h, w))
        v = C.c_int64()
        N.check(N.lib().tm_strip_autocorr(self.ctx.h, self.img.h, m, n, h, w, rank, world,
                                          C.c_double(rho_tb), slot, C.byref(v)))
        return v.value

    def commit(self, m, n, slot, h, w, trace):
        from .api import make_params
        tr = (N.EgsIter * max(1, len(trace)))()
        for k, c in enumerate(trace):
            tr[k].h, tr[k].w, tr[k].central = c["h"], c["w"], c["central"]
            tr[k].retained, tr[k].retained_cost = c["retained"], c["retained_cost"]
            tr[k].amortized, tr[k].total = c["amortized"], c["total"]
        p = make_params()
        h_out = C.c_void_p()
        N.check(N.lib().tm_strip_commit(self.ctx.h, self.img.h, m, n, slot, h, w, C.byref(p), tr,
                                        len(trace), C.byref(h_out)))
        self._preps.append(h_out)
        return h_out

    def prepare_opta(self, m, n, kernel=None):
        from .api import DEFAULT_PROFILE
        kernel = DEFAULT_PROFILE if kernel is None else kernel
        prep = self.ctx.prepare(self.img, m, n, mode="opta", kernel=kernel)
        self._preps.append(prep)
        return prep.h, prep.info["kappa"], len(kernel) // 2

    def search_begin(self, prep, t, rank, world, policy, init_threshold, seed_margin):
        from .api import make_params
        self._t = np.ascontiguousarray(t, dtype=np.float64)
        p = make_params(policy=policy, init_threshold=init_threshold, seed_margin=seed_margin,
                        parallel=True, threads=2)
        T0 = C.c_double()
        N.check(N.lib().tm_strip_search_begin(
            self.ctx.h, prep, self.img.h, self._t.ctypes.data_as(C.POINTER(C.c_double)),
            C.byref(p), rank, world, C.byref(T0)))
        return T0.value

    def fused_begin(self, t, rank, world, policy, init_threshold, pred, seed_margin):
        from .api import make_params
        if self.strip_local and pred + 2 > self.hold:  # the batch's largest candidate
            self.rank, self.world = rank, world
            self._extend(pred + 2)
        self._t = np.ascontiguousarray(t, dtype=np.float64)
        p = make_params(policy=policy, init_threshold=init_threshold, seed_margin=seed_margin,
                        parallel=True, threads=2)
        ok, T0 = C.c_int(), C.c_double()
        N.check(N.lib().tm_strip_fused_begin(
            self.ctx.h, self.img.h, self._t.ctypes.data_as(C.POINTER(C.c_double)),
            self._t.shape[0], self._t.shape[1], C.byref(p), rank, world, pred, C.byref(ok),
            C.byref(T0)))
        return bool(ok.value), T0.value

    def fused_seed(self, T):
        T1 = C.c_double()
        N.check(N.lib().tm_strip_fused_seed(self.ctx.h, C.c_double(T), C.byref(T1)))
        return T1.value

    def fused_egs(self, T):
        nc = C.c_int()
        hs = (C.c_int * 4)()
        nr = (C.c_int64 * 4)()
        N.check(N.lib().tm_strip_fused_egs(self.ctx.h, C.c_double(T), C.byref(nc), hs, nr))
        return [hs[k] for k in range(nc.value)], [nr[k] for k in range(nc.value)]

    def fused_finish(self):
        part = StripPart()
        N.check(N.lib().tm_strip_fused_finish(self.ctx.h, C.byref(part)))
        return {k: getattr(part, k) for k, _ in StripPart._fields_ if not k.startswith("_")}

    def search_seed(self, T):
        T1 = C.c_double()
        N.check(N.lib().tm_strip_search_seed(self.ctx.h, C.c_double(T), C.byref(T1)))
        return T1.value

    def search_finish(self, T):
        part = StripPart()
        N.check(N.lib().tm_strip_search_finish(self.ctx.h, C.c_double(T), C.byref(part)))
        return {k: getattr(part, k) for k, _ in StripPart._fields_ if not k.startswith("_")}

    def refine(self, t, row, col, d):
        return self.ctx.refine_localization(t, self.img, row, col, d)

    def close(self):
        for p in self._preps:
            if isinstance(p, C.c_void_p):
                N.lib().tm_prep_destroy(p)
            else:
                p.close()
        self._preps = []
