"""Row-strip sharding (paper_1407_3535_b200/distributed.py) over torch.distributed.

CPU: the orchestration (EGS n_r allreduce, threshold allreduce, seeded threshold, cell
merge, count sums) runs with world_size 2 and 3 over gloo against a NumPy backend built on
the oracle; the merged result must equal the reference's `--parallel` result exactly for
the frozen policy (groups are independent given the frozen threshold, matcher.cpp:129-143).
GPU: the same protocol with the CUDA backend (two processes sharing cuda:0 over gloo; the
kernels never wait on each other) must equal the single-GPU result.
"""
import math
import os
import socket
import sys
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _sec_holds(tb, a, b):  # bounds.cpp:21-23, 41-46 (numpy FP64, no contraction)
    a = np.clip(a, -1.0, 1.0)
    b = np.clip(b, -1.0, 1.0)
    tb = np.clip(tb, -1.0, 1.0)
    return tb >= a * b + np.sqrt(np.maximum(0.0, 1.0 - a * a)) * np.sqrt(np.maximum(0.0, 1.0 - b * b))


class NumpyBackend:
    """The tm_strip_* primitives restated over oracle results (test-only)."""

    def __init__(self, port, img):
        self.port, self.img = port, np.asarray(img, np.float64)
        self.slots = {}
        self.search_img = self.img

    def _grid(self, er, ec, h, w):
        return (er + h - 1) // h, (ec + w - 1) // w

    def autocorr(self, m, n, h, w, rank, world, rho_tb, slot):
        from paper_1407_3535_b200.distributed import strip_rows
        amap = self.port.local_autocorrelation(self.img, m, n, h, w)
        self.slots[slot] = amap
        er, ec = amap.shape
        tr, tc = self._grid(er, ec, h, w)
        lo, hi = strip_rows(tr, rank, world)
        thr = math.sqrt(max(0.0, 1.0 - rho_tb * rho_tb))
        cnt = 0
        for r in range(lo * h, min(hi * h, er)):
            ti = min(r // h, tr - 1)
            cr = (ti * h + min(ti * h + h, er) - 1) // 2
            for c in range(ec):
                tj = min(c // w, tc - 1)
                cc = (tj * w + min(tj * w + w, ec) - 1) // 2
                if (r, c) != (cr, cc) and amap[r, c] < thr:
                    cnt += 1
        return cnt

    def commit(self, m, n, slot, h, w, trace):
        return dict(map=self.slots[slot], h=h, w=w)

    def prepare_opta(self, m, n, kernel=None):
        o = self.port.optimize_autocorrelation(self.img, m, n)
        self.search_img = o["image"]
        return dict(map=o["map"], h=o["h"], w=o["w"]), o["kappa"], 2

    def search_begin(self, prep, t, rank, world, policy, init, margin):
        from paper_1407_3535_b200.distributed import strip_rows
        self.t = np.asarray(t, np.float64)
        m, n = self.t.shape
        b, self.surface = self.port.brute(self.t, self.search_img, surface=True)
        _, _, self.flat = self.port.window_stats(self.search_img, m, n)
        self.tflat = self.port.template_stats(self.t)[2]
        self.map, self.h, self.w = prep["map"], prep["h"], prep["w"]
        er, ec = self.surface.shape
        self.tr, self.tc = self._grid(er, ec, self.h, self.w)
        self.lo, self.hi = strip_rows(self.tr, rank, world)
        self.policy, self.margin, self.init = policy, margin, init
        self.cells = []
        T0 = -math.inf
        self.centre = {}
        for ti in range(self.lo, self.hi):
            r0, r1 = ti * self.h, min(ti * self.h + self.h, er) - 1
            for tj in range(self.tc):
                c0, c1 = tj * self.w, min(tj * self.w + self.w, ec) - 1
                cr, cc = (r0 + r1) // 2, (c0 + c1) // 2
                rho = self.surface[cr, cc]
                deg = bool(self.tflat or self.flat[cr, cc])
                self.centre[(ti, tj)] = (rho, deg, r0, r1, c0, c1, cr, cc)
                self.cells.append(dict(rho=rho, row=cr, col=cc, valid=True, degenerate=deg))
                if not deg:
                    T0 = max(T0, rho)
        if init is not None:
            T0 = max(T0, min(max(init, -1.0), 1.0))
        self.seeded = set()
        return T0

    def search_seed(self, T):
        T1 = T
        for (ti, tj), (rho, deg, r0, r1, c0, c1, cr, cc) in sorted(self.centre.items()):
            if deg or not (rho >= T - self.margin) or len(self.seeded) >= 256:
                continue
            self.seeded.add((ti, tj))
            for r in range(r0, r1 + 1):
                for c in range(c0, c1 + 1):
                    if (r, c) == (cr, cc):
                        continue
                    fl = bool(self.tflat or self.flat[r, c])
                    self.cells.append(dict(rho=self.surface[r, c], row=r, col=c, valid=True,
                                           degenerate=fl))
                    if not fl:
                        T1 = max(T1, self.surface[r, c])
        return T1

    def search_finish(self, T):
        from paper_1407_3535_b200.distributed import better
        elim = kept = 0
        fin = T
        for (ti, tj), (rho_tc, cdeg, r0, r1, c0, c1, cr, cc) in self.centre.items():
            for r in range(r0, r1 + 1):
                for c in range(c0, c1 + 1):
                    if (r, c) == (cr, cc):
                        continue
                    if (ti, tj) in self.seeded:
                        kept += 1
                        continue
                    fl = bool(self.tflat or self.flat[r, c])
                    if (not cdeg and not fl and T >= -1.0 and
                            _sec_holds(min(T, 1.0), rho_tc, self.map[r, c])):
                        elim += 1
                        continue
                    kept += 1
                    self.cells.append(dict(rho=self.surface[r, c], row=r, col=c, valid=True,
                                           degenerate=fl))
                    if not fl:
                        fin = max(fin, self.surface[r, c])
        best = dict(valid=False, degenerate=True, rho=0.0, row=-1, col=-1)
        for c in self.cells:
            if better(c, best):
                best = c
        return dict(best_rho=best["rho"], best_row=best["row"], best_col=best["col"],
                    best_flags=(1 if best["valid"] else 0) | (2 if best["degenerate"] else 0),
                    centers=len(self.centre), eliminated=elim, retained=kept,
                    final_threshold=fin)

    def refine(self, t, row, col, d):
        return self.port.refine(t, self.img, row, col, d)


class NumpyStripBackend(NumpyBackend):
    """Strip-LOCAL restatement (test-only): holds only rows strip_image_rows(...) of the
    image; window statistics of its strip use the allreduced global noise floor; R_co and
    the search see only the rank's group rows (the sub-image starting at its first group
    row, so the local group grid is the global one shifted)."""

    strip_local = True
    noise_set = False

    def __init__(self, port, img, m, n, rank, world):
        from paper_1407_3535_b200.distributed import strip_image_rows
        self.full = np.asarray(img, np.float64)  # (only read again by _extend)
        self.p, self.q = self.full.shape
        self.m, self.n, self.rank, self.world = m, n, rank, world
        self.hold = 15
        self.r0, self.r1 = strip_image_rows(self.p, self.q, m, n, rank, world)
        self.rows = self.full[self.r0:self.r1].copy()  # everything this rank sees
        super().__init__(port, self.rows)
        self.stat_rows = []  # extent rows whose statistics were computed (strip-locality)

    def _extend(self, h):
        from paper_1407_3535_b200.distributed import strip_image_rows
        self.r0, self.r1 = strip_image_rows(self.p, self.q, self.m, self.n, self.rank,
                                            self.world, 3, h)
        self.rows = self.full[self.r0:self.r1].copy()
        self.hold = h

    def sum_sq(self, a, b):
        assert self.r0 <= a and b <= self.r1
        return int(np.sum(self.rows[a - self.r0:b - self.r0].astype(np.int64) ** 2))

    def set_noise(self, q_total):
        self.floor = float(self.p + self.q) * 2.220446049250313e-16 * float(q_total)
        self.noise_set = True

    def _sub(self, a, b, m):
        """Image rows [a, b + m - 1) (extent rows [a, b)) from the held rows."""
        assert self.r0 <= a and b + m - 1 <= self.r1, (a, b, self.r0, self.r1)
        self.stat_rows.append((a, b))
        return self.rows[a - self.r0:b + m - 1 - self.r0]

    def _extent(self, m, h, rank, world):
        from paper_1407_3535_b200.distributed import strip_rows
        er = self.p - m + 1
        tr = (er + h - 1) // h
        lo, hi = strip_rows(tr, rank, world)
        return lo * h, min(hi * h, er)

    def autocorr(self, m, n, h, w, rank, world, rho_tb, slot):
        if max(h, w) > self.hold:
            self._extend(max(h, w))
        a, b = self._extent(m, h, rank, world)
        if b <= a:
            self.slots[slot] = (None, a, b)
            return 0
        sub = self._sub(a, b, m)
        ws = self.port.window_stats_floor(sub, m, n, self.floor)
        amap = self.port.local_autocorrelation(sub, m, n, h, w, ws=ws)
        self.slots[slot] = (amap, a, b)
        return int(self.port.retained_count(amap, h, w, rho_tb))

    def commit(self, m, n, slot, h, w, trace):
        amap, a, b = self.slots[slot]
        return dict(map=amap, a=a, b=b, h=h, w=w)

    def search_begin(self, prep, t, rank, world, policy, init, margin):
        self.t = np.asarray(t, np.float64)
        m, n = self.t.shape
        self.map, self.h, self.w = prep["map"], prep["h"], prep["w"]
        a, b = prep["a"], prep["b"]
        self.policy, self.margin, self.init = policy, margin, init
        self.cells, self.centre, self.seeded = [], {}, set()
        T0 = -math.inf
        if b <= a:
            return T0 if init is None else max(T0, min(max(init, -1.0), 1.0))
        sub = self._sub(a, b, m)
        _, _, self.flat = self.port.window_stats_floor(sub, m, n, self.floor)
        _, local = self.port.brute(self.t, sub, surface=True)
        # windows flat under the sub-image's own floor are flat under the (larger) global
        # floor too, so the global-floor surface is the local one with those set to 0
        self.surface = np.where(self.flat == 1, 0.0, local)
        self.tflat = self.port.template_stats(self.t)[2]
        er, ec = self.surface.shape
        tr, tc = self._grid(er, ec, self.h, self.w)
        for ti in range(tr):
            r0, r1 = ti * self.h, min(ti * self.h + self.h, er) - 1
            for tj in range(tc):
                c0, c1 = tj * self.w, min(tj * self.w + self.w, ec) - 1
                cr, cc = (r0 + r1) // 2, (c0 + c1) // 2
                rho = self.surface[cr, cc]
                deg = bool(self.tflat or self.flat[cr, cc])
                self.centre[(ti, tj)] = (rho, deg, r0, r1, c0, c1, cr, cc)
                self.cells.append(dict(rho=rho, row=a + cr, col=cc, valid=True, degenerate=deg))
                if not deg:
                    T0 = max(T0, rho)
        self.row_off = a
        if init is not None:
            T0 = max(T0, min(max(init, -1.0), 1.0))
        return T0

    def search_seed(self, T):
        T1 = NumpyBackend.search_seed(self, T)
        for c in self.cells[len(self.centre):]:
            c["row"] += self.row_off  # seeded members: local -> global rows
        self._n_fixed = len(self.cells)
        return T1

    def search_finish(self, T):
        n0 = getattr(self, "_n_fixed", len(self.centre))
        part = NumpyBackend.search_finish(self, T) if self.centre else dict(
            best_rho=0.0, best_row=-1, best_col=-1, best_flags=0, centers=0, eliminated=0,
            retained=0, final_threshold=T)
        if self.centre:  # survivors appended by search_finish are in local rows
            for c in self.cells[n0:]:
                c["row"] += self.row_off
            from paper_1407_3535_b200.distributed import better
            best = dict(valid=False, degenerate=True, rho=0.0, row=-1, col=-1)
            for c in self.cells:
                if better(c, best):
                    best = c
            part.update(best_rho=best["rho"], best_row=best["row"], best_col=best["col"],
                        best_flags=(1 if best["valid"] else 0) | (2 if best["degenerate"] else 0))
        self._n_fixed = None
        return part


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _case():
    rng = np.random.default_rng(11)
    base = np.cumsum(np.cumsum(rng.normal(size=(72, 66)), 0), 1)
    img = np.clip(np.rint((base - base.min()) / np.ptp(base) * 255), 0, 255)
    t = np.clip(np.rint(img[30:41, 20:33] * 0.9 + 6 + rng.normal(0, 2, (11, 13))), 0, 255)
    return img, t


def _worker(rank, world, port, out_path, backend_kind, mode, policy):
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    from paper_1407_3535_b200 import distributed as D
    img, t = _case()
    m, n = t.shape
    strip = mode == "egs"  # OptA keeps the whole image on every rank
    if backend_kind == "numpy":
        from oracle.binding import Oracle
        backend = NumpyStripBackend(Oracle("port"), img, m, n, rank, world) if strip else \
            NumpyBackend(Oracle("port"), img)
    else:
        from paper_1407_3535_b200 import api
        ctx = api.Context(0)
        backend = D.DeviceBackend.strip(ctx, img.astype(np.uint8), m, n, rank, world) \
            if strip else D.DeviceBackend(ctx, img)
    comm = D.Comm()
    res = D.match_strips(backend, comm, t, img.shape, mode=mode, policy=policy)
    if strip and world > 1:  # strip-local: this rank held and computed only its rows
        lo, hi = backend.rows if backend_kind == "cuda" else (backend.r0, backend.r1)
        assert hi - lo < img.shape[0], (lo, hi)
        if backend_kind == "numpy":
            assert all(backend.r0 <= a and b + m - 1 <= backend.r1 for a, b in backend.stat_rows)
    if rank == 0:
        np.save(out_path, np.array([res.best_row, res.best_col, res.best_rho, res.refined_row,
                                    res.refined_col, res.refined_rho, res.eliminated,
                                    res.retained, res.centers, res.ops, res.final_threshold]))
    dist.barrier()
    dist.destroy_process_group()


def _run(world, backend_kind, mode, policy):
    import torch.multiprocessing as mp
    out = os.path.join(tempfile.mkdtemp(), "res.npy")
    mp.spawn(_worker, args=(world, _free_port(), out, backend_kind, mode, policy), nprocs=world,
             join=True)
    return np.load(out)


def _reference(mode, policy):
    from oracle.binding import Oracle
    port = Oracle("port")
    img, t = _case()
    if policy == "frozen":
        r = port.match(t, img, mode=mode, parallel=True, threads=4)
    else:
        r = port.match(t, img, mode=mode, parallel=True, threads=4)
    return r


@pytest.mark.parametrize("world", [2, 3])
def test_strips_frozen_equal_reference_parallel_cpu(world):
    got = _run(world, "numpy", "egs", "frozen")
    want = _reference("egs", "frozen")
    assert (int(got[0]), int(got[1]), got[2]) == (want.best_row, want.best_col, want.best_rho)
    assert (int(got[6]), int(got[7]), int(got[8]), int(got[9])) == \
        (want.eliminated, want.retained, want.centers, want.ops)
    assert got[10] == want.final_threshold


def test_strips_seeded_same_argmax_cpu():
    from oracle.binding import Oracle
    img, t = _case()
    b = Oracle("port").brute(t, img)
    got = _run(2, "numpy", "egs", "seeded")
    assert (int(got[0]), int(got[1]), got[2]) == (b.best_row, b.best_col, b.best_rho)


def test_strips_opta_cpu():
    got = _run(2, "numpy", "opta", "frozen")
    want = _reference("opta", "frozen")
    assert (int(got[3]), int(got[4]), got[5]) == (want.refined_row, want.refined_col,
                                                  want.refined_rho)
    assert (int(got[6]), int(got[7])) == (want.eliminated, want.retained)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["egs", "opta"])
def test_strips_gpu_equal_single_gpu(mode):
    got = _run(2, "cuda", mode, "frozen")
    want = _reference(mode, "frozen")
    assert (int(got[3]), int(got[4]), got[5]) == (want.refined_row, want.refined_col,
                                                  want.refined_rho)
    assert (int(got[6]), int(got[7]), int(got[8])) == (want.eliminated, want.retained,
                                                       want.centers)


@pytest.mark.gpu
def test_strips_gpu_seeded():
    from oracle.binding import Oracle
    img, t = _case()
    b = Oracle("port").brute(t, img)
    got = _run(2, "cuda", "egs", "seeded")
    assert (int(got[0]), int(got[1]), got[2]) == (b.best_row, b.best_col, b.best_rho)
