#!/usr/bin/env python3
"""Benchmark: ZNCC-equivalent search locations/s and ms/search (BASELINE.json metric).

Default workload: BASELINE config 5, the configuration the metric's 1/2/4/8-GPU sweep is
quoted on -- a 16384x16384 8-bit image (1/f^2 noise + piecewise-constant rectangles +
high-frequency texture, 265,331,521 extent locations) and one 96x96 template; seeded,
bit-deterministic synthetic data (paper_1407_3535_b200/workloads.py).  `--config C1..C4`
selects the others (C3/C4: one step = the whole template batch on one preparation).

One step = one full exhaustive-accuracy search: window statistics + EGS group sizing
(prepare_egs) + centre scan + transitive-bound elimination + survivor ZNCC + argmax
(run_egs) -- tm_search, one call.  Nothing is cached across steps.

  value    : extent locations x templates per second of device time (CUDA events on the
             library's stream), image resident in HBM, L2 flushed between steps (untimed).
  e2e      : the same metric through the public 8-bit API from pinned HOST images, copies
             inside the timed region: tm_search_stream_u8 over a stream of DISTINCT images
             (the workload and seeded circular shifts of it), wall clock.
  frozen   : the reference's own --parallel policy on the GPU (like-for-like with the
             reference arm); the headline uses the B200 seeded policy (same argmax).
  parity   : every step's result is checked against the reference's recorded result for
             this config (tests/golden/configs/<C>.json); the CPU-baseline sample is
             searched on the GPU too and must equal the reference's result field for field.
             A mismatch exits non-zero.

--impl reference: the reference's own CPU implementation (oracle/_ref, compiled from
/root/reference) on a bounded sample of the same workload (a strip of image rows around the
template's true location; prepare + run, frozen --parallel policy, all host threads).

Multi-GPU (torchrun, NCCL): the search is sharded as row strips of the group grid
(distributed.py): per-rank window statistics and R_co of its strip, global EGS / threshold /
argmax through NCCL collectives.  value = all extent locations / max-over-ranks device time.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ZNCC-equivalent search locations/sec"
UNIT = "locations/s"
GOLDEN_DIR = os.path.join(ROOT, "tests", "golden", "configs")
# CPU-baseline sample: extent rows of a strip around the first template's cut location
SAMPLE_ROWS = {"C1": None, "C2": None, "C3": 160, "C4": 384, "C5": 512, "C6": 256}


def _json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


def peaks():
    """MEASURED_PEAKS.json (driver: HBM copy, cuBLAS bf16) + profiles/peaks_b200.json (this
    repo's tools/peaks: tcgen05 kind::i8 / kind::tf32, FFMA, DP4A)."""
    out = dict(_json(os.path.join(ROOT, "MEASURED_PEAKS.json")) or {})
    ours = _json(os.path.join(ROOT, "profiles", "peaks_b200.json")) or {}
    for k in ("i8_tops", "tf32_tflops", "ffma_tflops", "dp4a_tops"):
        if k in ours:
            out[k] = ours[k]
    return out


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region.

    In-process NVML polling every 2 ms (the timed region of a default run is only tens of
    ms); nvidia-smi ``-lms 20`` when NVML is unavailable.  ``start()`` returns once the
    first sample is in, so the samples cover the timed steps.
    """

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.nvml = None
        self.lines = []
        self.sm, self.smax, self.reasons = [], None, set()
        self.running = False

    def start(self):
        try:
            import pynvml as N
            N.nvmlInit()
            dev = N.nvmlDeviceGetHandleByIndex(self.index)
            self.smax = float(N.nvmlDeviceGetMaxClockInfo(dev, N.NVML_CLOCK_SM))
            self.nvml = (N, dev)
            self.running = True
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            while not self.sm and self.t.is_alive():
                time.sleep(0.001)
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5:
                time.sleep(0.005)
        except Exception:
            self.proc = None

    def _poll(self):
        N, dev = self.nvml
        bits = [N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
                N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap]
        while self.running:
            try:
                self.sm.append(float(N.nvmlDeviceGetClockInfo(dev, N.NVML_CLOCK_SM)))
                r = N.nvmlDeviceGetCurrentClocksEventReasons(dev)
                for nm, b in zip(self.NAMES, bits):
                    if r & b:
                        self.reasons.add(nm)
            except Exception:
                return
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.nvml:
            self.running = False
            self.t.join(timeout=1)
            sm = list(self.sm)
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.smax,
                    "reasons": sorted(self.reasons), "samples": len(sm), "source": "nvml"}
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi"}



# Functional check of the multi-rank path on a one-GPU box (never for numbers): every rank
# on cuda:0, collectives over gloo.  The strip kernels never wait on each other.
DIST_BACKEND = os.environ.get("BENCH_DIST_BACKEND", "nccl")


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if DIST_BACKEND != "nccl":
        local = 0
    return ws, rank, local


def coll_device(local):
    import torch
    return torch.device(f"cuda:{local}") if DIST_BACKEND == "nccl" else torch.device("cpu")


def golden(name):
    return _json(os.path.join(GOLDEN_DIR, f"{name}.json"))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def fail(msg):
    print(f"bench.py: PARITY FAILURE: {msg}", file=sys.stderr, flush=True)
    sys.exit(3)


def res_fields(r):
    return {k: getattr(r, k) for k in ("best_row", "best_col", "best_rho", "best_degenerate",
                                        "refined_row", "refined_col", "refined_rho",
                                        "final_threshold", "centers", "eliminated", "retained",
                                        "ops")}


def check_against_golden(name, results, policy):
    """Full-size results vs the reference's recorded results for this config."""
    g = golden(name)
    if not g:
        return {"checked": False, "why": "no golden for this config"}
    key = next(k for k in g if k.endswith("_frozen") and k.split("_")[0] == g["mode"])
    want = g[key]["results"]
    keys = ["best_row", "best_col", "best_rho", "refined_row", "refined_col", "refined_rho"]
    if policy == "frozen":
        keys += ["final_threshold", "centers", "eliminated", "retained", "ops"]
    for k, r in enumerate(results):
        got = res_fields(r)
        for f in keys:
            w = want[k][f]
            w = float.fromhex(w) if isinstance(w, str) else w
            if got[f] != w:
                fail(f"{name} template {k} {policy}: {f} = {got[f]!r}, reference {w!r}")
    return {"checked": True, "against": f"tests/golden/configs/{name}.json {key} (reference "
            f"library)", "templates": len(results), "fields": keys}


def sample_of(wl):
    """Bounded CPU-baseline sample: a strip of image rows around the first template's cut
    location (whole image for C1/C2)."""
    rows = SAMPLE_ROWS.get(wl.name)
    m, n = wl.templates[0].pixels.shape
    p = wl.image.shape[0]
    if rows is None or rows + m - 1 >= p:
        return wl.image, 0
    R = rows + m - 1
    r0 = max(0, min(wl.templates[0].row - rows // 2, p - R))
    return np.ascontiguousarray(wl.image[r0:r0 + R]), r0


def reference_sample(wl, threads=None):
    """The reference (oracle/_ref) on the bounded sample: prepare once + run every template,
    frozen --parallel policy on `threads` host threads (prepare_* is single-threaded in the
    reference)."""
    from oracle import binding as ob
    threads = threads or os.cpu_count()
    img, r0 = sample_of(wl)
    tm = [t.pixels.astype(np.float64) for t in wl.templates]
    m, n = tm[0].shape
    E = (img.shape[0] - m + 1) * (img.shape[1] - n + 1)
    kind = "reference" if ob.available("ref") else "port"
    lib = ob.Oracle("ref" if kind == "reference" else "port", autobuild=False)
    t0 = time.perf_counter()
    if kind == "reference":
        res, info, prep_ms, run_ms = lib.prepare_run_batch(tm, img.astype(np.float64),
                                                           mode=wl.mode, parallel=True,
                                                           threads=threads)
    else:  # the C restatement: one match per template (single-threaded)
        res = [lib.match(t, img.astype(np.float64), mode=wl.mode, parallel=True, threads=2)
               for t in tm]
        threads, prep_ms, run_ms = 1, float("nan"), []
    wall = time.perf_counter() - t0
    units = E * len(tm)
    return {"value": units / wall, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{wl.name} rows [{r0}, {r0 + img.shape[0]}) x all {img.shape[1]} "
                      f"columns ({E} extent locations x {len(tm)} template(s) = {units}; "
                      f"prepare_{wl.mode} {prep_ms:.0f} ms single-threaded + run_{wl.mode} "
                      f"frozen --parallel on {threads} threads)",
            "ms_per_step": wall * 1e3, "results": res, "image": img, "r0": r0}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from paper_1407_3535_b200 import workloads as W
    wl = W.make(args.config)
    per, steps_done, warm_done = [], 0, 0
    t_start = time.perf_counter()
    cb = None
    # bounded: warm-up and timed steps share one time budget; at least one timed step
    while warm_done < args.warmup and time.perf_counter() - t_start < args.reference_budget_s / 3:
        reference_sample(wl)
        warm_done += 1
    while steps_done < args.steps:
        cb = reference_sample(wl)
        per.append(cb["ms_per_step"])
        steps_done += 1
        if time.perf_counter() - t_start > args.reference_budget_s:
            break
    ms = statistics.mean(per)
    value = cb["value"] if len(per) == 1 else (cb["value"] * cb["ms_per_step"] / ms)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": steps_done, "warmup": warm_done,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded 1/f^beta, SURVEY 8d)",
            "config": {"workload": f"{wl.name}: {wl.description}", "extent": wl.extent,
                       "templates": len(wl.templates), "mode": wl.mode,
                       "policy": "reference frozen (--parallel)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cb["cores"],
                             "kind": cb["kind"], "sample": cb["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    if steps_done < args.steps or warm_done < args.warmup:
        line["note"] = (f"bounded by a {args.reference_budget_s:.0f} s budget: {warm_done} of "
                        f"{args.warmup} warm-up and {steps_done} of {args.steps} timed steps")
    print(json.dumps(line), flush=True)
    return 0


# ---- roofline -----------------------------------------------------------------------------
def roofline(phases, wl, res, pk, fp64_search=False):
    """Per-phase achieved vs peak; the dominant phase (largest device time) is the headline
    roofline.  Algorithmic amounts per launch group:
      window_stats   p*q + 17 B per extent location (u8 read; mu, omega, flat written)
      autocorr_sec   p*q + 18 B per location + 18 B per group (fused R_co + scan 2; h = 3:
                     k_rco3_s cross sums + k_rco_epi epilogue, whose u32 S round trip of
                     8 B per location is implementation traffic, not algorithmic)
      autocorr_u8    p*q + 25 B per location (R_co map written)
      autocorr_count p*q + 17 B per location (count-only EGS candidate, stops early)
      sec_compact    10 B per location (map 8 + flat 1 + visit 1)
      centre_scan    2*m*n ops per group centre (tcgen05 kind::i8); x 3 planes on a
                     non-integer search image (split variant)
    """
    p, q = wl.image.shape
    m, n = wl.templates[0].pixels.shape
    E = (p - m + 1) * (q - n + 1)
    G = res.centers
    hbm = pk.get("hbm_gbs", 6542.7)
    i8 = pk.get("i8_tops")
    total = max(sum(v["ms"] for v in phases.values()), 1e-9)
    defs = {
        "window_stats": ("hbm", p * q + 17.0 * E, "k_wstats4 (window statistics)"),
        "autocorr_sec": ("hbm", p * q + 18.0 * E + 18.0 * G,
                         "k_rco3_s + k_rco_epi<2> (h = 3; k_acg<h,...,FUSE=1> for h = 5): R_co "
                         "of the accepted EGS size with scan 2 fused (retained count + bound "
                         "test + survivor list)"),
        "autocorr_u8": ("hbm", p * q + 25.0 * E, "k_acg / k_acf (R_co map of one EGS size)"),
        "autocorr_count": ("hbm", p * q + 17.0 * E,
                           "k_acg count-only EGS candidate (stops at the EGS rejection point)"),
        "sec_compact": ("hbm", 10.0 * E, "k_sec_rows (scan-2 bound test + compaction)"),
        "centre_scan": ("tensor", 2.0 * m * n * G,
                        "k_tc_build_b + k_tc_corr<1> + k_centre_epi (tcgen05 kind::i8)"),
    }
    if fp64_search:
        # OptA with kappa > 0: the search image is non-integer.  Scan 1 runs on the three
        # byte planes of the split tensor-core variant (DESIGN 4.3a: 3 x 2*m*n integer ops
        # per centre, the exact FP64 replays of undecided centres included in the phase);
        # the window statistics are FP64 replica kernels (no u8 roofline).
        defs["centre_scan"] = ("tensor", 3 * 2.0 * m * n * G,
                               "k_tc_build_b + k_tc_corr<4> + k_split_centre_epi + k_split_pick "
                               "+ k_list_f64 (tcgen05 kind::i8 on three byte planes, bracketed "
                               "rho_c, exact replay of the undecided centres)")
        defs.pop("window_stats")
    rows = []
    for name, v in phases.items():
        per_launch = v["ms"] / max(v["count"], 1)
        row = {"phase": name, "kernel_ms": v["ms"], "launches": v["count"],
               "share_of_step": v["ms"] / total}
        if name in defs:
            bound, amount, kern = defs[name]
            row["kernel"] = kern
            row["bound"] = bound
            if bound == "hbm":
                row.update(achieved=amount / (per_launch / 1e3) / 1e9, peak=hbm, unit="GB/s",
                           algorithmic_per_launch=amount)
            elif i8:
                row.update(achieved=amount / (per_launch / 1e3) / 1e12, peak=i8, unit="TOP/s",
                           algorithmic_per_launch=amount)
            if "achieved" in row:
                row["frac"] = row["achieved"] / row["peak"]
        rows.append(row)
    rows.sort(key=lambda r: -r["kernel_ms"])
    head = next((r for r in rows if "frac" in r), None)
    return head, rows


def profiled_phases(ctx, step, nprof, flush, stream):
    import torch
    ctx.set_profiling(True)
    base = ctx.phase_times()
    for _ in range(nprof):
        with torch.cuda.stream(stream):
            flush.zero_()
        torch.cuda.synchronize()
        step()
    after = ctx.phase_times()
    ctx.set_profiling(False)
    out = {}
    for k, v in after.items():
        b = base.get(k, {"count": 0, "ms": 0.0})
        if v["ms"] - b["ms"] > 0:
            out[k] = {"count": (v["count"] - b["count"]) / nprof, "ms": (v["ms"] - b["ms"]) / nprof}
    return out


def variants(wl, k):
    """k distinct images for the e2e stream: the workload, then seeded circular shifts of it
    (different bytes, true locations and group alignments; each still contains the target,
    so the searches are of the workload's kind -- a mirrored image has no match and is a
    different, weak-elimination workload)."""
    rng = np.random.default_rng(4242)
    out = [wl.image]
    while len(out) < k:
        out.append(np.ascontiguousarray(np.roll(
            wl.image, (int(rng.integers(1, wl.image.shape[0])),
                       int(rng.integers(1, wl.image.shape[1]))), axis=(0, 1))))
    return out


def run_b200(args):
    import torch

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        if DIST_BACKEND == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(DIST_BACKEND)
    torch.cuda.set_device(local)
    from paper_1407_3535_b200 import api, workloads as W

    t_gen = time.perf_counter()
    wl = broadcast_workload(args.config, rank, local) if ws > 1 else W.make(args.config)
    gen_s = time.perf_counter() - t_gen
    g = golden(args.config)
    if g and wl.sha256() != g["sha256"]:
        fail(f"{args.config} inputs differ from the reference's (generator drift)")
    if ws > 1:
        return run_strips(args, wl, ws, rank, local)
    tm = [t.pixels for t in wl.templates]
    batch = np.ascontiguousarray(np.stack(tm))
    m, n = tm[0].shape
    single = len(tm) == 1 and wl.mode == "egs"
    ctx = api.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr, device=torch.device(f"cuda:{local}"))
    img = ctx.image(wl.image)  # resident in HBM for the device-timed value
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")

    def step(policy=args.policy, image=img):
        """One full search: window statistics, EGS, scans, survivors, argmax."""
        image.reset_cache()  # nothing cached across steps
        kw = dict(policy=policy, parallel=policy == "frozen", threads=2)
        if single:
            return [ctx.search(image, tm[0], mode="egs", **kw)]
        prep = ctx.prepare(image, m, n, mode=wl.mode)
        try:
            return ctx.run(prep, batch, **kw)
        finally:
            prep.close()

    def timed(policy, steps):
        times, res = [], None
        for _ in range(steps):
            with torch.cuda.stream(stream):
                flush.zero_()  # L2 flush (512 MB > 126 MB L2), outside the timed span
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record(stream)
            res = step(policy)
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        return times, res

    for _ in range(args.warmup):
        step()
    ctx.synchronize()
    # ---- timed region ------------------------------------------------------------------
    launches0 = ctx.launches
    clocks = ClockSampler(local)
    clocks.start()
    times, res = timed(args.policy, args.steps)
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = (ctx.launches - launches0) / args.steps
    ms = statistics.mean(times)
    units = wl.extent * len(tm)
    value = units / (ms / 1e3)
    parity = check_against_golden(args.config, res, args.policy)

    # ---- the reference's frozen policy on the GPU (like-for-like with the reference arm)
    nf = max(1, min(args.steps, 5))
    ftimes, fres = timed("frozen", nf)
    fparity = check_against_golden(args.config, fres, "frozen")
    frozen = {"value": units / (statistics.mean(ftimes) / 1e3), "unit": UNIT,
              "ms_per_step": statistics.mean(ftimes), "steps": nf,
              "eliminated": sum(r.eliminated for r in fres),
              "retained": sum(r.retained for r in fres),
              "elim_pct": statistics.mean(r.elim_pct for r in fres),
              "parity": fparity}

    # preparation details (h_e, kappa) from one untimed prepare
    prep = ctx.prepare(img, m, n, mode=wl.mode)
    info = prep.info
    prep.close()

    phases = profiled_phases(ctx, step, max(3, min(args.steps, 10)), flush, stream)

    # ---- e2e: distinct pinned host images through the public 8-bit API -------------------
    nvar = 3 if wl.image.size >= (1 << 26) else 4
    host = []
    for a in variants(wl, nvar):
        hb = torch.empty(a.shape, dtype=torch.uint8, pin_memory=True)
        hb.numpy()[:] = a
        host.append(hb)
    seq = [host[i % nvar].numpy() for i in range(args.steps)]
    s0 = ctx.search_stats()
    if single:
        ctx.search_stream(seq[:max(2, min(args.warmup, nvar))], tm[0], mode="egs",
                          policy=args.policy)
        with torch.cuda.stream(stream):
            flush.zero_()
        torch.cuda.synchronize()
        s0 = ctx.search_stats()
        t0 = time.perf_counter()
        rs = ctx.search_stream(seq, tm[0], mode="egs", policy=args.policy)
        e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
        e2e_path = ("tm_search_stream_u8 over K distinct pinned u8 host images: per image H2D "
                    "copy (overlapped with the previous search on a copy stream) + prepare_egs "
                    "+ run_egs + the result read on the host; wall clock of the K-image call / K")
    else:
        img_e2e = ctx.image(np.zeros(wl.image.shape, np.uint8))

        def e2e_step(hb):
            img_e2e.upload_u8(hb)
            prep = ctx.prepare(img_e2e, m, n, mode=wl.mode)
            try:
                return ctx.run(prep, batch, policy=args.policy)
            finally:
                prep.close()
        e2e_step(seq[0])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rs = [e2e_step(hb) for hb in seq]
        e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
        e2e_path = ("per step: tm_image_upload_u8 of a distinct pinned u8 host image + "
                    "tm_prepare + tm_run_u8 of the template batch + results on the host; wall "
                    "clock")
    s1 = ctx.search_stats()
    # the stream's result for the unmodified workload image equals the resident search
    if single and (rs[0].best_row, rs[0].best_col, rs[0].best_rho) != \
            (res[0].best_row, res[0].best_col, res[0].best_rho):
        fail("e2e stream result for the workload image differs from the resident search")

    # ---- CPU baseline: the reference on a bounded sample; the GPU must agree on it --------
    cpu = None
    sample_parity = None
    if not args.no_cpu_baseline:
        try:
            cb = reference_sample(wl)
        except Exception as e:  # the oracle library may be absent on a foreign box
            cb = None
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "port",
                   "sample": f"unavailable: {e}"}
        if cb:
            cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
            simg = ctx.image(cb["image"])
            sp = ctx.prepare(simg, m, n, mode=wl.mode)
            gres = ctx.run(sp, batch, policy="frozen", parallel=True, threads=2)
            sp.close()
            simg.close()
            for k, (a, b) in enumerate(zip(gres, cb["results"])):
                ga, gb = res_fields(a), {f: getattr(b, f) for f in res_fields(a)}
                bad = {f: (ga[f], gb[f]) for f in ga if ga[f] != gb[f]}
                if bad:
                    fail(f"CPU-baseline sample, template {k}: GPU vs reference {bad}")
            sample_parity = {"checked": True, "templates": len(gres),
                             "fields": sorted(res_fields(gres[0]))}
    pk = peaks()
    head, rows = roofline(phases, wl, res[0], pk,
                          fp64_search=wl.mode == "opta" and info["kappa"] > 0)
    traffic = None
    tr = _json(os.path.join(ROOT, "profiles", "r02_kernel_traffic.json")) or {}
    if head and head.get("phase") in tr.get("phases", {}):
        traffic = tr["phases"][head["phase"]]
    roof = None
    if head:
        roof = {"bound": head["bound"], "kernel": head["kernel"], "phase": head["phase"],
                "achieved": head["achieved"], "peak": head["peak"], "unit": head["unit"],
                "frac": head["frac"], "traffic": traffic,
                "traffic_source": "profiles/r02_kernel_traffic.json (ncu --set full: dram "
                                  "bytes read + written per launch)" if traffic else None,
                "algorithmic_bytes_per_launch": head.get("algorithmic_per_launch"),
                "kernel_ms": head["kernel_ms"] / max(head["launches"], 1),
                "share_of_step": head["share_of_step"],
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)"
                if head["bound"] == "hbm" else "profiles/peaks_b200.json i8_tops (measured, "
                "tools/peaks)",
                "phases": rows}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        # spread of the K timed steps (value uses the mean, as the contract says)
        "ms_per_step_min": min(times), "ms_per_step_median": statistics.median(times),
        "ms_per_step_max": max(times),
        "vs_baseline": None,
        "dtype": "u8 (s32 tensor-core dots, u32 window / cross sums), f64 epilogues",
        "data": "synthetic (seeded bit-deterministic 1/f^beta generator, SURVEY 8d)",
        "config": {"workload": f"{wl.name}: {wl.description}", "extent": wl.extent,
                   "templates": len(tm), "mode": wl.mode, "policy": args.policy,
                   "l2": "flushed between steps (512 MB write, untimed); inputs > L2"
                         if wl.image.size > (126 << 20) else
                         "flushed between steps (512 MB write, untimed)",
                   "parallelism": "single GPU", "generate_s": gen_s},
        "result": [{"best_row": r.best_row, "best_col": r.best_col, "best_rho": r.best_rho,
                    "refined_row": r.refined_row, "refined_col": r.refined_col,
                    "elim_pct": r.elim_pct, "eliminated": r.eliminated, "retained": r.retained,
                    "centers": r.centers, "ops": r.ops} for r in res[:4]],
        "h_e": info["h"], "kappa": info["kappa"],
        # non-integer search images (OptA, kappa > 0): centres / locations bracketed on the
        # tensor cores by the split-plane variant since the context was created
        "split_planes": ctx.split_stats(),
        "elimination_pct": statistics.mean(r.elim_pct for r in res),
        "parity": {"full_size_vs_reference": parity, "cpu_sample_vs_reference": sample_parity},
        "frozen": frozen,
        "phases_ms_per_step": {k: v["ms"] for k, v in phases.items()},
        "gpu_launches": launches,
        "e2e": {"value": units / (e2e_ms / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": int(wl.image.size + batch.size),
                "d2h_bytes_per_step": 112 * len(tm), "ms_per_step": e2e_ms, "path": e2e_path,
                "distinct_images": nvar,
                "h_e_prediction": {"hits": s1["fused_hits"] - s0["fused_hits"],
                                   "misses": s1["fused_misses"] - s0["fused_misses"]}},
        "roofline": roof,
        "cpu_baseline": cpu,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    return 0


def broadcast_workload(name, rank, local):
    """Rank 0 generates the workload, every rank receives it over NCCL (generating C5 on
    every rank at once would take minutes of host time)."""
    import torch
    import torch.distributed as dist
    from paper_1407_3535_b200 import workloads as W
    wl = W.make(name) if rank == 0 else None
    meta = [None]
    if rank == 0:
        meta = [dict(name=wl.name, mode=wl.mode, description=wl.description,
                     shape=wl.image.shape,
                     templates=[(t.row, t.col, t.gain, t.offset, t.noise_sigma,
                                 t.pixels.shape) for t in wl.templates])]
    dist.broadcast_object_list(meta, src=0)
    meta = meta[0]
    dev = coll_device(local)
    img = torch.empty(meta["shape"], dtype=torch.uint8, device=dev)
    k = len(meta["templates"])
    m, n = meta["templates"][0][5]
    tm = torch.empty((k, m, n), dtype=torch.uint8, device=dev)
    if rank == 0:
        img.copy_(torch.from_numpy(wl.image))
        tm.copy_(torch.from_numpy(np.stack([t.pixels for t in wl.templates])))
    dist.broadcast(img, src=0)
    dist.broadcast(tm, src=0)
    if rank != 0:
        ts = [W.Template(tm[i].cpu().numpy(), *meta["templates"][i][:5]) for i in range(k)]
        wl = W.Workload(meta["name"], img.cpu().numpy(), ts, meta["mode"], (1,),
                        meta["description"])
    return wl


def run_strips(args, wl, ws, rank, local):
    """N > 1: the search sharded as row strips of the group grid (distributed.py) over NCCL:
    each rank holds and computes only its strip (+ halo) of the image, statistics and R_co;
    the noise floor, EGS counts, thresholds and best cells are exchanged by collectives."""
    import torch
    import torch.distributed as dist
    from paper_1407_3535_b200 import api, distributed as D
    ctx = api.Context(local)
    dev = torch.device(f"cuda:{local}")
    stream = torch.cuda.ExternalStream(ctx.stream_ptr, device=dev)
    comm = D.Comm(device=coll_device(local))
    m, n = wl.templates[0].pixels.shape
    strip = wl.mode == "egs"
    backend = D.DeviceBackend.strip(ctx, wl.image, m, n, rank, ws) if strip else \
        D.DeviceBackend(ctx, wl.image)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        backend.reset()
        return [D.match_strips(backend, comm, t.pixels, wl.image.shape, mode=wl.mode,
                               policy=args.policy) for t in wl.templates]

    def timed(steps, fn):
        times, res = [], None
        for _ in range(steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            res = fn()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        t = torch.tensor([statistics.mean(times)], device=coll_device(local))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)  # device time, max over ranks
        return float(t.item()), res

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = ctx.launches
    ms, res = timed(args.steps, step)
    launches = (ctx.launches - launches0) / args.steps
    clk = clocks.stop()
    parity = check_against_golden(args.config, res, args.policy)

    # e2e: every step uploads the rank's rows of a distinct pinned host image (H2D inside
    # the timed region), recomputes the noise floor (allreduce) and searches
    lo, hi = backend.rows if strip else (0, wl.image.shape[0])
    host = []  # pinned copies of just this rank's rows of each distinct image
    for a in variants(wl, 3):
        hb = torch.empty((hi - lo, a.shape[1]), dtype=torch.uint8, pin_memory=True)
        hb.numpy()[:] = a[lo:hi]
        host.append(hb.numpy())
    ctr = [0]

    def e2e_step():
        rows = host[ctr[0] % len(host)]
        ctr[0] += 1
        if strip:
            backend.upload_rows(rows)
        else:
            backend.upload(rows)
        return step()
    e2e_step()
    e2e_ms, _ = timed(args.steps, e2e_step)
    rows = backend.rows if strip else (0, wl.image.shape[0])
    dist.barrier()
    if rank == 0:
        units = wl.extent * len(wl.templates)
        line = {"metric": METRIC, "value": units / (ms / 1e3), "unit": UNIT, "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "u8 (s32 tensor-core dots, u32 window / cross sums), f64 epilogues",
                "data": "synthetic (seeded bit-deterministic 1/f^beta generator, SURVEY 8d)",
                "config": {"workload": f"{wl.name}: {wl.description}", "extent": wl.extent,
                           "templates": len(wl.templates), "mode": wl.mode,
                           "policy": args.policy,
                           "parallelism": f"row strips x{ws} (NCCL collectives: noise-floor "
                                          "sum, EGS counts, thresholds, best cells)",
                           "rank0_image_rows": list(rows),
                           "l2": "flushed between steps (512 MB write, untimed)"},
                "result": [r.as_dict() for r in res[:4]],
                "elimination_pct": statistics.mean(r.elim_pct for r in res),
                "parity": {"full_size_vs_reference": parity},
                "gpu_launches": launches,
                "e2e": {"value": units / (e2e_ms / 1e3), "unit": UNIT,
                        "h2d_bytes_per_step": int((rows[1] - rows[0]) * wl.image.shape[1]),
                        "d2h_bytes_per_step": 64 * len(wl.templates),
                        "ms_per_step": e2e_ms,
                        "path": "per rank: tm_image_upload_strip_u8 of its rows of a distinct "
                                "pinned host image + the strip search; device time, max over "
                                "ranks (h2d bytes: rank 0's rows)"},
                "clocks": clk}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C5", choices=["C1", "C2", "C3", "C4", "C5", "C6"])
    ap.add_argument("--policy", default="seeded", choices=["seeded", "frozen"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--reference-budget-s", type=float, default=150.0)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    args.warmup = max(args.warmup, 3)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
