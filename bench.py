#!/usr/bin/env python3
"""Benchmark: ZNCC-equivalent search locations/s and ms/search (BASELINE.json metric).

One step = one full exhaustive-accuracy search of one template through the B200 path:
window statistics + EGS group sizing (prepare_egs) + centre scan + transitive-bound
elimination + survivor ZNCC + argmax (run_egs), on BASELINE config 2 (2048x2048 1/f^1.8
image with half the tiles blurred, one 64x64 template; seeded synthetic data).

  value : extent locations per second of device time, image resident in HBM, L2 flushed
          between steps (the device-timed step excludes the flush).
  e2e   : the same metric through the public 8-bit API (pinned host image ->
          tm_image_upload_u8 -> tm_prepare -> tm_run_u8 -> result on the host), wall clock.

--impl reference times the reference's own CPU implementation (oracle/_ref, compiled from
/root/reference) on the same workload with all host threads.

Multi-GPU (torchrun): each rank searches its own seeded C2 replica (weak scaling); the
best cells are all-gathered over NCCL and merged in better_candidate order.
"""
from __future__ import annotations

import argparse
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


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


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


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_baseline(workload, threads=None, kind=None):
    """Reference CPU path on the same C2 search (prepare_egs + run_egs, frozen policy)."""
    from oracle import binding as ob
    threads = threads or os.cpu_count()
    t = workload.templates[0].pixels.astype(np.float64)
    img = workload.image.astype(np.float64)
    if kind in (None, "reference") and ob.available("ref"):
        ref = ob.Oracle("ref", autobuild=False)
        t0 = time.perf_counter()
        res, prep_ms, run_ms = ref.prepare_run_egs(t, img, parallel=True, threads=threads)
        wall = time.perf_counter() - t0
        return {"value": workload.extent / wall, "unit": UNIT, "cores": threads,
                "kind": "reference",
                "sample": f"1 full {workload.name} search (reference prepare_egs {prep_ms:.0f} ms "
                          f"1 thread + run_egs frozen policy {run_ms:.0f} ms on {threads} "
                          f"threads)", "ms_per_search": wall * 1e3,
                "best": [res.best_row, res.best_col, res.best_rho],
                "elim_pct": res.elim_pct}
    port = ob.Oracle("port")
    t0 = time.perf_counter()
    res = port.match(t, img, mode="egs", parallel=True, threads=2)
    wall = time.perf_counter() - t0
    return {"value": workload.extent / wall, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"1 full {workload.name} search (C restatement, frozen policy, 1 thread)",
            "ms_per_search": wall * 1e3, "best": [res.best_row, res.best_col, res.best_rho],
            "elim_pct": res.elim_pct}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from paper_1407_3535_b200 import workloads as W
    wl = W.make(args.config)
    # bounded: each step is one full reference search (~seconds); cap the run time
    per = []
    t_start = time.perf_counter()
    steps_done = 0
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(wl)
        if i >= args.warmup:
            per.append(cb["ms_per_search"])
            steps_done += 1
        if time.perf_counter() - t_start > args.reference_budget_s and steps_done >= 1:
            break
    ms = statistics.mean(per)
    value = wl.extent / (ms / 1e3)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": steps_done, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded 1/f^beta, SURVEY 8d)",
            "config": {"workload": f"{wl.name}: {wl.description}", "extent": wl.extent,
                       "templates": 1, "mode": "egs", "policy": "reference frozen (--parallel)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cb["cores"],
                             "kind": cb["kind"], "sample": cb["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    if steps_done < args.steps:
        line["note"] = f"bounded: {steps_done} of {args.steps} steps within the time budget"
    print(json.dumps(line), flush=True)
    return 0


def run_b200(args):
    import torch

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    from paper_1407_3535_b200 import api, workloads as W

    wl = W.make(args.config, seed=W.CONFIGS[args.config].__defaults__[0] + 1000 * rank) \
        if ws > 1 else W.make(args.config)
    tmpl = wl.templates[0].pixels
    m, n = tmpl.shape
    ctx = api.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr, device=torch.device(f"cuda:{local}"))
    img = ctx.image(wl.image)  # resident in HBM for the device-timed value
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")

    tmpl_u8 = np.ascontiguousarray(tmpl, dtype=np.uint8)

    def step():
        """One full search (tm_search_u8: prepare_egs + run_egs in one call)."""
        img.reset_cache()  # recompute window statistics: nothing cached across steps
        return ctx.search(img, tmpl_u8, mode="egs", policy=args.policy)

    for _ in range(args.warmup):
        step()
    ctx.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    # ---- timed region: profiling off (no per-call event timers or syncs) --------------
    launches0 = ctx.launches
    clocks = ClockSampler(local)
    clocks.start()
    times = []
    res = info = None
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()  # L2 flush (512 MB > 126 MB L2), outside the timed span
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
        res = step()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = (ctx.launches - launches0) / args.steps
    ms = statistics.mean(times)
    if ws > 1:
        t = torch.tensor([ms], device=f"cuda:{local}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        torch.distributed.barrier()
    value = ws * wl.extent / (ms / 1e3)

    # preparation details (h_e, EGS trace) from one untimed prepare on the same image
    prep = ctx.prepare(img, m, n, mode="egs")
    info = prep.info
    prep.close()

    # ---- per-phase device times: a separate, untimed profiled pass ---------------------
    ctx.set_profiling(True)
    base = ctx.phase_times()
    nprof = max(3, min(args.steps, 10))
    for _ in range(nprof):
        with torch.cuda.stream(stream):
            flush.zero_()
        torch.cuda.synchronize()
        step()
    after = ctx.phase_times()
    ctx.set_profiling(False)
    phases = {k: {"count": (v["count"] - base.get(k, {"count": 0})["count"]) / nprof,
                  "ms": (v["ms"] - base.get(k, {"ms": 0.0})["ms"]) / nprof}
              for k, v in after.items() if v["ms"] - base.get(k, {"ms": 0.0})["ms"] > 0}

    # ---- e2e through the public 8-bit API -------------------------------------------------
    # (1) throughput: tm_search_stream_u8 over K pinned host images (two pinned buffers,
    #     alternating; every step copies its image host->device and reads its result back),
    #     the next image's copy overlapped with the current search -> e2e value;
    # (2) latency: one tm_image_upload_u8 + tm_search_u8 call per step, L2 flushed before
    #     each (wall clock) -> e2e latency_ms.
    img_host = [torch.empty(wl.image.shape, dtype=torch.uint8, pin_memory=True)
                for _ in range(2)]
    for hb in img_host:
        hb.numpy()[:] = wl.image
    t_host = torch.empty(tmpl.shape, dtype=torch.uint8, pin_memory=True)
    t_host.numpy()[:] = tmpl
    img_e2e = ctx.image(np.zeros(wl.image.shape, np.uint8))
    stream_imgs = [img_host[i & 1].numpy() for i in range(args.steps)]

    def e2e_step():
        img_e2e.upload_u8(img_host[0].numpy())
        return ctx.search(img_e2e, t_host.numpy(), mode="egs", policy=args.policy)

    for _ in range(max(1, args.warmup)):
        e2e_step()
    ctx.search_stream(stream_imgs[:max(2, args.warmup)], t_host.numpy(), mode="egs",
                      policy=args.policy)
    lat_ms = []
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r2 = e2e_step()
        lat_ms.append((time.perf_counter() - t0) * 1e3)
    lat = statistics.mean(lat_ms)
    with torch.cuda.stream(stream):
        flush.zero_()
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    rs = ctx.search_stream(stream_imgs, t_host.numpy(), mode="egs", policy=args.policy)
    e2e = (time.perf_counter() - t0) * 1e3 / args.steps
    if ws > 1:
        t = torch.tensor([e2e, lat], device=f"cuda:{local}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e, lat = float(t[0].item()), float(t[1].item())
    for r3 in rs:
        assert (r3.best_row, r3.best_col, r3.best_rho) == (res.best_row, res.best_col,
                                                           res.best_rho)
    assert (r2.best_row, r2.best_col, r2.best_rho) == (res.best_row, res.best_col, res.best_rho)

    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel ---------------------------------------------
    # R_co of the EGS candidates is the dominant phase.  On the tm_search path the first
    # candidate (h0 = the predicted h_e, always accepted) is the group-column kernel with
    # scan 2 fused into its epilogue (k_acg<3,256,0,1>): it reads the 8-bit image once (p*q
    # bytes), the centre/member statistics (mu, omega, flat: 17 B per extent location) and
    # the scan-1 values of each group (rho_c, sa_c: 8 + 8 B, degenerate + seeded flags: 2 B)
    # and writes one visit code per location (1 B); the E-sized R_co map is never written.
    # (TMATCH_FUSE_SCAN2=0: the map-writing launch, p*q + 25 B per location.)  Later
    # candidates run count-only and stop at the EGS rejection point (data-dependent work):
    # they are reported beside it with their measured time.
    peaks = _peaks()
    p_, q_ = wl.image.shape
    E = wl.extent
    hbm_peak = peaks.get("hbm_gbs", 6534.1)
    ph_step = max(sum(v["ms"] for v in phases.values()), 1e-9)
    fused = "autocorr_sec" in phases
    ac = phases.get("autocorr_sec" if fused else "autocorr_u8", {"count": 1, "ms": float("nan")})
    ac_launch_ms = ac["ms"] / max(ac["count"], 1)
    G = res.centers
    if fused:
        ac_bytes = p_ * q_ + 18.0 * E + 18.0 * G
        ac_alg = (f"p*q + 18 B x {E} extent locations (17 B statistics read, 1 B visit code "
                  f"written) + 18 B x {G} groups (scan-1 rho, half-gap factor, flags)")
        ac_name = ("k_acg<3,256,0,1> (group-column fused R_co of the first EGS candidate with "
                   "scan 2 in its epilogue: retained count + bound test + survivor list)")
        ac_key = "k_acg<3, 256, 0, 1>"
    else:
        ac_bytes = p_ * q_ + 25.0 * E
        ac_alg = (f"p*q + 25 B x {E} extent locations (image, 17 B statistics read, 8 B map "
                  "write)")
        ac_name = "k_acg<3,256,0,0> (group-column fused R_co, first EGS candidate: full map)"
        ac_key = "k_acg<3, 256, 0, 0>"
    ac_gbs = ac_bytes / (ac_launch_ms / 1e3) / 1e9
    traffic = None  # DRAM read+write of that launch from the committed ncu --set full capture
    traffic_src = os.path.join("profiles", "r01_kernel_traffic.json")
    try:
        kt = json.load(open(os.path.join(ROOT, traffic_src)))["kernels"]
        hit = [v for k, v in kt.items() if ac_key in k]
        if hit:
            traffic = hit[0]["dram_read_bytes"] + hit[0]["dram_write_bytes"]
    except Exception:
        traffic = None
    roofline = {"bound": "hbm", "kernel": ac_name,
                "achieved": ac_gbs, "peak": hbm_peak, "unit": "GB/s", "frac": ac_gbs / hbm_peak,
                "traffic": traffic, "traffic_unit": f"bytes per launch ({traffic_src})",
                "algorithmic_bytes_per_launch": ac_bytes,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)",
                "algorithmic": ac_alg,
                "kernel_ms": ac_launch_ms, "share_of_step": ac["ms"] / ph_step}
    sec = []
    cnt = phases.get("autocorr_count")
    if cnt:
        sec.append({"bound": "issue", "kernel": "k_acg<5,128,2,0> count-only EGS candidate, packed dp4a walk "
                    "(stops when the partial retained count rejects the size)",
                    "kernel_ms": cnt["ms"], "share_of_step": cnt["ms"] / ph_step})
    wsp = phases.get("window_stats")
    if wsp:
        ws_bytes = p_ * q_ + 17.0 * E
        ws_gbs = ws_bytes / (wsp["ms"] / 1e3) / 1e9
        sec.append({"bound": "hbm", "kernel": "k_wstats4<256,2> (window statistics)",
                    "achieved": ws_gbs, "peak": hbm_peak, "unit": "GB/s",
                    "frac": ws_gbs / hbm_peak, "algorithmic": f"p*q + 17 B x {E} locations",
                    "kernel_ms": wsp["ms"], "share_of_step": wsp["ms"] / ph_step})
    # the tensor-core centre scan (tcgen05 kind::i8), useful ops only
    G = res.centers
    cs = phases.get("centre_scan", {"count": 1, "ms": float("nan")})
    i8_peak = 2.0 * peaks.get("bf16_tflops", 1649.1)
    cs_tops = 2.0 * m * n * G / (cs["ms"] / 1e3) / 1e12
    sec.append({
        "bound": "tensor", "kernel": "k_tc_build_b + k_tc_corr<1> + k_centre_epi (centre scan, "
                                     "tcgen05 kind::i8)",
        "achieved": cs_tops, "peak": i8_peak, "unit": "TOP/s", "frac": cs_tops / i8_peak,
        "peak_source": "2 x MEASURED_PEAKS.json bf16_tflops (i8 MMA: K=32 per instruction "
                       "vs K=16 for bf16 at the same issue rate)",
        "algorithmic": f"2*m*n useful ops per centre x {G} centres (phase time incl. B build "
                       "and FP64 epilogue)", "kernel_ms": cs["ms"]})
    roofline["secondary"] = sec

    cpu = None
    if not args.no_cpu_baseline:
        try:
            cb = cpu_baseline(wl)
            cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as e:  # the oracle may be absent on a foreign box
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "port",
                   "sample": f"unavailable: {e}"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u8 (s32 tensor-core / exact-FP32 dots, u32 window sums), f64 epilogues",
        "data": "synthetic (seeded 1/f^beta generator, SURVEY 8d; BASELINE config 2)",
        "config": {"workload": f"{wl.name}: {wl.description}", "extent": wl.extent,
                   "templates": 1, "mode": "egs", "policy": args.policy,
                   "l2": "flushed between steps (512 MB write, untimed)",
                   "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU"},
        "result": {"best_row": res.best_row, "best_col": res.best_col, "best_rho": res.best_rho,
                   "elim_pct": res.elim_pct, "eliminated": res.eliminated,
                   "retained": res.retained, "centers": res.centers, "h_e": info["h"],
                   "prep_ms": info["prep_ms"]},
        "phases_ms_per_step": {k: v["ms"] for k, v in phases.items()},
        "gpu_launches": launches,
        "e2e": {"value": ws * wl.extent / (e2e / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": int(wl.image.size + tmpl.size),
                "d2h_bytes_per_step": 112, "ms_per_step": e2e,
                "path": "tm_search_stream_u8 over K pinned u8 host images: per image H2D copy "
                        "(overlapped with the previous search on a copy stream) + prepare_egs "
                        "+ run_egs + tm_match_result on the host; wall clock of the K-image "
                        "call / K; L2 not flushed between the streamed images (every step "
                        "rewrites its statistics and maps before reading them)",
                "latency_ms": lat,
                "latency_path": "one tm_image_upload_u8 + tm_search_u8 call (L2 flushed "
                                "before each, wall clock)"},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--policy", default="seeded",
                    choices=["seeded", "frozen", "sequential", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--reference-budget-s", type=float, default=150.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
